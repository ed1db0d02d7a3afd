python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
for C in 134217728 8388608 2097152 524288; do echo "chunk $C"; CHUNK=$C python tools/e2e_probe.py 2>&1 | grep "double-buffered\|host ms"; done
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench76.json 2> gpurun_out/r02_bench76.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench76.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6)
PY
