python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench79.json 2> gpurun_out/r02_bench79.err; echo "bench rc=$?"; tail -2 gpurun_out/r02_bench79.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench79.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6)
PY
