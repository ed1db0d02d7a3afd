python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
CHUNK=134217728 python tools/e2e_probe.py 2>&1 | grep "double-buffered\|host ms"
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench77.json 2> gpurun_out/r02_bench77.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench77.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6)
PY
