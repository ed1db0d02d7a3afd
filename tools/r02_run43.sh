mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
python tools/k9_time.py; python tools/k9_time.py
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_43.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_43.log
timeout 900 python bench.py --cpu-budget 2 > gpurun_out/r02_bench43.json 2> gpurun_out/r02_bench43.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench43.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6, d['config']['stage_ms_per_step'], d['config']['async_overlap']['pipelined_ms_per_step'])
PY
