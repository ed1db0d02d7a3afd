mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_104.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_104.log
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench104.json 2> gpurun_out/r02_bench104.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench104.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench104.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6, 'cfg', {k: d['config'].get(k) for k in ('stage_ms_per_step','serial_ms_per_step','replays')})
PY
