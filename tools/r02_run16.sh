mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_finder.py -q -x > gpurun_out/r02_pytest_finder.log 2>&1; echo "finder rc=$?"; tail -25 gpurun_out/r02_pytest_finder.log
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench16.json 2> gpurun_out/r02_bench16.err; echo "bench rc=$?"; head -c 1500 gpurun_out/r02_bench16.json; tail -5 gpurun_out/r02_bench16.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench16.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e'], 'cfg', {k: d['config'][k] for k in ('stage_ms_per_step','serial_ms_per_step','replays','match_hits')})
PY
