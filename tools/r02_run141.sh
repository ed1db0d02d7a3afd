# k_stream_ends segments + on-chip root lengths: full GPU suite, bench N = 1
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_pytest_141.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_141.log
timeout 600 python bench.py --no-c3 > gpurun_out/r02_bench141_n1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02_bench141_n1.json').read().strip().splitlines()[-1]); print('ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,1), d['config'].get('stage_ms_per_step'), d['clocks'])"
