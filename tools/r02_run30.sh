mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_30.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_30.log
for cfg in C2 C3 C5; do python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value']/1e6,1), 'Mops/s', round(d['ms_per_step'],3), 'ms', d['gpu_launches'], 'launches', round(d['roofline_hbm']['frac'],3))"; done
