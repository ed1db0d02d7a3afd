mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
python tools/replay_diag.py 2>&1 | tail -3
python tools/k9_time.py
for cfg in C3 C5; do for v in "" k1match; do
  if [ -n "$v" ]; then export APO_LIB=tools/variants/libapo_$v.so; else unset APO_LIB; fi
  python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --cpu-budget 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', '$v', round(d['value']/1e6,1), 'Mops/s', round(d['ms_per_step'],3), 'ms')"
done; done
unset APO_LIB
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_gpu14.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu14.log
