mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_96.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_96.log
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench96.json 2> gpurun_out/r02_bench96.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench96.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6, 'cfg', {k: d['config'].get(k) for k in ('stage_ms_per_step',)})
PY
timeout 900 bash tools/prof_kernel.sh k_window_sa 0 r02p_k_window_sa > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02p_k_window_sa.ncu-rep 16 > gpurun_out/r02p_ncu_k_window_sa.txt 2>&1; head -30 gpurun_out/r02p_ncu_k_window_sa.txt
