mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02_pytest_62.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_62.log
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench62.json 2> gpurun_out/r02_bench62.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench62.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench62.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']/1e6, 'cfg', {k: d['config'].get(k) for k in ('stage_ms_per_step','serial_ms_per_step','replays')})
PY
for k in k_window_select; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02k_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02k_$k.ncu-rep 25 > gpurun_out/r02k_ncu_$k.txt 2>&1; head -60 gpurun_out/r02k_ncu_$k.txt
done
