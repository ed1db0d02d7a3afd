mkdir -p gpurun_out
CMD="python bench.py --config C3 --steps 3 --warmup 3 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_c3.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_c3.log 2>&1; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/plain_c3.json').read().strip().splitlines()[-1])
print(round(d['value']/1e6,1), 'Mops/s', round(d['ms_per_step'],3), 'ms', d['gpu_launches'], 'launches', d['roofline_hbm'] if 'roofline_hbm' in d else d['roofline'])"
python tools/launch_summary.py gpurun_out/launches_c3.csv | head -30
