CMD="python bench.py --config C3 --steps 3 --warmup 2 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3b.csv $CMD > gpurun_out/ncu_c3.log 2>&1; echo rc=$?
cut -c1-600 gpurun_out/plain_c3.log
