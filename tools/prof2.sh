mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $CMD > gpurun_out/ncu_list2.log 2>&1
echo "list rc=$?"; tail -3 gpurun_out/ncu_list2.log
CMD3="python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD3 > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD3 > gpurun_out/ncu_list3.log 2>&1
echo "list3 rc=$?"
