mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10.csv $CMD1 > gpurun_out/ncu_list6.log 2>&1
echo "list rc=$?"
