# launch list of the C4 bench (1 warm-up + 1 timed + 1 profiled step: per-step = total / 3)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-c3 --cpu-budget 0.1 ${1:-}"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_now.csv $CMD > gpurun_out/ncu_list_now.log 2>&1
echo "list rc=$?"
python tools/launch_summary.py gpurun_out/launches_now.csv | head -40
