mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_tile or c3 or c2 or batched" > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu5.log
CMD="python bench.py --steps 2 --warmup 2 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"; cat gpurun_out/bench5.json
CMD1="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv $CMD1 > gpurun_out/ncu_list5.log 2>&1
echo "list rc=$?"
