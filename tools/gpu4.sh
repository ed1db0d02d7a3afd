mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trie.py -x -q --durations=5 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu4.log
timeout 900 python bench.py --steps 3 --warmup 2 --cpu-budget 2 --no-e2e > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"; cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --cpu-budget 1 --no-e2e > gpurun_out/bench4_c3.json 2> gpurun_out/bench4_c3.err; echo "c3 rc=$?"; cat gpurun_out/bench4_c3.json
