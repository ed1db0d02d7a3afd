mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trie.py -x -q --durations=5 > gpurun_out/pytest_trie.log 2>&1; echo "trie rc=$?"; tail -25 gpurun_out/pytest_trie.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "parity rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --cpu-budget 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; cat gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
