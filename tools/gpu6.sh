mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trie.py tests/test_gpu_parity.py -x -q -k "trie or match or c4 or batched or c1" > gpurun_out/pytest6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest6.log
timeout 600 python bench.py --steps 3 --warmup 2 --cpu-budget 1 --no-e2e > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?"; cut -c1-900 gpurun_out/bench6.json; tail -3 gpurun_out/bench6.err
bash tools/gpu_multi.sh 2 2>&1 | tail -4 | cut -c1-900
