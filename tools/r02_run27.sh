mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"; tail -3 gpurun_out/r02_build.log
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_trie.py -q -x > gpurun_out/r02_pytest_27.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_27.log
python tools/replay_time.py 2>&1 | tail -4
python tools/pipe_clock.py 2>&1 | tail -6
