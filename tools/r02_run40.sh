mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_trie.py -q -x -k indexed > gpurun_out/r02_pytest_40.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_40.log
python tools/replay_heavy.py 2>&1 | tail -4
