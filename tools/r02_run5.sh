mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x > gpurun_out/r02_pytest_replay.log 2>&1; echo "pytest replay rc=$?"; tail -30 gpurun_out/r02_pytest_replay.log
python tools/replay_time.py > gpurun_out/r02_replay_time.txt 2>&1; cat gpurun_out/r02_replay_time.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_pytest_gpu5.log
bash tools/prof_list.sh > gpurun_out/r02_list.log 2>&1; tail -3 gpurun_out/r02_list.log
