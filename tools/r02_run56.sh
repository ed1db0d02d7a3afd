mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x > gpurun_out/r02_pytest_56.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_pytest_56.log
