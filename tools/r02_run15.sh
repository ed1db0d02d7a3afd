mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests/test_gpu_finder.py -q -x > gpurun_out/r02_pytest_finder.log 2>&1; echo "finder rc=$?"; tail -25 gpurun_out/r02_pytest_finder.log
python tools/replay_diag.py 2>&1 | tail -5
