# k_replay rewrite: replay tests, timing, bench
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x > gpurun_out/r02_pytest_replay8.log 2>&1; echo "pytest replay rc=$?"; tail -15 gpurun_out/r02_pytest_replay8.log
python tools/replay_time.py > gpurun_out/r02_replay_time8.txt 2>&1; cat gpurun_out/r02_replay_time8.txt
timeout 900 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench8.json 2> gpurun_out/r02_bench8.err; echo "bench rc=$?"; head -c 1200 gpurun_out/r02_bench8.json; tail -5 gpurun_out/r02_bench8.err
