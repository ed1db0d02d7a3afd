# K9 rework: GPU suite + bench
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/r02_pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r02_pytest_gpu2.log
timeout 600 python bench.py --cpu-budget 2 > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench rc=$?"; head -c 1500 gpurun_out/r02_bench2.json; tail -5 gpurun_out/r02_bench2.err
