mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_pytest_gpu4.log
python tools/k9_phases.py > gpurun_out/r02_k9_phases4.txt 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_k9_phases4.txt
timeout 600 python bench.py --cpu-budget 2 --no-c3 > gpurun_out/r02_bench4.json 2> gpurun_out/r02_bench4.err; echo "bench rc=$?"; head -c 900 gpurun_out/r02_bench4.json; tail -3 gpurun_out/r02_bench4.err
