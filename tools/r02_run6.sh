# round 2 re-entry: GPU suite + default bench of HEAD (state check after container re-creation)
mkdir -p gpurun_out
(nproc; lscpu | grep -i "model name"; nvidia-smi -L) > gpurun_out/r02_host.txt 2>&1
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/r02_pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/r02_pytest_gpu6.log
timeout 900 python bench.py > gpurun_out/r02_bench6.json 2> gpurun_out/r02_bench6.err; echo "bench rc=$?"; head -c 4000 gpurun_out/r02_bench6.json; tail -5 gpurun_out/r02_bench6.err
python tools/k9_phases.py > gpurun_out/r02_k9_phases6.txt 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_k9_phases6.txt
