# round 2, GPU run 1: host facts, full GPU test suite (incl. full-size parity), default bench
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -i "model name\|socket\|thread\|core"; nvidia-smi -L) > gpurun_out/r02_host.txt 2>&1
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err; echo "bench rc=$?"; cat gpurun_out/r02_bench1.json | head -c 3000
