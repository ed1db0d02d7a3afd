mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"; tail -2 gpurun_out/r02_build.log
timeout 900 python -m pytest tests/test_gpu_dsa.py -q -x > gpurun_out/r02_pytest_dsa2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_pytest_dsa2.log
for c in C3 C5; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/dsa_time.py $c 2>&1 | grep '{' ; done
