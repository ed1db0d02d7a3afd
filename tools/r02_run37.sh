mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/exchange_overlap.py 2>&1 | grep -v OMP | grep -v '\*\*\*'
