# exchange parts at N = 2 / 4 (max over ranks)
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for N in 4 2; do
  echo "N=$N"; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N tools/exchange_overlap.py 2>&1 | grep " ms\|Error" | tail -8
done
