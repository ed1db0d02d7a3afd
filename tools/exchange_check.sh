N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 tools/exchange_check.py $2 2>&1 | grep -v OMP_NUM | grep -v '^\*' > gpurun_out/exch_$N$2.log; grep -v "^ " gpurun_out/exch_$N$2.log | tail -25
