N=${1:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 tools/exchange_parts.py 2>&1 | grep -v OMP_NUM | grep -v '^\*' | grep "ms\|Error" | tail -5
