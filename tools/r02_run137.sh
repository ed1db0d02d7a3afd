# pinned int32 offsets exchange: publish parts at N = 4, multi tests, bench N = 2 / 4
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
bash tools/exchange_parts.sh 4
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -1
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/r02_bench137_n$N.json 2> gpurun_out/r02_bench137_n$N.err
  echo "bench n$N rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r02_bench137_n$N.json').read().strip().splitlines()[-1]); print('N $N', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), d['config'].get('stage_ms_per_step'), d['clocks'])"
done
