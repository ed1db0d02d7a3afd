# trie keeps only reversed traces: trie/replay/multi/parity tests, bench N = 1 / 2 / 4
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_132.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_132.log
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 900 python bench.py --no-c3 > gpurun_out/r02_bench132_n$N.json 2> gpurun_out/r02_bench132_n$N.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/r02_bench132_n$N.json 2> gpurun_out/r02_bench132_n$N.err; fi
  echo "bench n$N rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r02_bench132_n$N.json').read().strip().splitlines()[-1]); print('N $N', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), d['config'].get('stage_ms_per_step'), d['clocks'])"
done
