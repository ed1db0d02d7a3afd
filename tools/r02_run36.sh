# 2 GPUs: stream-index split test, multi tests, bench N=1 and N=2
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_multi.py tests/test_gpu_finder.py -q -x > gpurun_out/r02_pytest_36.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_pytest_36.log
for N in 1 2; do
  if [ $N = 1 ]; then timeout 900 python bench.py --cpu-budget 1 --no-c3 > gpurun_out/r02_bench36_n$N.json 2> gpurun_out/r02_bench36_n$N.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/r02_bench36_n$N.json 2> gpurun_out/r02_bench36_n$N.err; fi
  echo "bench n$N rc=$?"; tail -2 gpurun_out/r02_bench36_n$N.err
  python - $N <<'PY'
import json, sys
N = sys.argv[1]
d=json.loads(open(f'gpurun_out/r02_bench36_n{N}.json').read().strip().splitlines()[-1])
print('N', N, 'value', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), {k: d['config'].get(k) for k in ('stage_ms_per_step','serial_ms_per_step','async_overlap','exchange_pulled_bytes_per_rank')})
PY
done
