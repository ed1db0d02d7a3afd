# 4 GPUs: final scaling lines N=1,2,4 (serial headline), multi tests
mkdir -p gpurun_out
nvidia-smi -L
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_dsa.py tests/test_gpu_multi.py -q -x > gpurun_out/r02_pytest_n4f.log 2>&1; echo "pytest multi rc=$?"; tail -3 gpurun_out/r02_pytest_n4f.log
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 900 python bench.py --cpu-budget 2 > gpurun_out/r02_bench_final_n$N.json 2> gpurun_out/r02_bench_final_n$N.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N > gpurun_out/r02_bench_final_n$N.json 2> gpurun_out/r02_bench_final_n$N.err; fi
  echo "bench n$N rc=$?"
  python - $N <<'PY'
import json, sys
N = sys.argv[1]
d=json.loads(open(f'gpurun_out/r02_bench_final_n{N}.json').read().strip().splitlines()[-1])
print('N', N, 'value', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), {k: d['config'].get(k) for k in ('stage_ms_per_step','exchange_pulled_bytes_per_rank','traces')}, d['config']['async_overlap']['pipelined_ms_per_step'], d['clocks'])
PY
done
