mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dsa.py -q -x 2>&1 | tail -2
for N in 2 4; do for MODE in "" "--serial-union"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 5 --warmup 3 --cpu-budget 1 $MODE > gpurun_out/r02_bench88_n$N.json 2> gpurun_out/r02_bench88_n$N.err; echo "bench n$N $MODE rc=$?"
  python - $N <<'PY'
import json, sys
N = sys.argv[1]
d=json.loads(open(f'gpurun_out/r02_bench88_n{N}.json').read().strip().splitlines()[-1])
print('N', N, 'value', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), d['config'].get('stage_ms_per_step'))
PY
done; done
