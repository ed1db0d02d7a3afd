# two GPUs: DSA 2-rank test, trace-exchange test, bench N=2, DSA timing
mkdir -p gpurun_out
nvidia-smi -L
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_dsa.py tests/test_gpu_multi.py -q -x > gpurun_out/r02_pytest_n2.log 2>&1; echo "pytest n2 rc=$?"; tail -5 gpurun_out/r02_pytest_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err; echo "bench n2 rc=$?"; head -c 600 gpurun_out/r02_bench_n2.json; tail -3 gpurun_out/r02_bench_n2.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench_n2.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e'], 'cfg', {k: d['config'].get(k) for k in ('stage_ms_per_step','serial_ms_per_step','async_overlap','exchange_pulled_bytes_per_rank','traces')})
PY
for c in C3 C5; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/dsa_time.py $c 2>&1 | grep '{' ; done
