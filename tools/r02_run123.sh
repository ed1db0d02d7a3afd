# final evidence: full GPU suite, bench N=1 (with C3), N=2, N=4, reference arm, launch list, matcher capture
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_pytest_gpu_123.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_123.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 900 python bench.py > gpurun_out/r02_bench123_n$N.json 2> gpurun_out/r02_bench123_n$N.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2930$N bench.py --gpus $N --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/r02_bench123_n$N.json 2> gpurun_out/r02_bench123_n$N.err; fi
  echo "bench n$N rc=$?"
  python - $N <<'PY'
import json, sys
N = sys.argv[1]
d=json.loads(open(f'gpurun_out/r02_bench123_n{N}.json').read().strip().splitlines()[-1])
c3 = d.get('c3')
print('N', N, 'value', round(d['value']/1e6,1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,1), {k: d['config'].get(k) for k in ('stage_ms_per_step','serial_ms_per_step')}, d['clocks'], 'c3', None if not c3 else round(c3['value']/1e6,1), 'roof', round(d['roofline']['frac'],4), 'launches', d['gpu_launches'])
PY
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench123_reference.json 2>&1; echo "ref rc=$?"
CUDA_VISIBLE_DEVICES=0 bash tools/prof_list.sh > gpurun_out/r02_list123.log 2>&1; head -40 gpurun_out/r02_list123.log; cp gpurun_out/launches_now.csv gpurun_out/launches_123.csv
CUDA_VISIBLE_DEVICES=0 timeout 900 bash tools/prof_kernel.sh k_stream_match_ids 0 r02r_k_stream_match_ids > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02r_k_stream_match_ids.ncu-rep 16 > gpurun_out/r02r_ncu_k_stream_match_ids.txt 2>&1; head -12 gpurun_out/r02r_ncu_k_stream_match_ids.txt
