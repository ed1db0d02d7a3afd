# round-2 evidence: full GPU suite, default bench, launch list, ncu full captures
mkdir -p gpurun_out
(nproc; lscpu | grep -i "model name"; nvidia-smi -L) > gpurun_out/r02_host.txt 2>&1
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r02_pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/r02_pytest_gpu_final.log
timeout 900 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench_final.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02_bench_final.json').read().strip().splitlines()[-1])
print('value', d['value']/1e6, 'ms', d['ms_per_step'], 'e2e', d['e2e'], 'roof', d['roofline']['frac'], d['roofline']['achieved'], 'c3', d['c3']['value']/1e6, 'cpu', d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])
PY
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/r02_bench_reference.json
bash tools/prof_list.sh > gpurun_out/r02_list39.log 2>&1; head -30 gpurun_out/r02_list39.log; cp gpurun_out/launches_now.csv gpurun_out/launches_39.csv
for k in k_window_sa k_stream_match k_stream_emit k_rp_decide; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02f_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02f_$k.ncu-rep 16 > gpurun_out/r02f_ncu_$k.txt 2>&1; head -30 gpurun_out/r02f_ncu_$k.txt
done
