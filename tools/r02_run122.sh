# k_ht_insert / k_trace_ids with 4 tokens per thread: parity, bench, launch list
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r02_pytest_122.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_122.log
for i in 1 2; do timeout 600 python bench.py --no-c3 > gpurun_out/r02_bench122_$i.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02_bench122_$i.json').read().strip().splitlines()[-1]); print('ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,1), d['config'].get('stage_ms_per_step'), d['clocks'])"; done
CUDA_VISIBLE_DEVICES=0 bash tools/prof_list.sh > gpurun_out/r02_list122.log 2>&1; grep -E "ht_insert|trace_ids|list rc" gpurun_out/r02_list122.log
