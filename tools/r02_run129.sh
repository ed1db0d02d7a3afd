# k_trace_ids: packed (token, rank) slots, absent tokens -> 1: N = 4 union probe, trie tests
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for i in 1 2; do timeout 600 python tools/union_match_probe.py 4 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_trace_ids --csv --log-file gpurun_out/tid4.csv python tools/union_match_probe.py 4 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "k_trace_ids" gpurun_out/tid4.csv | awk -F'","' '{print $NF}' | tail -3
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py -q -m gpu -x > gpurun_out/r02_pytest_127.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_127.log
