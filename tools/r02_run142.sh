# k_tree_par with a 1,024-deep on-chip stack (more warps per SM): tests + kernel time
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py -q -m gpu -x > gpurun_out/r02_pytest_142.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_142.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tree_par|k_tree_sweep" --csv --log-file gpurun_out/tp.csv python tools/union_match_probe.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "k_tree_par|k_tree_sweep" gpurun_out/tp.csv | awk -F'","' '{print $5, $NF}' | cut -c1-20,200- | tail -4
