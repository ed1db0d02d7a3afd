# matcher: tail trips without the cached-head select: tests + kernel time
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py -q -m gpu -x > gpurun_out/r02_pytest_144.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02_pytest_144.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_stream_match_ids --csv --log-file gpurun_out/sm.csv python tools/union_match_probe.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "k_stream_match_ids" gpurun_out/sm.csv | awk -F'","' '{print $NF}' | tail -3
