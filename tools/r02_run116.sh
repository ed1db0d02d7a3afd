python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_trie.py tests/test_gpu_replay.py tests/test_gpu_finder.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for r in 1 2 3; do python tools/match_time.py 2>&1 | tail -1; done
