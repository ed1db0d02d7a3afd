python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for r in 1 2; do python tools/analysis_time.py 2>&1 | tail -1; done
