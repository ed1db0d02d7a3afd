python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "edge_windows or fused" 2>&1 | tail -3
