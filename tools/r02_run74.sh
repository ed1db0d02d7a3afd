python tools/ce_probe2.py 2>&1 | tail -6
