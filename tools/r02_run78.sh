python tools/ce_probe3.py 2>&1 | tail -4
