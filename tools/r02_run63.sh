python tools/k9_phases.py 2>&1 | tail -14
