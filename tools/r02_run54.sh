python tools/replay_counts.py 2>&1 | tail -5
