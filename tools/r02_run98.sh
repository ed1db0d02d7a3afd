python tools/len_stats.py 2>&1 | tail -2
