python tools/bigram_stats.py 2>&1 | tail -3
