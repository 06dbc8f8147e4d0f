python tools/big_stats.py 3 max 2>&1 | tail -16
python tools/big_stats.py 3 min 2>&1 | tail -16
