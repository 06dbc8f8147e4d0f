timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/sort_stats.py
for c in 3 5; do python tools/kbench.py $c; done
