timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/big_stats.py 3 max 2>&1 | tail -6
python tools/big_stats.py 3 min 2>&1 | tail -3
python bench.py --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
