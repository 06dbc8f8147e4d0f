timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for i in 1 2; do python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['phases_ms']['discover'], [p['boruvka_rounds'] for p in d['report']['passes']])"; done
