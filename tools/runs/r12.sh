timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python tools/big_stats.py 3 max 2>&1 | sed -n 3,4p
LTS_SM100_LIB=var/lib_nopf.so python tools/big_stats.py 3 max 2>&1 | sed -n 3,4p
for i in 1 2; do python bench.py --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('pf', d['ms_per_step'], d['phases_ms']['localize'], d['phases_ms']['flood_kernel'])"
LTS_SM100_LIB=var/lib_nopf.so python bench.py --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('nopf', d['ms_per_step'], d['phases_ms']['localize'], d['phases_ms']['flood_kernel'])"; done
