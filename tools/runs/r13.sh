for v in base t128 t512 t1024; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  LTS_SM100_LIB=$L python bench.py --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['ms_per_step'], d['phases_ms']['localize'], d['phases_ms']['flood_kernel'])"
done
LTS_SM100_LIB=var/lib_t512.so python tools/big_stats.py 3 max 2>&1 | sed -n 3,4p
LTS_SM100_LIB=var/lib_t1024.so python tools/big_stats.py 3 max 2>&1 | sed -n 3,4p
LTS_SM100_LIB=var/lib_t512.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
