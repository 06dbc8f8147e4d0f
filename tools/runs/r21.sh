for v in base j1 j2 j5; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  LTS_SM100_LIB=$L python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],3), d['phases_ms']['discover'], d['phases_ms']['assemble'])"
done
