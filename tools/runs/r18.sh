for v in base mnever nomerge; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  for i in 1 2; do LTS_SM100_LIB=$L python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v cfg3', d['ms_per_step'], d['phases_ms']['localize'], d['phases_ms']['flood_kernel'])"; done
done
