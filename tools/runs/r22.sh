timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for c in 2 5; do python -m paper_2009_00083_b200.cli synth --config $c --output /tmp/cfg$c.sfgb; done
for v in base nomerge; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  for i in 1 2; do LTS_SM100_LIB=$L python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v cfg3', round(d['ms_per_step'],3), d['phases_ms']['flood_kernel'])"; done
  for c in 2 5; do
    K=$(python -c "from paper_2009_00083_b200 import synthetic as S; C=S.CONFIGS[$c]; print(C.n_keep_max, C.n_keep_min)")
    set -- $K
    echo -n "$v cfg$c "; LTS_SM100_LIB=$L python -m paper_2009_00083_b200.cli bench --input /tmp/cfg$c.sfgb --keep-max $1 --keep-min $2 --repeat 1 | cut -c60-120
  done
done
