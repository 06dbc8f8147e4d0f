for c in 1 2; do python -m paper_2009_00083_b200.cli synth --config $c --output /tmp/cfg$c.sfgb; done
for v in base th128 th1k th4k; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  LTS_SM100_LIB=$L python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v cfg3', round(d['ms_per_step'],3), d['phases_ms']['localize'])"
  for c in 1 2; do
    K=$(python -c "from paper_2009_00083_b200 import synthetic as S; C=S.CONFIGS[$c]; print(C.n_keep_max, C.n_keep_min)")
    set -- $K
    echo -n "$v cfg$c "; LTS_SM100_LIB=$L python -m paper_2009_00083_b200.cli bench --input /tmp/cfg$c.sfgb --keep-max $1 --keep-min $2 --repeat 1 | cut -c60-110
  done
done
