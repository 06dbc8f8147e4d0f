for c in 1 2; do python -m paper_2009_00083_b200.cli synth --config $c --output /tmp/cfg$c.sfgb; done
for v in base t128 t64; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  for c in 1 2; do
    K=$(python -c "from paper_2009_00083_b200 import synthetic as S; C=S.CONFIGS[$c]; print(C.n_keep_max, C.n_keep_min)")
    set -- $K
    echo -n "$v cfg$c "; LTS_SM100_LIB=$L python -m paper_2009_00083_b200.cli bench --input /tmp/cfg$c.sfgb --keep-max $1 --keep-min $2 --repeat 2 | cut -c60-140
  done
done
