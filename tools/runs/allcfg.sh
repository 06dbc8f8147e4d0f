for c in 1 2 3 4 5; do
  python -m paper_2009_00083_b200.cli synth --config $c --output /tmp/cfg$c.sfgb
  K=$(python -c "from paper_2009_00083_b200 import synthetic as S; C=S.CONFIGS[$c]; print(C.n_keep_max, C.n_keep_min)")
  set -- $K
  timeout 600 python -m paper_2009_00083_b200.cli bench --input /tmp/cfg$c.sfgb --keep-max $1 --keep-min $2 --repeat 1
  rm -f /tmp/cfg$c.sfgb
done
