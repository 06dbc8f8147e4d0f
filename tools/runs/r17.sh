timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in 1 2; do python -m paper_2009_00083_b200.cli synth --config $c --output /tmp/cfg$c.sfgb; done
for v in base avg40 nomerge; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  LTS_SM100_LIB=$L python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v cfg3', d['ms_per_step'], d['phases_ms']['localize'], d['phases_ms']['flood_kernel'])"
  for c in 1 2; do
    K=$(python -c "from paper_2009_00083_b200 import synthetic as S; C=S.CONFIGS[$c]; print(C.n_keep_max, C.n_keep_min)")
    set -- $K
    echo -n "$v cfg$c "; LTS_SM100_LIB=$L python -m paper_2009_00083_b200.cli bench --input /tmp/cfg$c.sfgb --keep-max $1 --keep-min $2 --repeat 2 | cut -c60-140
  done
done
