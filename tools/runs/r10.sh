LTS_RANK_BUCKET=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in 3 5; do python tools/kbench.py $c | grep sort; LTS_RANK_BUCKET=1 python tools/kbench.py $c | grep sort; LTS_SM100_LIB=var/lib_rb5.so LTS_RANK_BUCKET=1 python tools/kbench.py $c | grep sort; done
