for c in 3 5; do python tools/kbench.py $c | grep sort; LTS_SM100_LIB=var/lib_match.so python tools/kbench.py $c | grep sort; done
LTS_SM100_LIB=var/lib_match.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "order or golden" 2>&1 | tail -1
