for v in base k20 k12 t512; do
  if [ $v = base ]; then L=""; else L="var/lib_$v.so"; fi
  echo -n "$v "; LTS_SM100_LIB=$L python tools/kbench.py 3 | grep sort
done
LTS_SM100_LIB=var/lib_k20.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "order" 2>&1 | tail -1
