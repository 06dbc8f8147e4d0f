timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for zc in 8 12 16 24 32; do echo "cfg3 zc=$zc"; LTS_CZ_ZC=$zc python tools/kbench.py 3 | grep classify; done
for zc in 32 64 128; do echo "cfg5 zc=$zc"; LTS_CZ_ZC=$zc python tools/kbench.py 5 | grep classify; done
echo minb2; LTS_SM100_LIB=var/lib_minb2.so python tools/kbench.py 3 | grep classify
