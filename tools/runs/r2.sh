set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pt_parity.log 2>&1; tail -3 gpurun_out/pt_parity.log
for c in 3 5; do python tools/kbench.py $c; LTS_NO_TMA=1 python tools/kbench.py $c; done
