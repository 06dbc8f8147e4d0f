ncu --set full --import-source on --clock-control none -k regex:k_classify_zreg -s 3 -c 3 -o gpurun_out/ncu_zreg3 python tools/kbench.py 3 > gpurun_out/ncu_cls.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_classify_zreg -s 3 -c 3 -o gpurun_out/ncu_zreg5 python tools/kbench.py 5 >> gpurun_out/ncu_cls.log 2>&1
tail -3 gpurun_out/ncu_cls.log
