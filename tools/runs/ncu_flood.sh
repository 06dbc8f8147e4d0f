ncu --set full --import-source on --clock-control none -k regex:k_big_flood -s 1 -c 1 -o gpurun_out/ncu_flood python tools/profile_step.py 3 1 > gpurun_out/ncu_flood.log 2>&1
tail -2 gpurun_out/ncu_flood.log
