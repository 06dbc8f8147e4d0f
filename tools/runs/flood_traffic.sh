ncu --set full --clock-control none -k regex:"k_big_flood" -c 3 -o gpurun_out/prof_r01e python tools/profile_step.py 3 1 > gpurun_out/ncu_flood2.log 2>&1
python tools/ncu_traffic.py gpurun_out/prof_r01e.ncu-rep gpurun_out/ncu_traffic_flood.json
