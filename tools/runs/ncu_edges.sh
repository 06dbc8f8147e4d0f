ncu --set full --import-source on --clock-control none --cache-control none -k regex:"k_edges_tile" -c 1 -o gpurun_out/ncu_edges python tools/profile_step.py 3 1 > gpurun_out/ncu_edges.log 2>&1
tail -1 gpurun_out/ncu_edges.log
