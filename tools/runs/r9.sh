ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:"k_rank|onesweep" -c 6 --csv python tools/kbench.py 5 > gpurun_out/rank5.csv 2>&1
tail -2 gpurun_out/rank5.csv
