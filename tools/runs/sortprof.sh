python tools/sort_stats.py
ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:"k_hist|k_onesweep" -c 6 --csv python tools/kbench.py 5 > gpurun_out/sort5.csv 2>&1
ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:"k_hist|k_onesweep" -c 6 --csv python tools/kbench.py 3 > gpurun_out/sort3.csv 2>&1
grep -E "onesweep|k_hist" gpurun_out/sort5.csv | awk -F'","' '{print $5" "$(NF-2)" "$NF}' | cut -c1-150
grep -E "onesweep|k_hist" gpurun_out/sort3.csv | awk -F'","' '{print $5" "$(NF-2)" "$NF}' | cut -c1-150
