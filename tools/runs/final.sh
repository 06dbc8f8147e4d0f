set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/profile_step.py 3 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_cfg3.csv 0.5 > gpurun_out/launches_cfg3_summary.txt
ncu --set full --import-source on --clock-control none -k regex:"k_hist|k_onesweep|k_classify_zreg|k_big_flood|k_edges_tile" -c 16 -o gpurun_out/prof_r01d python tools/profile_step.py 3 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/prof_r01d.ncu-rep gpurun_out/ncu_traffic.json
bash tools/runs/allcfg.sh > gpurun_out/allcfg.log 2>&1
head -c 300 gpurun_out/bench.json
