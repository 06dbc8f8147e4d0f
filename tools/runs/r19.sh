timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pairs.py -x -q 2>&1 | tail -1
for i in 1 2; do python bench.py --no-cpu --no-large --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['phases_ms'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_mark_maxima|k_region_label|k_jump" -c 8 --csv python tools/profile_step.py 3 1 2>/dev/null | grep -E "k_mark|k_region|k_jump" | awk -F'","' '{print $5, $NF}' | cut -c1-80
