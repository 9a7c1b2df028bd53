# ncu launch durations of single-step k_env_step launches (cold, serialised)
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:k_env_step -s 30 -c 6 --csv python scripts/env_bench.py ${N:-4096} 20 > /tmp/e.csv 2>/dev/null
grep -E "k_env_step" /tmp/e.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | tr -d '"' | head -20
