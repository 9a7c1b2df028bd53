mkdir -p gpurun_out
CMD="python scripts/env_bench.py 4096 200"
$CMD > gpurun_out/env_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_env_step" -s 2 -c 1 -o gpurun_out/prof_env $CMD > gpurun_out/ncu_env.log 2>&1
echo "rc=$?"; cat gpurun_out/env_plain.log; tail -3 gpurun_out/ncu_env.log
