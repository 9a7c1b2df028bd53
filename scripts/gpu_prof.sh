mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --cpu-seconds 0.1"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth_cta|k_fuzz_reset" -s 2 -c 2 -o gpurun_out/prof_cta $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
