# ncu --set full capture of the headline step kernels (k_fuzz_reset + k_synth_cta) at 4096 envs
mkdir -p gpurun_out
H="python scripts/headline_step.py 5"
$H > gpurun_out/headline_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth_warp|k_fuzz_reset" -s 2 -c 2 -o gpurun_out/r2_headline_b $H > gpurun_out/ncu_headline.log 2>&1
echo "headline rc=$?"; cat gpurun_out/headline_plain.log; tail -3 gpurun_out/ncu_headline.log
