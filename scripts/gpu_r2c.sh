# round 2: validate tests + ncu evidence at the shipped configs
# (headline 4096 Place step, k_env_step at 4096, k_label at the 2^20 sizing config)
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_validate.py 2>&1 | tail -3
H="python scripts/headline_step.py 5"
$H > gpurun_out/headline_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth_cta|k_fuzz_reset" -s 2 -c 2 -o gpurun_out/r2_headline $H > gpurun_out/ncu_headline.log 2>&1
echo "headline rc=$?"; cat gpurun_out/headline_plain.log
E="python scripts/env_bench.py 4096 200"
$E > gpurun_out/env_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_env_step" -s 2 -c 1 -o gpurun_out/r2_env $E > gpurun_out/ncu_env.log 2>&1
echo "env rc=$?"; cat gpurun_out/env_plain.log
S="python scripts/label_sizing.py"
$S > gpurun_out/sizing_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 0 -c 1 -o gpurun_out/r2_label_sizing $S > gpurun_out/ncu_sizing.log 2>&1
echo "sizing rc=$?"; cat gpurun_out/sizing_plain.log
