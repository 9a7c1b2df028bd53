# round evidence: GPU tests (product + checked build), default bench line, reference arm,
# ncu launch list of the bench command and --set full captures of the headline step kernels,
# the env step and the label sizing run (each after its plain command exits 0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_check_build.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --cpu-seconds 0.1 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
H="python scripts/headline_step.py 5"
$H > gpurun_out/headline_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth_warp|k_fuzz_reset|k_scan_emit" -s 3 -c 3 -o gpurun_out/r2_headline $H > gpurun_out/ncu_headline.log 2>&1
echo "headline rc=$?"
E="python scripts/env_bench.py 4096 200"
$E > gpurun_out/env_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_env_step" -s 2 -c 1 -o gpurun_out/r2_env $E > gpurun_out/ncu_env.log 2>&1
echo "env rc=$?"
S="python scripts/label_sizing.py"
$S > gpurun_out/sizing_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 0 -c 1 -o gpurun_out/r2_label_sizing $S > gpurun_out/ncu_sizing.log 2>&1
echo "sizing rc=$?"
