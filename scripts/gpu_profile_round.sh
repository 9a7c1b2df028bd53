# ncu evidence for profiles/: launch list of the bench command and one
# --set full capture of the C2 step kernels (each after the plain run exits 0)
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --cpu-seconds 0.1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth_cta|k_fuzz_reset" -s 4 -c 2 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
