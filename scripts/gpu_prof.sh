mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15 > gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
CMD="python bench.py --steps 3 --warmup 1 --cpu-seconds 0.1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_synth|k_fuzz_reset|k_scan_emit" -s 3 -c 3 -o gpurun_out/prof_synth $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
timeout 600 python bench.py --steps 100 --warmup 3 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 600; echo; tail -3 gpurun_out/bench.err
