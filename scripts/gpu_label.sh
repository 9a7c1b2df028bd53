mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -25 > gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 300 python scripts/label_sizing.py > gpurun_out/label_sizing.json 2>&1; cat gpurun_out/label_sizing.json
CMD="python scripts/label_sizing.py 65536"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 1 -c 1 -o gpurun_out/prof_label2 $CMD > gpurun_out/ncu_full3.log 2>&1
echo "rc=$?"
