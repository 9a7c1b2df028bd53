mkdir -p gpurun_out
CMD="python scripts/label_sizing.py 65536"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 1 -c 1 -o gpurun_out/prof_label $CMD > gpurun_out/ncu_full3.log 2>&1
echo "rc=$?"; cat gpurun_out/plain3.log
