mkdir -p gpurun_out
for s in ${SUBTASKS:-pick place}; do
CMD="python scripts/label_sizing.py 65536 $s"
$CMD > gpurun_out/plain_$s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 1 -c 1 -o gpurun_out/prof_label_$s $CMD > gpurun_out/ncu_$s.log 2>&1
echo "ncu $s rc=$?"
done
