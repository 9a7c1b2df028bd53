# A/B of the k_label vec4 bodies: compile-time arm_dof (default) vs runtime-dof (TL_LABEL_V4GEN=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_random_records.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_dof.py -q -x --timeout 900 2>&1 | tail -3
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export TL_LABEL_V4GEN=1; else unset TL_LABEL_V4GEN; fi
  echo "V4GEN=$v"; timeout 300 python scripts/label_sizing.py $((1<<20)) 2>&1 | tail -1
done
unset TL_LABEL_V4GEN
CMD="python scripts/label_sizing.py 65536"
$CMD > gpurun_out/plain_v4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 1 -c 1 -o gpurun_out/prof_label_v4d $CMD > gpurun_out/ncu_v4d.log 2>&1
echo "ncu rc=$?"
