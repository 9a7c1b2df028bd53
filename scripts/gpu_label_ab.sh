mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x --timeout 600 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export TL_LABEL_TMA=1; fi
  echo "TMA=$v"; timeout 300 python scripts/label_sizing.py 2>&1 | tail -1
done
unset TL_LABEL_TMA
CMD="python scripts/label_sizing.py 65536"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_label" -s 1 -c 1 -o gpurun_out/prof_label_pf $CMD > gpurun_out/ncu_full3.log 2>&1
echo "ncu rc=$?"
