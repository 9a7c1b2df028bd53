# k_label: GPU tests, sizing run for every subtask, ncu capture of the Pick sizing kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -3
for s in pick place open close; do
  echo "$s $(timeout 300 python scripts/label_sizing.py $((1<<20)) $s 2>&1 | tail -1)" | tee gpurun_out/sizing_$s.json | cut -c1-200
done
for s in pick place; do
CMD="python scripts/label_sizing.py 65536 $s"
$CMD > gpurun_out/plain_$s.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_label<float, \(int\)7, \(int\)1>' -s 1 -c 1 -o gpurun_out/prof_label_$s $CMD > gpurun_out/ncu_$s.log 2>&1
echo "ncu $s rc=$?"
done
