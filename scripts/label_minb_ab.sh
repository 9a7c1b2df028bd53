# A/B of k_label builds (.so files in scripts/_ab/) over the sizing run of each subtask
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  for s in ${SUBTASKS:-pick place open close}; do
    echo "$m $s $(timeout 300 python scripts/label_sizing.py $((1<<20)) $s 2>&1 | tail -1 | grep -o '"avg_launch_ms": [0-9.]*\|"frac": [0-9.]*' | tr '\n' ' ')"
  done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
