# A/B of k_label variants (records per lane x blocks of 8 warps per SM); .so files in scripts/_ab/
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-r4m2 r4m4 r2m2 r2m3 r2m4 r2m5 r2m6}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m $(timeout 300 python scripts/label_sizing.py $((1<<20)) 2>&1 | tail -1 | cut -c80-200)"
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
