# A/B of realize-kernel builds (.so files in scripts/_ab/) on the C2 batch (scripts/synth_ab.py)
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m $(timeout 300 python scripts/synth_ab.py ${N:-1024} 2>&1 | tail -1)"
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
