# A/B of builds (.so in scripts/_ab/) on C5 (scripts/c5_probe.py), C3 and C2 realize batches
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for round in 1 2 3; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m c5 $(timeout 300 python scripts/c5_probe.py 5 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')  c3 $(timeout 300 python scripts/c3_probe.py 2>&1 | tail -1 | grep -o '"ms": [0-9.]*' | head -1)"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
