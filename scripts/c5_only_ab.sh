# C5 A/B of .so variants in scripts/_ab/, alternating, 4 rounds
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for round in 1 2 3 4; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m c5 $(timeout 300 python scripts/c5_probe.py 8 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
