# C5 (1M fuzz episodes -> labels -> filter) under env-knob variants of the A/B build
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
for round in 1 2; do
for v in $ENVS; do
  echo "$v c5 $(env $v timeout 300 python scripts/c5_probe.py 5 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
