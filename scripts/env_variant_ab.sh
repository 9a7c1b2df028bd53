# A/B of env-step builds (.so files in scripts/_ab/) with scripts/env_bench.py
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-envbase}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  for n in ${NS:-4096 65536}; do
    echo "$m $n $(timeout 300 python scripts/env_bench.py $n 2>&1 | tail -1 | cut -c1-300)"
  done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
