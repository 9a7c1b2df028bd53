# env API timing (scripts/env_bench.py) of the A/B build under env knobs: ENVS="A=1 B=2"
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
for v in $ENVS; do
  for r in 1 2; do echo "$v $(env $v timeout 300 python scripts/env_bench.py ${N:-4096} 200 2>&1 | tail -1 | cut -c1-220)"; done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
