# reset-kernel block-0 timelines (profiling + A/B build: -DTL_PROFILE -DTL_AB) for env-knob variants
cp paper_2412_13211_b200/libtrajlab_b200_prof.so /tmp/prof_orig.so 2>/dev/null
cp scripts/_ab/abprof.so paper_2412_13211_b200/libtrajlab_b200_prof.so
for v in $ENVS; do
  for n in ${NS:-4096 1024}; do echo "$v $(env $v python scripts/reset_probe.py $n)"; done
done
cp /tmp/prof_orig.so paper_2412_13211_b200/libtrajlab_b200_prof.so 2>/dev/null
