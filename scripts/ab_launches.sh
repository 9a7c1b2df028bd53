# per-kernel durations (ncu launch list, cold serialised) of the headline step for env-knob variants
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
mkdir -p gpurun_out
for v in $ENVS; do
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 9 --csv python scripts/headline_step.py 3 ${N:-4096} > /tmp/l.csv 2>/dev/null
  echo "$v: $(grep -E 'k_' /tmp/l.csv | awk -F'","' '{split($5,a,"(");print a[1], $NF}' | tr -d '"' | tr '\n' ';')"
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
