# A/B of env-var knobs on the probe build (scripts/_ab/ab.so, -DTL_AB): ENVS="A=1 A=2 ..."
# on the headline step configs (4096 / 1024 Place long, 4096 Open default), alternating twice
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
for round in 1 2; do
for v in $ENVS; do
  echo "$v | $(env $v python scripts/headline_step.py 20 2>&1 | tail -1 | cut -d' ' -f3) | $(env $v python scripts/headline_step.py 20 1024 2>&1 | tail -1 | cut -d' ' -f3) | $(env $v python scripts/headline_step.py 20 4096 2 default 2>&1 | tail -1 | cut -d' ' -f3)"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
