# warp phase breakdown for phases A/B builds scripts/_ab/<name>.so under env knobs
for m in $SOS; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200_phases.so
  for v in $ENVS; do echo "== $m $v"; env $v python scripts/warp_phases.py ${ARGS:-1024} | head -7; done
done
