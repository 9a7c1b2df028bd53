# warp phase breakdown of the A/B phases build under env knobs: ENVS="A=1 B=2" ARGS="1024"
cp scripts/_ab/ph_ab.so paper_2412_13211_b200/libtrajlab_b200_phases.so
for v in $ENVS; do echo "== $v"; env $v python scripts/warp_phases.py ${ARGS:-1024}; done
for v in $ENVS; do echo "== $v"; env $v python scripts/warp_timeline.py ${ARGS:-1024}; done
