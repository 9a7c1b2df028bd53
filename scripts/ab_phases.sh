# warp phase breakdown (scripts/warp_phases.py) for phases builds scripts/_ab/ph_<name>.so
for m in ${VARIANTS:-head}; do
  cp scripts/_ab/ph_$m.so paper_2412_13211_b200/libtrajlab_b200_phases.so
  echo "== $m"; python scripts/warp_phases.py ${ARGS:-4096}
done
