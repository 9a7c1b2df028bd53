for g in ${GS:-16 4 8 16 4 8}; do
  echo "grid/SM=$g $(TL_LABEL_GRID_PER_SM=$g timeout 300 python scripts/label_sizing.py $((1<<20)) pick 2>&1 | tail -1 | grep -o '"avg_launch_ms": [0-9.]*\|"frac": [0-9.]*' | tr '\n' ' ')"
done
