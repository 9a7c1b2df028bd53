# A/B of k_fuzz_reset modes / episodes per warp on C5 (scripts/c5_probe.py)
for cfg in "1 8" "2 8" "2 16" "1 8" "2 8" "2 16"; do
  set -- $cfg
  echo "mode=$1 epw=$2 $(TL_RESET_MODE=$1 TL_RESET_EPW=$2 timeout 300 python scripts/c5_probe.py 3 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')"
done
