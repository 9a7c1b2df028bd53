# episodes per reset warp (streamed seeding) on C5 / C3
for round in 1 2; do
for epw in 2 4 8 16; do
  echo "epw=$epw c5 $(TL_RESET_EPW=$epw timeout 300 python scripts/c5_probe.py 5 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')  c3 $(TL_RESET_EPW=$epw timeout 300 python scripts/c3_probe.py 2>&1 | tail -1 | grep -o '"ms": [0-9.]*' | head -1)"
done
done
