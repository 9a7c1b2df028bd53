# A/B of the realize CTA wave size (TL_SYNTH_WAVE=64 forces the 3-warp CTA) on C5 / C3 / C2
for round in 1 2; do
for w in 64 32; do
  echo "W=$w c5 $(TL_SYNTH_WAVE=$w timeout 300 python scripts/c5_probe.py 5 2>&1 | tail -1 | grep -o '"ms": [0-9.]*')  c3 $(TL_SYNTH_WAVE=$w timeout 300 python scripts/c3_probe.py 2>&1 | tail -1 | grep -o '"ms": [0-9.]*' | head -1)"
done
done
