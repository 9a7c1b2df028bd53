# A/B of .so variants (scripts/_ab/<name>.so) end to end: scripts/e2e_variants.py
# (host seeds -> host labels + event lists) and the headline step, alternating
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  if [ -n "$TESTS" ]; then
    cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
    echo "$m tests: $(timeout 900 python -m pytest -q -x tests/test_gpu_shipped.py tests/test_gpu_parity.py tests/test_gpu_api.py 2>&1 | tail -1)"
  fi
done
for round in 1 2; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m | $(python scripts/headline_step.py 20 2>&1 | tail -1 | cut -d' ' -f3) | $(python scripts/e2e_variants.py 2>&1 | grep -E '^(a|d|e):' | tail -3 | awk '{print $1, $(NF-4)}' | tr '\n' ' ')"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
