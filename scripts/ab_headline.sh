# A/B of .so variants (scripts/_ab/<name>.so) on the headline step configs, alternating twice;
# TESTS=1 also runs the fused-event-list / shipped-config parity tests per variant
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  if [ -n "$TESTS" ]; then
    cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
    echo "$m tests: $(timeout 600 python -m pytest -q -x tests/test_gpu_shipped.py tests/test_gpu_parity.py -k 'fuzz_ev or shipped_fuzz or fused or window or many_events' 2>&1 | tail -1)"
  fi
done
for round in 1 2; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  echo "$m | $(python scripts/headline_step.py 20 2>&1 | tail -1 | cut -d' ' -f3) | $(python scripts/headline_step.py 20 1024 2>&1 | tail -1 | cut -d' ' -f3) | $(python scripts/headline_step.py 20 4096 2 default 2>&1 | tail -1 | cut -d' ' -f3)"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
