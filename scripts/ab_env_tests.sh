# parity tests of the A/B build under each env-knob variant: ENVS="A=1 B=2"
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
for v in $ENVS; do
  echo "$v tests: $(env $v timeout 600 python -m pytest -q -x tests/test_gpu_shipped.py tests/test_gpu_parity.py -k "${TESTK:-fuzz or window or realize or many}" 2>&1 | tail -1)"
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
