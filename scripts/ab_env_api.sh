# env API (scripts/env_bench.py 4096 200) for .so variants in scripts/_ab/; TESTS=1 runs tests/test_gpu_env.py per variant
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  [ -n "$TESTS" ] && echo "$m tests: $(timeout 600 python -m pytest -q -x tests/test_gpu_env.py 2>&1 | tail -1)"
  for r in 1 2; do echo "$m $(timeout 300 python scripts/env_bench.py ${N:-4096} 200 2>&1 | tail -1)"; done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
