# GPU tests (shipped/parity/env/dof/api) of the A/B build with env knobs: ENVS="A=1"
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/ab.so paper_2412_13211_b200/libtrajlab_b200.so
for v in $ENVS; do
  echo "$v tests: $(env $v timeout 900 python -m pytest -q -x tests/test_gpu_shipped.py tests/test_gpu_parity.py tests/test_gpu_env.py tests/test_gpu_dof.py tests/test_gpu_api.py 2>&1 | tail -2 | tr '\n' ' ')"
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
