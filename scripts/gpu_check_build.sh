# memory-safety evidence without compute-sanitizer (closed on this GPU pool):
# the checked build (-DTL_CHECK: bounds / invariant asserts that trap) runs the
# whole GPU test suite and the sanitizer cases; a failed check kills the test.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -shared -DTL_CHECK -I include -o /tmp/libtrajlab_b200_check.so paper_2412_13211_b200/csrc/trajlab_b200.cu
export TRAJLAB_B200_LIB=/tmp/libtrajlab_b200_check.so
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -3 > gpurun_out/check_build_tests.log
cat gpurun_out/check_build_tests.log
for c in fuzz_ev fuzz label env filter validate predicates; do
  timeout 300 python tests/sanitize_cases.py $c 2>&1 | tail -1
done > gpurun_out/check_build_cases.log
cat gpurun_out/check_build_cases.log
