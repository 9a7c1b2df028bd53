# round 2: validate kernel tests, writer tests, filter manifest tests; then
# compute-sanitizer over every entry point (logs -> gpurun_out/sanitize_*.log)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_validate.py tests/test_io_golden.py tests/test_host_messages.py \
  "tests/test_gpu_api.py::test_filter_manifest_bytes_vs_reference" 2>&1 | tail -15
python tests/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/sanitize_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  for c in fuzz_ev fuzz label env filter validate predicates; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tests/sanitize_cases.py $c \
      > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${c}.log | tail -1)"
  done
done
