# round-end evidence: GPU tests, the default bench line, smoke, ncu launch
# list + one --set full capture of the step kernels (after plain runs exit 0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3 > gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
bash scripts/gpu_profile_round.sh
