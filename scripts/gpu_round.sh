mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -25 > gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 3 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/gpu_tests.log | tail -25; tail -3 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
