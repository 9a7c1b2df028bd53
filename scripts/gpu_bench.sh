mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 3 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "rc=$?"
cat gpurun_out/bench.json; tail -20 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.json 2>&1
cat gpurun_out/bench_ref.json
nproc; lscpu | grep "Model name"
