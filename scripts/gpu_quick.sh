# fast iteration: fused-event-list parity at the shipped configs + headline step timing
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_shipped.py -k "fuzz_ev or shipped_fuzz" 2>&1 | tail -25
python scripts/headline_step.py 20
python scripts/headline_step.py 20 1024
python scripts/headline_step.py 20 4096 2 default
