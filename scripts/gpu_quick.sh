# fast iteration: realize/fused-event-list parity at the shipped configs + multi-window
# scripts + headline step timing
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_shipped.py tests/test_gpu_parity.py -k "fuzz_ev or shipped_fuzz or window or many_events or realize or fused or g64" 2>&1 | tail -4
python scripts/headline_step.py 20
python scripts/headline_step.py 20 1024
python scripts/headline_step.py 20 4096 2 default
