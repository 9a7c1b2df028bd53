mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -25 > gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 100 --warmup 3 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.3g ms/step %.4f e2e %.3g synth_ms %.4f frac %.4f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac']))
" ; tail -3 gpurun_out/bench.err
CMD="python bench.py --steps 3 --warmup 1 --cpu-seconds 0.1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
grep -E "k_synth|k_fuzz|k_scan_emit" gpurun_out/launches.csv | awk -F'","' '{print $5, $NF}' | head -12
