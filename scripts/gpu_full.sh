# full GPU evidence pass: product tests, checked-build tests, default bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3 > gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
bash scripts/gpu_check_build.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.4g ms/step %.4f e2e %.4g frac %.4f c2 %.4f c3 %.4f c5 %.2f env1 %.3g' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['c2_1024']['ms'], d['c3']['open']['ms'], d['c5']['ms'], d['env_api']['per_step_launch']['env_steps_per_s']))
"; tail -3 gpurun_out/bench.err
