# full GPU test suite + headline step + bench line (one call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -5
python scripts/headline_step.py 20
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value %.4g ms/step %.4f e2e %.4g frac %.4f c2 %.4f c3 %.4f/%.4f c5 %.2f env1 %.3f envK %.3f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['c2_1024']['ms'], d['c3']['open']['ms'], d['c3']['close']['ms'], d['c5']['ms'], d['env_api']['one_launch']['ms'], d['env_api']['per_step_launch']['ms']))
"; tail -3 gpurun_out/bench.err
