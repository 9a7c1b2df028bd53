# A/B of .so variants on the flushed bench line (bench.py --no-extras): device value, ms/step, e2e
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for round in 1 2; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  python bench.py --no-extras --cpu-seconds 0.2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']/1e9,4), round(d['ms_per_step'],5), 'e2e', round(d['e2e']['value']/1e9,4))"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
