# A/B of .so variants in scripts/_ab/ on the bench headline (value, e2e), alternating
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for round in 1 2; do
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  python bench.py --cpu-seconds 0.1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']/1e9,4), round(d['e2e']['value']/1e9,4), round(d['ms_per_step'],5), 'c5', round(d['c5']['ms'],2), 'c3', round(d['c3']['open']['ms'],4))"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
