# like ab_env.sh for a named A/B build: SO=<name> ENVS="..."
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
cp scripts/_ab/${SO:-ab}.so paper_2412_13211_b200/libtrajlab_b200.so
for round in 1 2; do
for v in $ENVS; do
  echo "${SO:-ab} $v | $(env $v python scripts/headline_step.py 20 2>&1 | tail -1 | cut -d' ' -f3) | $(env $v python scripts/headline_step.py 20 1024 2>&1 | tail -1 | cut -d' ' -f3) | $(env $v python scripts/headline_step.py 20 4096 2 default 2>&1 | tail -1 | cut -d' ' -f3) | $(env $v python scripts/headline_step.py 10 16384 2>&1 | tail -1 | cut -d' ' -f3)"
done
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
