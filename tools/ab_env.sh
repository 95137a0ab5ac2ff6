#!/bin/bash
# A/B of an environment setting on bench.py: ENVS="A=1 A=2" CONFIGS="1 2" bash tools/ab_env.sh
for c in ${CONFIGS:-1}; do for env in ${ENVS:-X=0}; do
  env $env timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$c', '$env', round(d['value']), {k: round(v['ms_per_step'], 2) for k, v in d['phases'].items()})" || tail -3 gpurun_out/ab.err
done; done
