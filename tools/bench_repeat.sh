#!/bin/bash
# Repeat short bench runs to see run-to-run stability: N=4 CONFIG=1 STEPS=5 bash tools/bench_repeat.sh
for i in $(seq 1 ${N:-4}); do
  python bench.py --config ${CONFIG:-1} --steps ${STEPS:-5} --no-cpu-baseline --no-per-config > gpurun_out/rep.json 2> gpurun_out/rep.err
  python -c "
import json
d=json.loads(open('gpurun_out/rep.json').read().strip().splitlines()[-1])
print('${CONFIG:-1}', '$BENCH_NO_CLOCKS', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['roofline']['kernel'][:20], round(d['roofline']['frac'],3), d['clocks'].get('samples'))" || tail -3 gpurun_out/rep.err
done
