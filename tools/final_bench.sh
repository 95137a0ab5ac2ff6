#!/bin/bash
# Round-end evidence: default bench line (driver arguments), the reference arm, every BASELINE
# config, and the launch list of the default command (ncu, cold-cache serialised launches:
# shares, not absolutes).
python bench.py --steps 20 --warmup 5 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
python bench.py --config 0 --steps 20 --warmup 5 --no-per-config > gpurun_out/final_c0.json 2> gpurun_out/final_c0.err
for c in 2 3 4; do python bench.py --config $c --no-cpu-baseline --no-per-config > gpurun_out/final_c$c.json 2> gpurun_out/final_c$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/final_ncu.log 2>&1
for c in 0 1 2 3 4; do python -c "
import json
d=json.loads(open('gpurun_out/final_c$c.json').read().strip().splitlines()[-1])
print($c, round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), 'k3', round(d['full_tensor_rooflines']['k3_full']['frac'],3), d['clocks'])
"; done
tail -c 400 gpurun_out/final_ref.json
