#!/bin/bash
# Block-pass check on the GPU box: GPU tests, then iters/s and the per-phase split per config.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-1 2 3 4}; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err || tail -5 gpurun_out/bench_c$c.err; done
python - <<'PY'
import json, os
for c in os.environ.get("CONFIGS", "1 2 3 4").split():
    try:
        d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
        ph = {k: round(v["ms_per_step"], 2) for k, v in d["phases"].items()}
        print(c, round(d["value"]), d["iterations_per_solve"], d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), ph)
    except Exception as e:
        print(c, e)
PY
