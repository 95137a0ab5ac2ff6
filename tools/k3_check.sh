#!/bin/bash
# K3 quick check on the GPU box: the K3 tests, then the K3 roofline of every BASELINE config >= 1.
python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_k3.log 2>&1; tail -3 gpurun_out/pytest_k3.log
for c in ${CONFIGS:-1 2 3 4}; do python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
python - <<'PY'
import json, os
for c in os.environ.get("CONFIGS", "1 2 3 4").split():
    try:
        d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
        k = d["full_tensor_rooflines"]["k3_full"]
        print(c, round(d["value"]), "k3 us", round(k["launch_us"]), "GB/s", round(k["achieved"]), "frac", round(k["frac"], 3))
    except Exception as e:
        print(c, e)
PY
