#!/bin/bash
# Round-2 ncu evidence (run under gpurun; each command only after the same command exited 0 without ncu):
#   1. launch list of the default bench command (gpu__time_duration.sum per launch)
#   2. --set full captures of the sampled-block passes at configs 1, 2, 4 (one steady-state iteration each)
set -x
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_pre_bench.json 2> gpurun_out/ncu_pre_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_launches_config1_v2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_launches.log 2>&1
for c in 1 2 4; do
  python tools/solve_once.py --config $c --iters 7 --warm 1 > gpurun_out/ncu_pre_c$c.log 2>&1 || exit 1
done
# config 1: iteration 7 of the second solve (warm eigensolver path): skip the first solve's launches
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_gather_fibers|k_block_pass|k_wcols|k_hgram|k_eig|k_fiber_areduce' \
    -s 160 -c 16 -o gpurun_out/r02_full_config1 -f python tools/solve_once.py --config 1 --iters 7 --warm 1 > gpurun_out/ncu_full_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass' \
    -s 28 -c 6 -o gpurun_out/r02_full_config2 -f python tools/solve_once.py --config 2 --iters 7 --warm 1 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_block_pass|k_gather' \
    -s 60 -c 12 -o gpurun_out/r02_full_config4 -f python tools/solve_once.py --config 4 --iters 7 --warm 1 > gpurun_out/ncu_full_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep
