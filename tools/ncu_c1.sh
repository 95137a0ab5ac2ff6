#!/bin/bash
# --set full capture of one warm-path iteration of config 1 (second solve, iterations 6-7)
python tools/solve_once.py --config 1 --iters 7 --warm 1 > gpurun_out/ncu_pre_c1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_gather_fibers|k_block_pass|k_wcols|k_hgram|k_eig|k_fiber_areduce' \
    -s 118 -c 20 -o gpurun_out/r02_full_config1 -f python tools/solve_once.py --config 1 --iters 7 --warm 1 > gpurun_out/ncu_full_c1.log 2>&1
tail -2 gpurun_out/ncu_full_c1.log
