#!/bin/bash
# --set full captures of the sampled-block kernels on the round's final build (configs 1, 2, 4)
for c in 1 2 4; do python tools/solve_once.py --config $c --iters 7 --warm 1 > gpurun_out/ncu_pre_c$c.log 2>&1 || exit 1; done
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_gather_fibers|k_block_pass|k_wcols|k_hgram|k_eig|k_fiber_areduce' \
    -s 118 -c 20 -o gpurun_out/r02_full_config1 -f python tools/solve_once.py --config 1 --iters 7 --warm 1 > gpurun_out/ncu_full_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_fiber_areduce' \
    -s 40 -c 8 -o gpurun_out/r02_full_config2 -f python tools/solve_once.py --config 2 --iters 7 --warm 1 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_fiber_pass|k_block_pass|k_gather' \
    -s 60 -c 12 -o gpurun_out/r02_full_config4 -f python tools/solve_once.py --config 4 --iters 7 --warm 1 > gpurun_out/ncu_full_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -2 gpurun_out/ncu_full_c1.log
# summaries on the box (the reports together exceed what gpurun copies back)
for c in 1 2 4; do
  python tools/ncu_raw_subset.py gpurun_out/r02_full_config$c.ncu-rep > gpurun_out/r02_ncu_config${c}_v3_raw.csv
  python tools/ncu_summary.py gpurun_out/r02_ncu_config${c}_v3_raw.csv > gpurun_out/r02_ncu_config${c}_v3_summary.csv
done
rm -f gpurun_out/*.ncu-rep
