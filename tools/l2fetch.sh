# Diagnostic: k_gather time / DRAM traffic vs the L2 fetch granularity limit.
for g in 32 64 128; do
  RTCUR_L2_FETCH=$g python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/l2_$g.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/l2_$g.json')); print($g, round(d['value'],1), {k: round(v['ms_per_step'],3) for k,v in d['phases'].items()})"
done
python -c "import torch; import ctypes; v=ctypes.c_size_t(); l=ctypes.CDLL('libcudart.so.12') if False else None; print('default', torch.cuda.is_available())"
RTCUR_L2_FETCH=32 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_gather -s 60 -c 2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__bytes|duration|lts__t" 
