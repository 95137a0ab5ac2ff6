"""Diagnostic: streamed TNSR write/read throughput between HBM and a file."""
import os, sys, tempfile, time
import torch
sys.path.insert(0, ".")
from paper_2108_10448_b200.tensor import DeviceTensor
from paper_2108_10448_b200.tensorfile import read_tensor_device, write_tensor_device

shape = tuple(int(v) for v in (sys.argv[1:] or ["400", "400", "400"]))
n = 1
for d in shape:
    n *= d
x = DeviceTensor(torch.randn(n, dtype=torch.float64, device="cuda"), shape)
d = tempfile.mkdtemp(dir=os.environ.get("TNSR_DIR", "/tmp"))
p = os.path.join(d, "x.tnsr")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); write_tensor_device(p, x); t1 = time.perf_counter()
    y = read_tensor_device(p); torch.cuda.synchronize(); t2 = time.perf_counter()
    y32 = read_tensor_device(p, dtype=torch.float32, slab=(0, shape[0] // 2)); torch.cuda.synchronize(); t3 = time.perf_counter()
    gb = n * 8 / 1e9
    print(f"shape {shape}: write {gb / (t1 - t0):.2f} GB/s, read f64 {gb / (t2 - t1):.2f} GB/s, "
          f"read f32 half-slab {gb / (t3 - t2):.2f} GB/s (file {gb:.2f} GB), equal={torch.equal(x.flat, y.flat)}")
os.remove(p)
