"""Profiling driver: one batched complex64 LMME of `batch` d x d N(0,1) products (config 2's
shape), repeated `reps` times (for ncu / nsys-free CUDA-event timing)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 256
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g._lib.load()
import os
if os.environ.get("PERSIST_L2_MB"):  # probe: L2 set-aside for evict_last lines
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    torch.cuda.init()
    if rt is not None:
        print("set limit rc", rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(int(os.environ["PERSIST_L2_MB"]) << 20)))
A = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
B = torch.ops.goom.from_real(torch.randn(batch, d, d, device="cuda"), float("-inf"), False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(reps):
    flush.add_(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch.ops.goom.lmme(A, B)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ts.sort()
gbs = 24 * d * d * batch / (ts[len(ts) // 2] * 1e-3) / 1e9
print(f"d={d} batch={batch} median {ts[len(ts) // 2]:.4f} ms min {ts[0]:.4f} ms ({gbs:.0f} GB/s)")
