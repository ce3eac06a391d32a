"""A/B probe: the device leaf generator from two libgoom.so builds, bit for bit (a 4,096-leaf
d = 512 chain), and each build's time per 32,768-leaf window."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_03426_b200 import _lib  # noqa: E402

res = {}
for path in sys.argv[1:3]:
    lib = ctypes.CDLL(path)
    fn = lib.goom_random_normal_ts
    fn.restype = ctypes.c_int
    fn.argtypes = _lib.SIGNATURES["goom_random_normal_ts"][1]
    T, d = 4096, 512
    U = torch.empty(T * d * d, dtype=torch.float32, device="cuda")
    q = torch.empty(T * d * (d // 256), dtype=torch.float32, device="cuda")
    G = torch.empty(T * (d // 256), dtype=torch.int32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert fn(U.data_ptr(), q.data_ptr(), G.data_ptr(), T, d, 3, 777, st) == 0
    torch.cuda.synchronize()
    res[path] = U.clone()
    W = 32768
    U2 = torch.empty(W * d * d, dtype=torch.float32, device="cuda")
    q2 = torch.empty(W * d * 2, dtype=torch.float32, device="cuda")
    G2 = torch.empty(W * 2, dtype=torch.int32, device="cuda")
    for _ in range(2):
        fn(U2.data_ptr(), q2.data_ptr(), G2.data_ptr(), W, d, 1, 0, st)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(5):
        fn(U2.data_ptr(), q2.data_ptr(), G2.data_ptr(), W, d, 1, i * W, st)
    e.record()
    torch.cuda.synchronize()
    print(f"{path.split('/')[-1]}: {s.elapsed_time(e) / 5:.2f} ms per window")
    del U2, q2, G2
a, b = res.values()
print("bitwise equal:", torch.equal(a, b))
