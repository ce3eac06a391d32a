import sys, torch
sys.path.insert(0, ".")
from paper_2510_03426_b200 import ops
dev = torch.device("cuda")
L = ops.ts_random_normal(4096, 512, 3, 777, dev)
torch.save(L.U.cpu(), sys.argv[1])
T = 32768
L = None
torch.cuda.synchronize()
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(5):
        L = ops.ts_random_normal(T, 512, 1, i * T, dev)
        del L
    e.record(); torch.cuda.synchronize()
    print(sys.argv[1], f"{s.elapsed_time(e) / 5:.2f} ms per window")
