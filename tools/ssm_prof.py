import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2510_03426_b200 import ssm
rng = np.random.default_rng(5)
d, S, T = 64, 32, 4096
a = rng.standard_normal((d, d)); a *= 1.2 / np.max(np.abs(np.linalg.eigvals(a)))
p = ssm.SsmParams(a, rng.standard_normal((d, d)), rng.standard_normal((2*d, d)), rng.standard_normal((2*d, d)))
x0 = rng.standard_normal((S, d)); u = rng.standard_normal((S, T, d))
ssm.ssm_forward_batched(p, x0[:2], u[:2, :256])
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    st = ssm._chunked_states(p, x0, u, 64); torch.cuda.synchronize(); t1 = time.perf_counter()
    out = ssm._finish(p, x0, u, st); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"states {t1-t0:.3f} s  finish {t2-t1:.3f} s")
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    st = ssm._chunked_states(p, x0, u, 64); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
