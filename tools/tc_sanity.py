"""Quick tcgen05 LMME sanity check vs the SIMT kernel (run under `timeout`)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402

torch.manual_seed(0)
for (n, k, m, batch) in ((128, 32, 128, 1), (128, 128, 128, 2), (256, 512, 256, 3), (512, 512, 512, 8)):
    A = torch.complex(torch.randn(batch, n, k, device="cuda"), torch.zeros(batch, n, k, device="cuda"))
    B = torch.complex(torch.randn(batch, k, m, device="cuda"), torch.zeros(batch, k, m, device="cuda"))
    A.imag[A.real < 0] = 3.14159265
    A.real.abs_().log_()
    B.imag[B.real < 0] = 3.14159265
    B.real.abs_().log_()
    g._lib.set_backend(1)
    ref = torch.ops.goom.lmme(A, B)
    g._lib.set_backend(2)
    out = torch.ops.goom.lmme(A, B)
    torch.cuda.synchronize()
    d = (out.real - ref.real).abs()
    sign_diff = ((out.imag != 0) != (ref.imag != 0)).sum().item()
    print(f"n={n} k={k} m={m} batch={batch}: max|dlog|={d.max().item():.3e} median={d.median().item():.3e} "
          f"sign_diffs={sign_diff} nan={torch.isnan(out.real).sum().item()}", flush=True)
