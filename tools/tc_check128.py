"""Debug aid: tcgen05 d=128 LMME vs the SIMT path, per batch size (pattern of mismatches)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_03426_b200 as g  # noqa: E402
lib = g._lib.load()
for batch in (1, 6, 147, 148, 149, 300):
    torch.manual_seed(batch)
    A = torch.ops.goom.from_real(torch.randn(batch, 128, 128, device="cuda"), float("-inf"), False)
    B = torch.ops.goom.from_real(torch.randn(batch, 128, 128, device="cuda"), float("-inf"), False)
    tc = torch.ops.goom.lmme(A, B)
    lib.goom_set_lmme_backend(1)
    ref = torch.ops.goom.lmme(A, B)
    lib.goom_set_lmme_backend(0)
    torch.cuda.synchronize()
    err = (tc.real - ref.real).abs()
    bad = err > 1e-3
    print(batch, "max err", err.max().item(), "bad frac", bad.float().mean().item())
    if bad.any():
        idx = bad.nonzero()
        print("  products", idx[:, 0].unique()[:10].tolist(), "rows", idx[:, 1].unique()[:40].tolist(),
              "cols", idx[:, 2].unique()[:40].tolist())
        print("  sample tc", tc[idx[0, 0], idx[0, 1], idx[0, 2]].item(), "ref", ref[idx[0, 0], idx[0, 1], idx[0, 2]].item())
