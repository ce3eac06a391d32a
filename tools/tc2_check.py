"""tcgen05 pair kernel (lmme_tc2) vs the one-SM kernel and the SIMT kernel: numerics +
timing (run under `timeout`; GOOM_TC2 is read once per process, so each arm is a subprocess)."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")


def arm():
    import paper_2510_03426_b200 as g  # noqa: F401
    torch.manual_seed(0)
    res = {}
    for (n, k, m, batch) in ((256, 16, 256, 1), (256, 512, 256, 3), (512, 512, 512, 8), (1024, 1024, 1024, 2),
                             (512, 512, 512, 1024), (1024, 1024, 1024, 256)):
        A = torch.complex(torch.randn(batch, n, k, device="cuda"), torch.zeros(batch, n, k, device="cuda"))
        B = torch.complex(torch.randn(batch, k, m, device="cuda"), torch.zeros(batch, k, m, device="cuda"))
        for X in (A, B):
            X.imag[X.real < 0] = 3.14159265
            X.real.abs_().log_()
        out = torch.ops.goom.lmme(A, B)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5 if batch > 8 else 1
        s.record()
        for _ in range(reps):
            torch.ops.goom.lmme(A, B)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        torch.save(out[:2].cpu(), f"gpurun_out/tc2_{os.environ.get('ARM')}_{n}_{batch}.pt")
        print(f"ARM {os.environ.get('ARM')} n={n} k={k} m={m} batch={batch}: {ms:.3f} ms "
              f"{2*n*k*m*batch/ms/1e9:.1f} TF/s nan={torch.isnan(out.real).sum().item()}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        arm()
        sys.exit(0)
    for name, env in (("tc2", {"GOOM_TC2": "1"}), ("tc1", {"GOOM_TC2": "0"})):
        r = subprocess.run(["timeout", "120", sys.executable, __file__, "arm"],
                           env={**os.environ, **env, "ARM": name}, capture_output=True, text=True)
        print(r.stdout, r.stderr[-2000:], "rc", r.returncode, flush=True)
    import glob
    for f in sorted(glob.glob("gpurun_out/tc2_tc2_*.pt")):
        a = torch.load(f)
        b = torch.load(f.replace("tc2_tc2_", "tc2_tc1_"))
        d = (a.real - b.real).abs()
        fin = torch.isfinite(d)
        sd = ((a.imag != 0) != (b.imag != 0)).sum().item()
        print(f"{f}: max|dlog| {d[fin].max().item():.3e} median {d[fin].median().item():.3e} "
              f"nonfinite {(~fin).sum().item()} sign_diffs {sd}")
