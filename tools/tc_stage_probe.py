"""Kernel-only timing of the LMME tcgen05 kernels with pipeline stages disabled
(GOOM_TC_DEBUG; results invalid except for debug 0) — finds the bottleneck stage.
usage: python tools/tc_stage_probe.py  (spawns one subprocess per (arm, debug))"""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")


def arm(d, batch):
    import paper_2510_03426_b200 as g
    lib = g._lib
    A = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
    B = torch.complex(torch.randn(batch, d, d, device="cuda"), torch.zeros(batch, d, d, device="cuda"))
    for X in (A, B):
        X.imag[X.real < 0] = 3.14159265
        X.real.abs_().log_()
    C = torch.empty_like(A)
    ra = A.real.amax(dim=2).clamp_min(0).contiguous()
    cb = B.real.amax(dim=1).clamp_min(0).contiguous()
    strm = torch.cuda.current_stream().cuda_stream

    def call():
        lib.call("goom_lmme_scaled_c64", lib.goom_operand(A.data_ptr(), d * d, 1), ra.data_ptr(), d,
                 lib.goom_operand(B.data_ptr(), d * d, 1), cb.data_ptr(), d, C.data_ptr(), d * d,
                 batch, d, d, d, strm)
    call()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        call()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{os.environ.get('ARM')} dbg={os.environ.get('GOOM_TC_DEBUG', '0')} d={d} batch={batch}: "
          f"{ms:.3f} ms  {2*d**3*batch/ms/1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        arm(int(sys.argv[1]), int(sys.argv[2]))
        sys.exit(0)
    cases = [(512, 1024), (1024, 256)]
    for name, tc2 in (("tc2", "1"), ("tc1", "0")):
        for dbg in os.environ.get("DBGS", "0 1 2 3 5").split():
            for d, b in cases:
                r = subprocess.run(["timeout", "120", sys.executable, __file__, str(d), str(b)],
                                   env={**os.environ, "GOOM_TC2": tc2, "GOOM_TC_DEBUG": dbg, "ARM": name},
                                   capture_output=True, text=True)
                print(r.stdout.strip(), r.stderr[-500:] if r.returncode else "", flush=True)
