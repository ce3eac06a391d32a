"""Kernel timing of lmme_ts per ring-depth configuration (GOOM_TS_STAGES, one process each):
kind 1 (phase-1 shape: batch 128, distinct operands) and kind 2 (phase-3 shape: batch 8192,
carry per 64)."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")


def arm():
    from paper_2510_03426_b200 import ops
    d = 512
    dev = torch.device("cuda")
    L = ops.ts_random_normal(8192, d, 1, 0, dev)
    C = ops.ts_random_normal(128, d, 2, 0, dev)

    def ev(fn, reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    t1 = ev(lambda: ops.lmme_ts(L[0:128], C, 1), 20)
    t2 = ev(lambda: ops.lmme_ts(L, C, 2, b_div=64), 3)
    print(f"stages={os.environ.get('GOOM_TS_STAGES','0')} dbg={os.environ.get('GOOM_TS_DEBUG','0')}: "
          f"kind1 b128 {t1*1e3:.0f} us ({2*d**3*128/t1/1e9:.0f} TF/s) | kind2 b8192 {t2:.2f} ms "
          f"({2*d**3*8192/t2/1e9:.0f} TF/s)", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        arm()
        sys.exit(0)
    for dbg in os.environ.get("DBGS", "0").split():
        for st in os.environ.get("STAGES", "0 1 2 3").split():
            r = subprocess.run(["timeout", "120", sys.executable, __file__, "arm"],
                               env={**os.environ, "GOOM_TS_STAGES": st, "GOOM_TS_DEBUG": dbg},
                               capture_output=True, text=True)
            print(r.stdout.strip(), r.stderr[-300:] if r.returncode else "", flush=True)
