"""Per-position chain errors (scaled-real and kappa-masked rel-log) of the GPU chain scan
vs the float64 oracle, next to the reference's own float32 runs. GOOM_CHAIN_TS selects the
engine (run twice: 1 and 0)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2510_03426_b200 as g  # noqa: E402
from goom_testlib import chain_parity, to_np  # noqa: E402
from oracle import gooms_port as G  # noqa: E402

for d, T, block in ((256, 64, 8), (256, 33, 64), (512, 24, 5)):
    rng = np.random.default_rng(d * T + block)
    mats = rng.standard_normal((T, d, d))
    al, as_ = G.log_sign(mats)
    out = g.scan_chain(g.join(al, as_), block_size=block)
    gl, gs = to_np(out)
    want = G.chain_blocked(al, as_, T)
    l32, s32 = G.log_sign(mats.astype(np.float32))
    refs = [G.chain_blocked(l32, s32, block), G.chain_blocked(l32, s32, T)]
    r = chain_parity(gl, gs, al, as_, want, refs)
    from goom_testlib import scaled_real_err
    sg = scaled_real_err(gl, gs, *want)
    sr = np.max([scaled_real_err(x[0], x[1], *want) for x in refs], axis=0)
    print(f"TS={os.environ.get('GOOM_CHAIN_TS','1')} d={d} T={T} block={block}: ok={r['ok']} "
          f"scaled gpu max {sg.max():.2e} ref32 max {sr.max():.2e}  worst ratio {np.max(sg/np.maximum(sr,1e-30)):.2f} "
          f"e_gpu max {r['e_gpu'].max():.2e} e_ref max {r['e_ref'].max():.2e} bad {r['scaled_bad']}", flush=True)
    print("   gpu scaled at", [f"{x:.1e}" for x in sg[::max(1, T // 8)]], flush=True)
    print("   ref scaled at", [f"{x:.1e}" for x in sr[::max(1, T // 8)]], flush=True)
