import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2510_03426_b200 as g
from oracle import gooms_port as G
from goom_testlib import chain_parity, to_np, TC_CHAIN_FLOOR
g._lib.load()
for T in (257, 320, 1087):
    d = 8
    rng = np.random.default_rng(T)
    x = rng.standard_normal((T + 1, d, d))
    al, as_ = G.log_sign(x)
    for carry_mode in ("carry", "nocarry"):
        if carry_mode == "carry":
            out = torch.ops.goom.scan_chain_long(g.join(al[1:], as_[1:]), g.join(al[0], as_[0]))
            gl, gs = to_np(out)
            gl = np.concatenate([al[:1], gl]); gs = np.concatenate([as_[:1], gs])
            A_l, A_s = al, as_
        else:
            out = torch.ops.goom.scan_chain_long(g.join(al, as_), None)
            gl, gs = to_np(out); A_l, A_s = al, as_
        want = G.chain_blocked(A_l, A_s, T + 1)
        l32, s32 = G.log_sign(x.astype(np.float32))
        ref = G.chain_blocked(l32, s32, T + 1)
        seq = torch.ops.goom.scan_chain(g.join(A_l, A_s), T + 1, None)
        sl, ss = to_np(seq)
        r = chain_parity(gl, gs, A_l, A_s, want, [ref], floor=TC_CHAIN_FLOOR)
        r2 = chain_parity(sl, ss, A_l, A_s, want, [ref], floor=TC_CHAIN_FLOOR)
        print(T, carry_mode, "long ok", r["ok"], "bad", r["bad"][:4], "e_gpu", np.round(r["e_gpu"][r["bad"][:4]], 6), "e_ref", np.round(r["e_ref"][r["bad"][:4]], 6), "scaled_bad", r["scaled_bad"][:3], "scaled_max", r["scaled_max"], "| seq-fold ok", r2["ok"], r2["bad"][:4], r2["scaled_max"])
