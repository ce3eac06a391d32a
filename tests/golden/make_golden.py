"""Generate golden vectors for the GOOM LMME prefix-scan path from the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package (`/root/reference/pkg/src/gooms`)
and the reference's own scan-test helpers (`pkg/tests/test_scan.py`:
`rotation_leaves`, `norm_threshold_policy`), runs the reference functions on
seeded inputs, and writes small `.npz` fixtures next to this script. The GPU
box has no reference checkout; the tests there read only these fixtures and
the numpy oracle (`oracle/gooms_port.py`), which `tests/test_oracle_golden.py`
pins against the same fixtures.
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    import gooms.core as core  # noqa: E402
    import gooms.lyapunov as lyap  # noqa: E402
    import gooms.scan as scan  # noqa: E402
    import gooms.systems as systems  # noqa: E402
    import gooms.util as util  # noqa: E402
    import test_scan as ts  # noqa: E402

    return core, scan, lyap, systems, util, ts


def stack_arrays(pairs):
    al = np.stack([p.A.log_mag for p in pairs])
    as_ = np.stack([p.A.sign for p in pairs])
    bl = np.stack([p.B.log_mag for p in pairs])
    bs = np.stack([p.B.sign for p in pairs])
    fl = np.array([p.reset_applied for p in pairs], dtype=bool)
    return al, as_, bl, bs, fl


def state_arrays(pairs):
    return (np.stack([p.state.log_mag for p in pairs]),
            np.stack([p.state.sign for p in pairs]),
            np.array([p.reset_applied for p in pairs], dtype=bool))


def lorenz96(core_systems, d, F=8.0, dt=0.01):
    """Lorenz-96 built with the reference's own RK4 machinery (systems._flow_system)."""

    def f(x):
        return (np.roll(x, -1) - np.roll(x, 2)) * np.roll(x, 1) - x + F

    def df(x):
        J = -np.eye(d)
        for i in range(d):
            J[i, (i + 1) % d] += x[(i - 1) % d]
            J[i, (i - 2) % d] -= x[(i - 1) % d]
            J[i, (i - 1) % d] += x[(i + 1) % d] - x[(i - 2) % d]
        return J

    x0 = np.full(d, F)
    x0[0] += 0.01
    return core_systems._flow_system("lorenz96", d, dt, f, df, x0)


def main():
    core, scan, lyap, systems, util, ts = _import_reference()
    rng = util.make_rng
    out = {}

    # ---- LMME known-answer tests (pkg/tests/test_core.py:174-249) ----------
    a = core.GoomMatrix.from_real([[1.0, 2.0], [3.0, 4.0]])
    b = core.GoomMatrix.from_real([[5.0, 6.0], [7.0, 8.0]])
    r = core.lmme(a, b)
    out["lmme_2x2"] = dict(alog=a.log_mag, asign=a.sign, blog=b.log_mag, bsign=b.sign,
                           olog=r.log_mag, osign=r.sign)
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        g = rng(8)
        A = g.standard_normal((64, 64)).astype(dt)
        B = g.standard_normal((64, 64)).astype(dt)
        ga = core.GoomMatrix.from_real(A, dtype=dt)
        gb = core.GoomMatrix.from_real(B, dtype=dt)
        r = core.lmme(ga, gb)
        out[f"lmme_64_{tag}"] = dict(alog=ga.log_mag, asign=ga.sign, blog=gb.log_mag,
                                     bsign=gb.sign, olog=r.log_mag, osign=r.sign)
    # batched, rectangular, with zeros, huge and tiny magnitudes (float32 backing)
    g = rng(101)
    alog = g.uniform(-30, 30, (16, 5, 7)).astype(np.float32)
    blog = g.uniform(-30, 30, (16, 7, 3)).astype(np.float32)
    alog[0, 1, :] = -np.inf  # all-zero row
    alog[1, :, 2] = -np.inf
    blog[2, :, 0] = -np.inf  # all-zero column
    alog[3] += 1e6           # huge magnitudes
    blog[4] -= 200.0         # clamp regime: tiny column, scale stays 0
    asign = g.choice([-1.0, 1.0], alog.shape).astype(np.float32)
    bsign = g.choice([-1.0, 1.0], blog.shape).astype(np.float32)
    asign[alog == -np.inf] = 1.0
    bsign[blog == -np.inf] = 1.0
    ol, os_ = core._lmme_arrays(alog, asign, blog, bsign)
    out["lmme_batched_f32"] = dict(alog=alog, asign=asign, blog=blog, bsign=bsign, olog=ol, osign=os_)
    # row scaling invariance input (test_core.py:205-218)
    g = rng(9)
    A = g.standard_normal((5, 5))
    B = g.standard_normal((5, 5))
    S = A.copy()
    S[2] *= 3.7e50
    r0 = core.lmme(core.GoomMatrix.from_real(A), core.GoomMatrix.from_real(B))
    r1 = core.lmme(core.GoomMatrix.from_real(S), core.GoomMatrix.from_real(B))
    out["lmme_rowscale"] = dict(a=A, s=S, b=B, olog0=r0.log_mag, osign0=r0.sign,
                                olog1=r1.log_mag, osign1=r1.sign)

    # ---- gadd (test_core.py:327-348) -----------------------------------------
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        g = rng(22)
        n = 4096
        la = g.uniform(-100, 100, n).astype(dt)
        lb = g.uniform(-100, 100, n).astype(dt)
        sa = g.choice([-1.0, 1.0], n).astype(dt)
        sb = g.choice([-1.0, 1.0], n).astype(dt)
        lb[:256] = la[:256]
        sb[:256] = -sa[:256]          # exact cancellation
        la[256:300] = -np.inf
        sa[256:300] = 1.0
        lb[280:320] = -np.inf         # both -inf on 280..299
        sb[280:320] = 1.0
        ol, os_ = core._gadd_arrays(la, sa, lb, sb)
        out[f"gadd_{tag}"] = dict(alog=la, asign=sa, blog=lb, bsign=sb, olog=ol, osign=os_)

    # ---- conversions ----------------------------------------------------------
    g = rng(20)
    xs = g.standard_normal(4096) * np.exp(g.uniform(-200, 200, 4096))
    xs[:7] = 0.0
    ml, ms = core._log_sign_arrays(xs)
    out["from_real_f64"] = dict(x=xs, olog=ml, osign=ms)
    xs32 = (g.standard_normal(4096) * np.exp(g.uniform(-40, 40, 4096))).astype(np.float32)
    xs32[:5] = 0.0
    ml, ms = core._log_sign_arrays(xs32)
    out["from_real_f32"] = dict(x=xs32, olog=ml, osign=ms)
    logs = g.uniform(-1e4, 1e4, (6, 5, 4))
    signs = g.choice([-1.0, 1.0], logs.shape)
    scaled = [core.to_real_scaled(core.GoomMatrix(logs[i], signs[i])) for i in range(6)]
    out["to_real_scaled"] = dict(log=logs, sign=signs,
                                 out=np.stack([s[0] for s in scaled]),
                                 c=np.array([s[1] for s in scaled]))
    logs = g.uniform(-500, 500, (6, 6))
    out["col_log_norms"] = dict(log=logs, out=core._col_log_norms(logs))

    # ---- affine scans (pkg/tests/test_scan.py:217-337) -------------------------
    g = rng(39)
    leaves = ts.random_leaves(g, 64, 4)
    al, as_, bl, bs, fl = stack_arrays(leaves)
    seq = scan.scan_sequential(leaves, scan.combine_affine)
    par = scan.scan_parallel(leaves, scan.combine_affine, block_size=8)
    out["affine_T64_d4"] = dict(alog=al, asign=as_, blog=bl, bsign=bs, flags=fl,
                                seq=np.array(stack_arrays(seq)[:4]),
                                par8=np.array(stack_arrays(par)[:4]))
    # config 1: d=8, T=1000 chain of N(0,1) leaves, zero biases; f64 and f32 references
    g = rng(1)
    mats = g.standard_normal((1000, 8, 8))
    cfg1 = {}
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        lv = [ts.pair_from_real(m, dtype=dt) for m in mats]
        seq = scan.scan_sequential(lv, scan.combine_affine)
        par = scan.scan_parallel(lv, scan.combine_affine, block_size=32)
        cfg1[f"seq_{tag}"] = np.array(stack_arrays(seq)[:2])
        cfg1[f"par32_{tag}"] = np.array(stack_arrays(par)[:2])
    cfg1["mats"] = mats
    out["config1_chain"] = cfg1

    # ---- selective scans ------------------------------------------------------
    g = rng(43)
    leaves = ts.rotation_leaves(g, 300, 4)
    policy = ts.norm_threshold_policy(12.0)
    s_states, s_sites = scan.scan_selective(leaves, policy)
    p_states, p_sites = scan.scan_selective(leaves, policy, block_size=7)
    assert s_sites == p_sites
    al, as_, bl, bs, fl = stack_arrays(leaves)
    out["sel_norm_T300_d4"] = dict(alog=al, asign=as_, sites=np.array(s_sites),
                                   seq_state=np.array(state_arrays(s_states)[:2]),
                                   seq_flags=state_arrays(s_states)[2],
                                   par_state=np.array(state_arrays(p_states)[:2]))
    g = rng(45)
    leaves = ts.rotation_leaves(g, 64, 3)
    policy = ts.norm_threshold_policy(5.0, interval=8)
    s_states, s_sites = scan.scan_selective(leaves, policy)
    al, as_, bl, bs, fl = stack_arrays(leaves)
    out["sel_norm_interval8"] = dict(alog=al, asign=as_, sites=np.array(s_sites),
                                     seq_state=np.array(state_arrays(s_states)[:2]))
    g = rng(44)
    leaves = ts.rotation_leaves(g, 120, 4, biases=True)
    policy = ts.norm_threshold_policy(12.0)
    s_states, s_sites = scan.scan_selective(leaves, policy)
    al, as_, bl, bs, fl = stack_arrays(leaves)
    out["sel_norm_bias"] = dict(alog=al, asign=as_, blog=bl, bsign=bs, sites=np.array(s_sites),
                                seq_state=np.array(state_arrays(s_states)[:2]),
                                seq_flags=state_arrays(s_states)[2])
    # lyapunov colinearity policy on a Lorenz chain (spectrum_parallel stage (a))
    ch = lyap.integrate_chain(systems.lorenz(), burn_in=1000, T=3000, seed=2)
    d = ch.dim
    alog = np.empty((ch.T, d, d))
    asign = np.empty((ch.T, d, d))
    alog[0], asign[0] = core._log_sign_arrays(np.eye(d))
    alog[1:], asign[1:] = core._log_sign_arrays(ch.mats[: ch.T - 1])
    pol = lyap.colinearity_policy(0.99, 12)
    V, Vs, sites = scan._selective_chain_core(alog, asign, pol, 256)
    out["sel_colin_lorenz"] = dict(mats=ch.mats, alog=alog, asign=asign, Vlog=V, Vsign=Vs,
                                   sites=np.array(sites))
    pol1 = lyap.colinearity_policy(0.99, 1)
    V1, Vs1, sites1 = scan._selective_chain_core(alog[:600], asign[:600], pol1, 64)
    out["sel_colin_lorenz_walk"] = dict(Vlog=V1, Vsign=Vs1, sites=np.array(sites1))
    # Lorenz-96 Jacobians (config 4 system) built with the reference's RK4 machinery
    sys96 = lorenz96(systems, 16)
    ch96 = lyap.integrate_chain(sys96, burn_in=200, T=40, seed=0)
    out["lorenz96_d16"] = dict(mats=ch96.mats)

    # colinearity predicate / reset KATs (pkg/tests/test_lyapunov.py:164-215)
    g = rng(56)
    q, _ = lyap.qr_factor(g.standard_normal((4, 4)))
    qm = core.GoomMatrix.from_real(q)
    rq = lyap.orthonormal_reset(qm)
    logs = np.array([[1e6, 1e6 - 1.0], [1e6 - 2.0, 1e6 - 0.5]])
    rh = lyap.orthonormal_reset(core.GoomMatrix(logs, np.ones((2, 2))))
    out["orthonormal_reset"] = dict(qlog=qm.log_mag, qsign=qm.sign, rlog=rq.log_mag,
                                    rsign=rq.sign, hlog=logs, hrlog=rh.log_mag, hrsign=rh.sign)

    # Appendix C worked example (pkg/tests/test_scan.py:142-178)
    g = rng(35)
    x0 = g.standard_normal((3, 3))
    a1, a2, a3 = (g.standard_normal((3, 3)) for _ in range(3))
    out["appendix_c"] = dict(x0=x0, a1=a1, a2=a2, a3=a3,
                             want1=a1 @ x0,
                             want2=(a1 @ x0) / (1.0 + np.linalg.norm(a1 @ x0)),
                             want3=a3 @ ((a1 @ x0) / (1.0 + np.linalg.norm(a1 @ x0))))

    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print("wrote", len(out), "fixtures to", HERE)


if __name__ == "__main__":
    main()
