"""Golden vectors for the Lyapunov stages (b)-(d) and the LLE
from the REFERENCE (run in the build container, where /root/reference exists):

    python tests/golden/make_golden_lyap.py

Imports the unmodified reference (`gooms.lyapunov`, `gooms.systems`) and writes small
.npz fixtures next to this script; the GPU tests read only the fixtures.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference, lorenz96  # noqa: E402


def main():
    core, scan, lyap, systems, util, ts = _import_reference()
    out = {}
    # batched Householder QR (lyapunov.py:79-99) incl. a rank-deficient and a zero matrix
    g = np.random.default_rng(71)
    ms = g.standard_normal((6, 5, 5))
    ms[3, :, 2] = ms[3, :, 1]
    ms[4] = 0.0
    q, r = lyap.qr_factor_batched(ms)
    out["qr_batched"] = dict(ms=ms, q=q, r=r)
    # spectrum_parallel / spectrum_sequential on the reference's own Lorenz system
    ch = lyap.integrate_chain(systems.lorenz(), burn_in=1000, T=3000, seed=2)
    par = lyap.spectrum_parallel(ch, check_interval=8)
    seq = lyap.spectrum_sequential(ch)
    out["spectrum_lorenz"] = dict(mats=ch.mats, dt=np.array(ch.dt), lambdas=par.lambdas,
                                  resets=np.array(par.resets), seq=seq.lambdas)
    # Lorenz-96 d = 16 (config 4's system at a CPU-sized d), default policy
    ch96 = lyap.integrate_chain(lorenz96(systems, 16), burn_in=500, T=1200, seed=0)
    par = lyap.spectrum_parallel(ch96)
    seq = lyap.spectrum_sequential(ch96)
    out["spectrum_l96_d16"] = dict(mats=ch96.mats, dt=np.array(ch96.dt), lambdas=par.lambdas,
                                   resets=np.array(par.resets), seq=seq.lambdas)
    # LLE: random chains (pkg/tests/test_lyapunov.py:264-273)
    g = util.make_rng(58)
    mats, u0s, lp, ls = [], [], [], []
    for _ in range(5):
        m = g.standard_normal((100, 3, 3))
        u0 = g.standard_normal(3)
        u0 /= np.linalg.norm(u0)
        c = lyap.JacobianChain(dt=0.5, mats=m)
        mats.append(m)
        u0s.append(u0)
        lp.append(lyap.lle_parallel(c, u0))
        ls.append(lyap.lle_sequential(c, u0))
    out["lle_random"] = dict(mats=np.array(mats), u0=np.array(u0s), par=np.array(lp),
                             seq=np.array(ls))
    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
