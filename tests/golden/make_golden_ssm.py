"""Golden vectors for the SSM forward pass (ssm.py) from the REFERENCE
(run in the build container, where /root/reference exists):

    python tests/golden/make_golden_ssm.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402


def main():
    _import_reference()
    import gooms.ssm as ssm  # noqa: E402
    from gooms.util import make_rng  # noqa: E402

    def random_params(rng, d, spectral_radius=None):
        a = rng.standard_normal((d, d))
        if spectral_radius is not None:
            a *= spectral_radius / np.max(np.abs(np.linalg.eigvals(a)))
        return ssm.SsmParams(A=a, B=rng.standard_normal((d, d)),
                             C=rng.standard_normal((2 * d, d)), D=rng.standard_normal((2 * d, d)))

    out = {}
    for name, seed, d, T, rho in (("ssm_random_d4", 64, 4, 257, None),
                                  ("ssm_growing_d8", 65, 8, 512, 1.5),
                                  ("ssm_explode_d8", 67, 8, 1024, 2.0)):
        rng = make_rng(seed)
        p = random_params(rng, d, rho)
        x0 = rng.standard_normal(d) * (10.0 if name == "ssm_explode_d8" else 1.0)
        u = rng.standard_normal((T, d))
        par = ssm.ssm_forward_parallel(p, x0, u)
        seq = ssm.ssm_forward_sequential(p, x0, u)
        out[name] = dict(A=p.A, B=p.B, C=p.C, D=p.D, x0=x0, u=u, state_log=par.state_log,
                         state_sign=par.state_sign, scales=par.scales, y=par.y,
                         seq_state_log=seq.state_log, seq_y=seq.y)
    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
