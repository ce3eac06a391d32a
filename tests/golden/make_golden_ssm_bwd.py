"""Golden gradients for the SSM backward pass (SURVEY §8d config 5 "forward+backward").

The reference has no autodiff, so the gradients come from torch float64 autograd of the
reference's forward (ssm.py:84-98, 99-108) written in real arithmetic, on chains short
enough that no state leaves float64 range; the forward's log-domain states come from the
REFERENCE itself (run in the build container, where /root/reference exists), and the
autograd forward is checked against them before anything is written:

    python tests/golden/make_golden_ssm_bwd.py
"""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _import_reference  # noqa: E402


def autograd_ssm(A, B, C, D, x0, u, gy):
    """sum(gy * y) differentiated by torch: x_t = A x_{t-1} + B u_t, c_t = max log|x_t|
    (torch.max: gradient to the first argmax), y_t = C x_t e^{2 - c_t} + D u_t."""
    t = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
         for k, v in dict(A=A, B=B, C=C, D=D, x0=x0, u=u).items()}
    x = t["x0"]
    ys = []
    logs = []
    for i in range(u.shape[0]):
        x = t["A"] @ x + t["B"] @ t["u"][i]
        lx = torch.log(torch.abs(x))
        c = torch.max(lx, dim=0).values
        ys.append(t["C"] @ (x * torch.exp(2.0 - c)) + t["D"] @ t["u"][i])
        logs.append(lx.detach())
    y = torch.stack(ys)
    (y * torch.tensor(gy)).sum().backward()
    return y.detach().numpy(), torch.stack(logs).numpy(), {k: v.grad.numpy() for k, v in t.items()}


def main():
    _import_reference()
    import gooms.ssm as ssm  # noqa: E402
    from gooms.util import make_rng  # noqa: E402

    out = {}
    for name, seed, d, T, rho in (("ssm_bwd_d4", 71, 4, 64, 1.2),
                                  ("ssm_bwd_d8", 72, 8, 200, 0.95),
                                  ("ssm_bwd_growing_d8", 73, 8, 300, 1.5)):
        rng = make_rng(seed)
        a = rng.standard_normal((d, d))
        a *= rho / np.max(np.abs(np.linalg.eigvals(a)))
        p = ssm.SsmParams(A=a, B=rng.standard_normal((d, d)), C=rng.standard_normal((2 * d, d)),
                          D=rng.standard_normal((2 * d, d)))
        x0 = rng.standard_normal(d)
        u = rng.standard_normal((T, d))
        gy = rng.standard_normal((T, 2 * d))
        run = ssm.ssm_forward_parallel(p, x0, u)
        y, logs, g = autograd_ssm(p.A, p.B, p.C, p.D, x0, u, gy)
        assert np.max(np.abs(logs - run.state_log)) < 1e-9 * max(1.0, np.abs(logs).max()), name
        assert np.allclose(y, run.y, rtol=1e-9, atol=1e-9), name
        out[name] = dict(A=p.A, B=p.B, C=p.C, D=p.D, x0=x0, u=u, gy=gy,
                         state_log=run.state_log, state_sign=run.state_sign, scales=run.scales,
                         y=run.y, **{"d" + k: v for k, v in g.items()})
    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
        print("wrote", name, {k: v.shape for k, v in arrays.items()})


if __name__ == "__main__":
    main()
