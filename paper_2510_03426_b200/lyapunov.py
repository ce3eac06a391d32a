"""Selective-reset policy of the Lyapunov estimator — drop-in for the policy part
of `gooms.lyapunov` (lyapunov.py:137-278).

`colinearity_policy` returns a built-in device policy: the predicate
(max off-diagonal |cos| of the log-unit-normalised columns > threshold, or
log|det| < log(volume_floor), or an all-zero column) and the CGS2 orthonormal
reset run inside the scan on the GPU in FP64. The spectrum estimator stages
(b)-(d) are the next row of SURVEY §8f and are not part of this package yet.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .core import GoomMatrix
from .scan import ResetPolicy, builtin_policy


def colinearity_policy(threshold=0.99, check_interval=12, volume_floor=1e-9) -> ResetPolicy:
    """lyapunov.colinearity_policy (lyapunov.py:239-278): consume_leaf False."""
    if not (0.0 < threshold < 1.0):
        raise ValueError("threshold must be in (0, 1)")
    return builtin_policy(_lib.POLICY_COLINEARITY, threshold=float(threshold),
                          log_volume_floor=math.log(volume_floor),
                          check_interval=check_interval, consume_leaf=False)


def colinearity_select(m: GoomMatrix, threshold) -> bool:
    """True when a column pair has |cos| > threshold (lyapunov.py:146-155).

    Pure cosine test: the volume floor is disabled (log floor = -inf).
    """
    if not (0.0 < threshold < 1.0):
        raise ValueError("threshold must be in (0, 1)")
    fire = torch.ops.goom.policy_select(m.data, _lib.POLICY_COLINEARITY, float(threshold),
                                        float("-inf"))
    return bool(fire.item())


def orthonormal_reset(m: GoomMatrix) -> GoomMatrix:
    """CGS2 orthonormal basis of the column span (lyapunov.py:197-219)."""
    if m.rows != m.cols:
        raise ValueError("expected a square matrix")
    return GoomMatrix._wrap(torch.ops.goom.policy_reset(m.data, _lib.POLICY_COLINEARITY))
