"""Shared helpers for the test suite (fixture loading, tolerances)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


NEG_INF = float("-inf")


def to_np(z):
    """complex64 torch tensor -> (log float64, sign float64) numpy."""
    zc = z.detach().cpu()
    log = zc.real.double().numpy()
    sign = np.where(np.cos(zc.imag.double().numpy()) < 0, -1.0, 1.0)
    return log, sign


def rel_log_diff_per(x, y, axis_keep=0):
    """_rel_log_diff (pkg/tests/test_scan.py:209-213) reduced over all but axis 0."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    denom = np.maximum(1.0, np.abs(y))
    both = (x == NEG_INF) & (y == NEG_INF)
    with np.errstate(invalid="ignore"):
        diff = np.where(both, 0.0, np.abs(x - y) / denom)
    diff = np.where(np.isnan(diff), np.inf, diff)
    return diff.reshape(diff.shape[0], -1).max(axis=1)


def lmme_parity(got, alog, asign, blog, bsign, tol=1e-4, kappa_min=1e-2, sign_kappa=1e-4):
    """Per-LMME parity criterion of SURVEY §8c: rel-log error <= tol where the
    cancellation ratio kappa >= kappa_min; signs exact where kappa >= sign_kappa.
    The oracle runs in float64 on the same (float32-representable) inputs."""
    from oracle import gooms_port as G

    gl, gs = got
    wl, ws = G.lmme(alog.astype(np.float64), asign.astype(np.float64),
                    blog.astype(np.float64), bsign.astype(np.float64))
    kappa = G.cancellation(alog.astype(np.float64), asign.astype(np.float64),
                           blog.astype(np.float64), bsign.astype(np.float64))
    mask = kappa >= kappa_min
    denom = np.maximum(1.0, np.abs(wl))
    both = (gl == NEG_INF) & (wl == NEG_INF)
    with np.errstate(invalid="ignore"):
        diff = np.where(both, 0.0, np.abs(gl - wl) / denom)
    diff = np.where(np.isnan(diff), np.inf, diff)
    err = float(np.max(np.where(mask, diff, 0.0))) if diff.size else 0.0
    smask = kappa >= sign_kappa
    flips = int(np.sum((gs != ws) & smask))
    return err, flips
