"""B200-native GOOM LMME prefix scan (arXiv 2510.03426 hot path).

Drop-in for the hot path of the reference package `gooms`: the same public
names (SPEC.md `goom-core` / `pscan`), backed by sm_100a CUDA kernels in
`libgoom.so` through `torch.ops.goom.*` custom ops. GOOMs are complex64
tensors: real part log|x|, imaginary part 0 or pi.
"""

from . import _lib, ops  # noqa: F401  (registers torch.ops.goom.*)
from .core import (  # noqa: F401
    BACKINGS,
    NEG_INF,
    SENTINEL,
    Goom,
    GoomMatrix,
    ZeroPolicy,
    _col_log_norms,
    _gadd_arrays,
    _lmme_arrays,
    _log_sign_arrays,
    floor_for,
    from_real,
    gadd,
    gmul,
    join,
    lmme,
    log_matmul_exp,
    log_unit_norm_columns,
    lse_reduce,
    split,
    to_real,
    to_real_scaled,
)
from .lyapunov import (JacobianChain, SpectrumResult, colinearity_policy,  # noqa: F401
                       colinearity_select, integrate_chain, lle_parallel, lle_sequential,
                       orthonormal_reset,
                       load_jacobian_chain, qr_factor, qr_factor_batched, save_jacobian_chain,
                       spectrum_parallel, spectrum_sequential)
from .scan import (  # noqa: F401
    ResetPolicy,
    ScanPair,
    SelectiveCombiner,
    _scan_affine_stack,
    _selective_chain_core,
    _Stack,
    builtin_policy,
    combine_affine,
    combine_selective,
    never_policy,
    norm_threshold_policy,
    scan_chain,
    scan_parallel,
    scan_selective,
    scan_sequential,
)

__version__ = "0.1.0"
