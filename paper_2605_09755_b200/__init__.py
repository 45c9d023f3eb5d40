"""B200-native sketched power method (arXiv 2605.09755), drop-in for the
reference ``skpower`` hot path.

Public surface mirrors /root/reference/pkg/src/skpower/__init__.py:25-86 for
the accelerated path (sketching, power methods, dense linalg).  Every
arithmetic step runs in hand-written sm_100a kernels in ``libskp.so``
(include/skp.h) behind a ctypes binding; there is no CPU fallback.  Row-
sharded multi-GPU drivers live in ``paper_2605_09755_b200.distributed``.
"""
from ._convert import DeviceMatrix, device_matrix
from .linalg import (
    SvdResult,
    as_matrix,
    frobenius_norm,
    matmul,
    norms,
    orthonormalize,
    pinv,
    spectral_norm,
    thin_svd,
)
from .power import (
    FactorizationResult,
    NystromResult,
    RangeFinderSpec,
    choose_q,
    lowrank_factorize,
    nystrom_psd,
    power_iterate,
    randsvd,
    range_finder_classical,
    range_finder_sketched,
    rsvd,
)
from .sketching import (
    SKETCH_KINDS,
    SketchOperator,
    apply_left_transpose,
    apply_right,
    densify,
    make_sketch,
    substream,
)

__version__ = "0.2.0"


def library_path() -> str:
    from ._lib import LIB_PATH
    return LIB_PATH
