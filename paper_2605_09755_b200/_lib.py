"""ctypes binding of libskp.so (include/skp.h).

The product path has no CPU fallback: if the shared library is missing or CUDA
is unavailable, every entry point raises.  Status codes map to exceptions the
way the reference raises them: argument errors -> ValueError, CUDA errors ->
RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libskp.so")

SKP_OK, SKP_ERR_ARG, SKP_ERR_CUDA, SKP_ERR_UNSUPPORTED, SKP_ERR_NUMERIC = range(5)

_vp, _i64, _i32, _u64, _f32, _f64 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                     ctypes.c_uint64, ctypes.c_float, ctypes.c_double)
_int = ctypes.c_int

# name -> (restype, argtypes); mirrors include/skp.h one to one
SIGNATURES = {
    "skp_last_error": (ctypes.c_char_p, []),
    "skp_abi_version": (_int, []),
    "skp_has_tcgen05": (_int, []),
    "skp_launch_count": (_i64, []),
    "skp_countsketch_ws_bytes": (_i64, [_i64, _i64, _i32]),
    "skp_countsketch_gen": (_int, [_u64, _u64, _u64, _u64, _i64, _i64, _i32, _i64, _i64,
                                   _vp, _vp, _vp, _i64, _vp]),
    "skp_countsketch_csc_ws_bytes": (_i64, [_i64, _i32, _i64]),
    "skp_countsketch_csc": (_int, [_vp, _vp, _i64, _i32, _i64, _vp, _vp, _vp, _i64, _vp]),
    "skp_sketch_right_ws_bytes": (_i64, [_i64, _i32, _i64, _i32]),
    "skp_sketch_right_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _vp, _i64,
                                    _vp, _vp, _vp, _i64, _vp]),
    "skp_sketch_right_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _vp, _i64,
                                    _vp, _vp, _vp, _i64, _vp]),
    "skp_gaussian_ws_bytes": (_i64, [_i64]),
    "skp_gaussian_f32": (_int, [_u64, _u64, _u64, _u64, _i64, _i64, _f64, _vp, _i64, _vp, _vp,
                                _i64, _vp]),
    "skp_gaussian_f64": (_int, [_u64, _u64, _u64, _u64, _i64, _i64, _f64, _vp, _i64, _vp, _vp,
                                _i64, _vp]),
    "skp_sketch_gather_plan_bytes": (_i64, [_i64, _i64]),
    "skp_sketch_gather_plan_fail_offset": (_i64, [_i64]),
    "skp_sketch_gather_plan": (_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "skp_sketch_gather_f32": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, ctypes.c_float, _vp, _i64,
                                     _vp, _vp, _vp, _vp]),
    "skp_sketch_gather_variant": (_int, [_i64, _i64]),
    "skp_sketch_gather_f32_acc64": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _f64, _vp, _i64, _vp,
                                           _vp, _vp]),
    "skp_sketch_left_t_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _vp, _i64,
                                     _vp]),
    "skp_sketch_left_t_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i32, _i64, _vp, _i64,
                                     _vp]),
    "skp_gemm_ws_bytes": (_i64, [_int, _int, _i64, _i64, _i64, _i32, _i32]),
    "skp_gemm_f32": (_int, [_int, _int, _i64, _i64, _i64, _f32, _vp, _i64, _vp, _i64, _f32,
                            _vp, _i64, _i32, _vp, _i64, _vp]),
    "skp_gemm_f64": (_int, [_int, _int, _i64, _i64, _i64, _f64, _vp, _i64, _vp, _i64, _f64,
                            _vp, _i64, _i32, _vp, _i64, _vp]),
    "skp_cholesky_f64": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "skp_trinv_lower_f64": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "skp_cholinv_ws_bytes": (_i64, [_i64]),
    "skp_cholinv_f64": (_int, [_vp, _i64, _i64, _f64, _f64, _vp, _vp, _vp, _i64, _vp]),
    "skp_syevj_ws_bytes": (_i64, [_i64]),
    "skp_syevj_f64": (_int, [_vp, _i64, _vp, _vp, _i32, _vp, _i64, _vp, _vp]),
    "skp_cast_f32_f64": (_int, [_vp, _vp, _i64, _vp]),
    "skp_cast_f64_f32": (_int, [_vp, _vp, _i64, _vp]),
    "skp_split_h2_f32": (_int, [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _i64, _vp, _i32, _vp]),
    "skp_split_h2_inplace_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _i32, _vp]),
    "skp_gemm_h3_ws_bytes": (_i64, [_int, _i64, _i64, _i64]),
    "skp_gemm_h3": (_int, [_int, _i64, _i64, _i64, _f32, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                           _f32, _vp, _i64, _vp, _i64, _vp]),
    "skp_gemm_h3_emit_t": (_int, [_int, _i64, _i64, _i64, _f32, _vp, _vp, _i64, _vp, _vp, _vp, _i64,
                                  _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _i64,
                                  _vp]),
    "skp_gesvj_ws_bytes": (_i64, [_i64, _i64]),
    "skp_gesvj_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _i64, _vp,
                             _vp]),
    "skp_gesvj_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _i64, _vp,
                             _vp]),
    "skp_sym_check_f32": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "skp_sym_check_f64": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "skp_syrk_h3_ws_bytes": (_i64, [_i64, _i64]),
    "skp_syrk_h3": (_int, [_i32, _i64, _i64, _f32, _vp, _vp, _i64, _vp, _f32, _vp, _i64, _vp, _i64,
                           _vp]),
    "skp_gemm_h3s_ws_bytes": (_i64, [_i64, _i64, _i64]),
    "skp_gemm_h3s": (_int, [_i64, _i64, _i64, _f32, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _f32, _vp,
                            _i64, _vp, _vp, _i64, _vp]),
    "skp_h2_exponent_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _i32, _i32, _vp]),
    "skp_srht_apply_f32": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _f64, _vp,
                                  _i64, _i64, _vp]),
    "skp_srht_apply_f64": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _f64, _vp,
                                  _i64, _i64, _vp]),
    "skp_gram_f32_f64_ws_bytes": (_i64, [_i64, _i64]),
    "skp_gram_f32_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "skp_unpermute_cols_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "skp_unpermute_cols_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "skp_permute_rows_f32": (_int, [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _vp]),
    "skp_permute_rows_f64": (_int, [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _vp]),
    "skp_cast2d_f32_f64": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    "skp_cast2d_f64_f32": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    "skp_sumsq_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "skp_sumsq_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "skp_symmetrize_f32": (_int, [_vp, _i64, _i64, _vp]),
    "skp_symmetrize_f64": (_int, [_vp, _i64, _i64, _vp]),
    "skp_scale_cols_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "skp_scale_cols_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "skp_orth_dev_f64": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "skp_eig_orth_f64": (_int, [_vp, _vp, _i64, _f64, _vp, _vp, _vp]),
    "skp_sqrt_eigs_f64": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "skp_chol_pivot_check_f64": (_int, [_vp, _i64, _i64, _f64, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


class SkpLibraryError(RuntimeError):
    """libskp.so missing or unusable: there is no CPU fallback."""


def load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise SkpLibraryError(
                f"{LIB_PATH} not built; run `python -m paper_2605_09755_b200._build` "
                "(the sketched power method has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().skp_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == SKP_OK:
        return
    msg = last_error()
    if rc in (SKP_ERR_ARG, SKP_ERR_UNSUPPORTED):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
