"""ctypes binding of the C ABI (include/lumisplit_b200.h).

The shared library is built in-tree (paper_1908_01961_b200/build.py).  There
is no fallback: if the library is missing or no CUDA device is present, the
solver entry points raise.  `symbols()` lists every exported entry point so
the CPU test suite can check the ABI without a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# LS_LIB_PATH selects another build of the same library (tools/ablate.py)
LIB_PATH = Path(os.environ.get("LS_LIB_PATH") or Path(__file__).resolve().parent / "liblumisplit_b200.so")

LS_OK, LS_ERR_NONFINITE, LS_ERR_ARG, LS_ERR_CUDA = 0, 1, 2, 3
NUM_TERMS = 8
MAX_K = 12
TERM_NAMES = ("data", "clustering", "r_sparsity", "r_consistency", "monochrome",
              "i_sparsity", "smoothness", "non_neg")


class Weights(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "lambda_data", "lambda_clustering", "lambda_r_sparsity", "p",
        "lambda_r_consistency", "lambda_monochrome", "lambda_i_sparsity",
        "lambda_smoothness", "lambda_non_neg", "lambda_ir", "lambda_cr",
        "eps_nonneg", "eps_irls")] + [("chroma_reg", C.c_int)]


class SolveCfg(C.Structure):
    _fields_ = [("pcg_iterations", C.c_int), ("max_halvings", C.c_int),
                ("svd_truncation", C.c_double), ("max_delta_b", C.c_double)]


class GNRecord(C.Structure):
    _fields_ = [("energy_before", C.c_double), ("energy_after", C.c_double),
                ("alpha", C.c_double), ("accepted", C.c_int), ("pcg_iterations", C.c_int),
                ("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("terms_before", C.c_double * NUM_TERMS), ("terms", C.c_double * NUM_TERMS)]


class DenseRecord(C.Structure):
    _fields_ = [("energy_before", C.c_double), ("energy_after", C.c_double),
                ("alpha", C.c_double), ("delta_b_norm", C.c_double),
                ("accepted", C.c_int), ("solved_nonzero", C.c_int)]


class Pairs(C.Structure):
    """ls_pairs: device arrays of the consistency partner rows."""
    _fields_ = [("n", C.c_int64), ("src", C.c_void_p), ("dst", C.c_void_p), ("temporal", C.c_void_p),
                ("weight", C.c_void_p)]


P = C.c_void_p
I64 = C.c_int64
U64 = C.c_uint64
DBL_P = C.POINTER(C.c_double)

# name -> (argtypes); every function returns int except the two string getters
SIGNATURES = {
    "ls_ctx_create": [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Weights),
                      C.POINTER(SolveCfg), C.POINTER(P)],
    "ls_ctx_destroy": [P],
    "ls_set_weights": [P, C.POINTER(Weights), C.POINTER(SolveCfg)],
    "ls_set_stream": [P, P],
    "ls_profile": [P, C.c_int],
    "ls_profile_read": [P, DBL_P],
    "ls_pack_hwc": [P, P, C.c_int, P],
    "ls_unpack_hwc": [P, P, C.c_int, P],
    "ls_set_image": [P, P],
    "ls_sample_consistency": [P, P, P, U64, U64, U64, U64, C.POINTER(I64)],
    "ls_set_pairs": [P, I64, P, P, P, P],
    "ls_pair_count": [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)],
    "ls_get_pairs": [P, P, P, P],
    "ls_set_edge": [P, P],
    "ls_set_prev_r": [P, P],
    "ls_set_anchor": [P, P, P],
    "ls_get_edge": [P, P],
    "ls_get_chroma": [P, P],
    "ls_device_copy": [P, P, I64, P],
    "ls_scan_i32": [P, P, I64, C.c_int, P, P],
    "ls_flood_fill": [P, C.c_int, P, C.c_int, C.c_int, P, P, P],
    "ls_recompose": [P, C.c_int, C.c_int, C.c_int, DBL_P, C.c_int, DBL_P, P, P, P, P, P],
    "ls_all_finite": [P, I64, P, C.POINTER(C.c_int)],
    "ls_chromaticity": [P, C.c_int, C.c_int, P, P],
    "ls_edge_from_chroma": [P, C.c_int, C.c_int, P, P],
    "ls_segment": [P, DBL_P, P],
    "ls_initialize": [P, DBL_P, P, P],
    "ls_energy_terms": [P, DBL_P, P, P, DBL_P],
    "ls_grad_diag": [P, DBL_P, P, P, P],
    "ls_apply_normal": [P, DBL_P, P, P, P],
    "ls_pcg": [P, DBL_P, P, C.c_int, P, DBL_P],
    "ls_gn_step": [P, DBL_P, P, P, C.POINTER(GNRecord)],
    "ls_flip_flop_stream": [P, DBL_P, P, P, P, C.c_int, C.c_int, C.c_double, C.POINTER(GNRecord),
                            C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ls_flip_flop_graph": [P, DBL_P, P, P, C.c_int, C.c_int, C.c_double, C.POINTER(GNRecord),
                           C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ls_flip_flop_batch": [C.POINTER(P), C.c_int, DBL_P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.c_int,
                           C.c_int, C.c_double, C.POINTER(GNRecord), C.POINTER(C.c_int), C.POINTER(C.c_int),
                           C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ls_dense_normal": [P, DBL_P, P, C.c_int, DBL_P, DBL_P],
    "ls_svd_solve": [P, C.c_int, DBL_P, DBL_P, C.c_double, DBL_P],
    "ls_dense_step": [P, DBL_P, P, DBL_P, C.POINTER(DenseRecord)],
    "ls_estimate_palette": [P, C.c_int, C.c_int, C.c_int, U64, U64, U64, U64, DBL_P, C.POINTER(C.c_int), P],
    # per-block residual protocol (energy.py:194-452)
    "ls_block_rows": [P, C.c_int, I64, C.POINTER(I64)],
    "ls_block_residual": [P, DBL_P, P, C.c_int, C.POINTER(Pairs), P, P],
    "ls_block_apply_j": [P, DBL_P, P, C.c_int, C.POINTER(Pairs), P, P],
    "ls_block_apply_jt": [P, DBL_P, P, C.c_int, C.POINTER(Pairs), P, P],
    "ls_block_add_diag": [P, DBL_P, P, C.c_int, C.POINTER(Pairs), P],
    # row bands
    "ls_launch_count": [P, C.POINTER(I64)],
    "ls_add_launches": [P, I64],
    "ls_state_key": [P, P, I64, C.POINTER(I64)],
    "ls_band_set": [P, C.c_int, C.c_int, C.c_int, C.c_int],
    "ls_band_clear": [P],
    "ls_band_buffers": [P, C.POINTER(C.c_void_p)],
    "ls_band_dirs": [P, C.c_int, C.POINTER(P)],
    "ls_band_finalize_group": [C.POINTER(P), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int],
    "ls_copy_slabs": [C.c_int, C.POINTER(P), C.POINTER(P), C.POINTER(I64), C.POINTER(I64), C.POINTER(I64),
                      C.POINTER(C.c_int), P],
    "ls_band_zero_scan": [P, U64, U64, U64, U64, U64, U64, P],
    "ls_band_set_zeros": [P, P, C.c_int],
    "ls_band_eg": [P, DBL_P, P],
    "ls_band_pcg_apply": [P, DBL_P, P, C.c_int],
    "ls_band_pcg_update": [P, C.c_int],
    "ls_band_pcg_finish": [P],
    "ls_band_trial": [P, DBL_P, P, C.c_double, P],
    "ls_band_finalize": [P, C.c_int, P, C.c_int, C.c_int, C.c_double],
    "ls_band_read": [P, DBL_P],
    "ls_band_frame_begin": [P],
    "ls_band_trial_dev": [P, DBL_P, P, C.c_double, P, C.c_int],
    "ls_band_finalize_dev": [P, C.c_int, P, C.c_int, C.c_int, C.c_double, C.c_int],
    "ls_band_step_end": [P, P, P, C.c_int],
    "ls_band_outer_end": [P, C.c_double],
    "ls_band_frame_end": [P, C.c_int, C.POINTER(GNRecord), C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ls_band_dense_accum": [P, DBL_P, P, C.c_int],
    "ls_band_dense_nsums": [P],
    "ls_band_dense_solve": [P, DBL_P, P, C.c_int, C.c_int, DBL_P],
    "ls_band_segment": [P, DBL_P, P],
    "ls_band_segment_final": [P, P, C.c_int, C.c_int, P],
}
BAND_EG, BAND_APPLY, BAND_UPDATE, BAND_TRIAL = 0, 1, 2, 3
ZERO_LIST = 17          # 1 + kMaxRejections
STRING_FUNCS = ("ls_version", "ls_last_error")
# name -> argtypes of the functions returning int64_t
INT64_FUNCS = {"ls_scan_scratch_bytes": [I64]}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    pass


def load(path: Path | str | None = None):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeError(
                f"{p} is missing: build it with `python -m paper_1908_01961_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, argt in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = C.c_int
        for name in STRING_FUNCS:
            fn = getattr(lib, name)
            fn.argtypes = []
            fn.restype = C.c_char_p
        for name, argt in INT64_FUNCS.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = I64
        _lib = lib
        return lib


def symbols():
    return list(SIGNATURES) + list(STRING_FUNCS) + list(INT64_FUNCS)


def last_error() -> str:
    return load().ls_last_error().decode()


def dptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def dbl_array(values):
    import numpy as np
    a = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
    if a.size == 0:
        a = np.zeros(1)
    return a, a.ctypes.data_as(DBL_P)
