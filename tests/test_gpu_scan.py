"""The device int32 scan (csrc/ls_aux.cu k_scan: int4 I/O, decoupled look-back
by a whole warp) against numpy, at sizes around its 2048-value tiles and
large enough that the look-back walks several 32-tile windows."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _scan(x: np.ndarray, op: int) -> np.ndarray:
    from paper_1908_01961_b200 import _lib as L
    lib = L.load()
    n = x.size
    t = torch.as_tensor(x, dtype=torch.int32, device="cuda")
    out = torch.full_like(t, -7)
    scratch = torch.empty(max(1, int(lib.ls_scan_scratch_bytes(n))), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.ls_scan_i32(C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr()), n, op,
                         C.c_void_p(scratch.data_ptr()), C.c_void_p(st))
    assert rc == L.LS_OK, L.last_error()
    return out.cpu().numpy()


@pytest.mark.parametrize("n", [1, 7, 8, 9, 2047, 2048, 2049, 65536 + 3, 2073601, 8 * 2048 * 64 + 5])
def test_exclusive_sum_matches_numpy(n):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 9, size=n).astype(np.int32)
    ref = np.concatenate([[0], np.cumsum(x)[:-1]]).astype(np.int32)
    assert np.array_equal(_scan(x, 0), ref)


@pytest.mark.parametrize("n", [1, 5, 2048, 2051, 300001, 2073600])
def test_inclusive_max_matches_numpy(n):
    rng = np.random.default_rng(n + 1)
    x = rng.integers(-1000, 1000, size=n).astype(np.int32)
    x[rng.random(n) < 0.5] = np.iinfo(np.int32).min      # runs of "no value" (segmentation's -1 keys)
    assert np.array_equal(_scan(x, 1), np.maximum.accumulate(x))


def test_unaligned_views_take_the_scalar_path():
    rng = np.random.default_rng(3)
    base = torch.as_tensor(rng.integers(0, 5, size=10007), dtype=torch.int32, device="cuda")
    from paper_1908_01961_b200 import _lib as L
    lib = L.load()
    src, n = base[1:], base.numel() - 1                    # 4-byte aligned, not 16
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")[1:]
    scratch = torch.empty(int(lib.ls_scan_scratch_bytes(n)), dtype=torch.uint8, device="cuda")
    rc = lib.ls_scan_i32(C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr()), n, 0,
                         C.c_void_p(scratch.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == L.LS_OK
    x = src.cpu().numpy()
    assert np.array_equal(out.cpu().numpy(), np.concatenate([[0], np.cumsum(x)[:-1]]).astype(np.int32))
