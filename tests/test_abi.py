"""CPU checks of the C-ABI boundary: the in-tree library loads, exports every
entry point include/lumisplit_b200.h declares, and the ctypes binding covers
them.  No device calls (there is no GPU in the build container)."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "lumisplit_b200.h"
LIB = ROOT / "paper_1908_01961_b200" / "liblumisplit_b200.so"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"LS_API\s+[\w\s\*]*?\b(ls_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for name in ("ls_ctx_create", "ls_gn_step", "ls_pcg", "ls_apply_normal", "ls_grad_diag",
                 "ls_energy_terms", "ls_dense_step", "ls_svd_solve", "ls_sample_consistency",
                 "ls_segment", "ls_dense_normal"):
        assert name in syms


@pytest.fixture(scope="module")
def built():
    from paper_1908_01961_b200 import build
    build.build(verbose=False)
    return LIB


def test_library_exports_every_header_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", str(built)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(ls_\w+)", out))
    missing = set(header_symbols()) - exported
    assert not missing, missing


def test_ctypes_binding_matches_header(built):
    from paper_1908_01961_b200 import _lib
    assert set(_lib.symbols()) == set(header_symbols())
    lib = _lib.load()
    assert lib.ls_version().decode().startswith("lumisplit_b200")
    for name in _lib.symbols():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_struct_layouts():
    from paper_1908_01961_b200 import _lib
    assert ctypes.sizeof(_lib.Weights) == 13 * 8 + 8
    assert ctypes.sizeof(_lib.GNRecord) == 3 * 8 + 2 * 4 + 2 * 8 + 16 * 8
    assert ctypes.sizeof(_lib.DenseRecord) == 4 * 8 + 2 * 4


def test_product_path_has_no_oracle_import():
    pkg = ROOT / "paper_1908_01961_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, re.M), py
        assert "lumisplit_oracle" not in src, py
