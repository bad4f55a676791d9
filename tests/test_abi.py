"""Host-only checks of the C-ABI boundary: libkrp.so loads, exports every symbol that
include/krp.h declares, and validates arguments before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "krp.h")).read()
    return sorted(set(re.findall(r"KRP_API\s+[\w\s\*]*?\b(krp_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def krp():
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    return krp


def test_header_declares_the_boundary():
    syms = _header_symbols()
    for name in ["krp_sketch_all_modes", "krp_sketch_mode", "krp_rhosvd", "krp_sthosvd"]:
        assert name in syms


def test_library_exports_every_declared_symbol(krp):
    lib = krp.lib()
    declared = _header_symbols()
    assert sorted(krp.EXPORTED_SYMBOLS) == declared
    for name in declared:
        assert hasattr(lib, name), name


def test_status_strings_and_version(krp):
    lib = krp.lib()
    assert lib.krp_status_string(0) == b"ok"
    assert b"invalid" in lib.krp_status_string(1)
    assert lib.krp_version() >= 10000


def test_argument_validation_without_device(krp):
    lib = krp.lib()
    dims = (ctypes.c_int64 * 3)(8, 8, 8)
    ptrs = (ctypes.c_void_p * 3)(1, 1, 1)
    # null X
    assert lib.krp_sketch_all_modes(None, 3, dims, ptrs, 4, ptrs, None, 0, None) == 1
    # d out of range
    assert lib.krp_sketch_all_modes(1, 1, dims, ptrs, 4, ptrs, None, 0, None) == 1
    assert lib.krp_sketch_all_modes(1, 9, dims, ptrs, 4, ptrs, None, 0, None) == 1
    # R out of range
    assert lib.krp_sketch_all_modes(1, 3, dims, ptrs, 0, ptrs, None, 0, None) == 1
    assert lib.krp_sketch_all_modes(1, 3, dims, ptrs, 257, ptrs, None, 0, None) == 1
    # rhosvd / sthosvd take R <= 64 (reading R20)
    r3 = (ctypes.c_int * 3)(2, 2, 2)
    big = (ctypes.c_int64 * 3)(128, 128, 128)
    assert lib.krp_rhosvd(1, 3, big, r3, 65, ptrs, ptrs, 1, None, None, 0, None) == 1
    # empty mode (a dimension of size 0) and negative sizes are rejected before any launch
    for bad_dims in ((8, 0, 8), (0, 8, 8), (8, 8, -1)):
        dz = (ctypes.c_int64 * 3)(*bad_dims)
        assert lib.krp_sketch_all_modes(1, 3, dz, ptrs, 4, ptrs, None, 0, None) == 1
        assert b"dims" in lib.krp_last_error_message()
    # null omega entry
    bad = (ctypes.c_void_p * 3)(1, None, 1)
    assert lib.krp_sketch_all_modes(1, 3, dims, bad, 4, ptrs, None, 0, None) == 1
    # mode out of range
    assert lib.krp_sketch_mode(1, 3, dims, 3, ptrs, 4, 1, None, 0, None) == 1
    # omega[n] may be null for the single-mode sketch: validation passes on to the workspace step
    # ranks > R, and R > min(I_n, N/I_n) are shape errors
    ranks = (ctypes.c_int * 3)(5, 2, 2)
    assert lib.krp_rhosvd(1, 3, dims, ranks, 4, ptrs, ptrs, 1, None, None, 0, None) == 2
    ranks = (ctypes.c_int * 3)(2, 2, 2)
    assert lib.krp_rhosvd(1, 3, dims, ranks, 9, ptrs, ptrs, 1, None, None, 0, None) == 2
    # workspace too small is reported before any launch
    assert lib.krp_sketch_all_modes(1, 3, dims, ptrs, 4, ptrs, 256, 1, None) == 6
    # inconsistent slab
    assert lib.krp_sketch_all_modes_dist(1, 3, dims, 4, 0, ptrs, 4, ptrs, None, 0, 1, None) == 2
    assert b"slab" in lib.krp_last_error_message()


def test_workspace_sizes_are_sane(krp):
    for op in (krp.OP_SKETCH_ALL, krp.OP_SKETCH_MODE):
        assert krp.krp_workspace_bytes(op, (64, 64, 64), 10) > 0
    assert krp.krp_workspace_bytes(krp.OP_RHOSVD, (64, 64, 64), 10, (5, 5, 5)) > 0
    e = krp.krp_workspace_bytes(krp.OP_RHOSVD_ERR, (64, 64, 64), 10, (5, 5, 5))
    assert e > krp.krp_workspace_bytes(krp.OP_RHOSVD, (64, 64, 64), 10, (5, 5, 5))
    assert krp.krp_workspace_bytes(krp.OP_STHOSVD, (16, 16, 16, 16), 6, (4, 4, 4, 4)) > 0
    h = krp.krp_workspace_bytes(krp.OP_SKETCH_ALL_HOST, (64, 64, 64), 10)
    assert h >= 64 ** 3 * 4
    assert krp.krp_workspace_bytes(99, (4, 4), 2) == 0


def test_product_path_does_not_import_oracle():
    """The CUDA path and the oracle share no code and neither imports the other."""
    pkg = os.path.join(ROOT, "paper_2507_23207_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2507_23207_b200" not in txt and "from paper_2507_23207_b200" not in txt
