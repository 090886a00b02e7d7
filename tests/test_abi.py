"""CPU checks of the C-ABI boundary: libp2p.so loads without a GPU, exports every function include/p2p.h declares,
the ctypes structs match the header, and the status strings are wired.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "p2p.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(p2p_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2511_21535_b200 as P
    from paper_2511_21535_b200 import build as B
    B.build()
    return P.lib()


def test_header_declares_the_north_star_entry_points():
    decl = _declared()
    for name in ["p2p_plan_create", "p2p_restructure", "p2p_eval", "p2p_destroy"]:
        assert name in decl


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_names_match_the_abi(lib):
    import paper_2511_21535_b200 as P
    for name in _declared():
        assert callable(getattr(P, name)), name


def test_status_strings_and_version(lib):
    import paper_2511_21535_b200 as P
    assert P.p2p_status_string(P.P2P_OK) == "P2P_OK"
    assert P.p2p_status_string(P.P2P_ERR_OUT_OF_DOMAIN) == "P2P_ERR_OUT_OF_DOMAIN"
    assert lib.p2p_abi_version() == 1


def test_struct_layout():
    import paper_2511_21535_b200 as P
    # offsets follow the C layout of p2p_config / p2p_info (x86-64 SysV)
    assert P.P2PConfig.box_size.offset == 16
    assert P.P2PConfig.lo.offset == 24
    assert P.P2PConfig.nbox.offset == 48
    assert P.P2PConfig.stream.offset == 88
    assert ctypes.sizeof(P.P2PConfig) == 104
    assert ctypes.sizeof(P.P2PInfo) == 56


def test_argument_validation_without_gpu(lib):
    """pure-host validation paths run before any CUDA call"""
    import paper_2511_21535_b200 as P
    cfg = P.make_config(P.P2P_GRAVITY, P.P2P_FP32, 0.25, (0, 0, 0), (4, 4, 4), 0b111, eps=0.0)
    out = ctypes.c_void_p()
    s = lib.p2p_plan_create(ctypes.byref(cfg), 0, None, None, ctypes.byref(out))
    assert s == P.P2P_ERR_INVALID_ARGUMENT and "eps" in P.p2p_last_error()
    cfg = P.make_config(P.P2P_GRAVITY, P.P2P_FP32, 0.25, (0, 0, 0), (2, 4, 4), 0b111, eps=1e-3)
    s = lib.p2p_plan_create(ctypes.byref(cfg), 0, None, None, ctypes.byref(out))
    assert s == P.P2P_ERR_INVALID_ARGUMENT and "nbox >= 3" in P.p2p_last_error()
    cfg = P.make_config(P.P2P_GRAVITY, P.P2P_FP32, -1.0, (0, 0, 0), (4, 4, 4), 0, eps=1e-3)
    assert lib.p2p_plan_create(ctypes.byref(cfg), 0, None, None, ctypes.byref(out)) == P.P2P_ERR_INVALID_ARGUMENT
    cfg = P.make_config(P.P2P_HELMHOLTZ2D, P.P2P_FP32, 1.0, (0, 0), (4, 4), 0, k=1.0, t=15)
    assert lib.p2p_plan_create(ctypes.byref(cfg), 0, None, None, ctypes.byref(out)) == P.P2P_ERR_INVALID_ARGUMENT
    cfg = P.make_config(P.P2P_GRAVITY, P.P2P_FP32, 1e-3, (0, 0, 0), (2048, 4, 4), 0, eps=1e-3)
    assert lib.p2p_plan_create(ctypes.byref(cfg), 0, None, None, ctypes.byref(out)) == P.P2P_ERR_UNSUPPORTED
    assert lib.p2p_eval(None, 0, None, None) == P.P2P_ERR_INVALID_ARGUMENT
    lib.p2p_destroy(None)  # NULL-safe


def test_product_does_not_import_oracle():
    """the product package never references oracle/ (parity would be void otherwise)"""
    pkg = os.path.join(ROOT, "paper_2511_21535_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "p2p_oracle" not in txt, f


def test_binding_rejects_dtype_and_shape_mismatch():
    """the ABI cannot see dtypes, so the binding checks them (float64 masses with float32 positions
    would otherwise be read as float32 and return P2P_OK with garbage)"""
    import torch
    import paper_2511_21535_b200 as P
    pos = torch.zeros(8, 3, dtype=torch.float32)
    with pytest.raises(P.P2PError):
        P._check_inputs(P.P2P_GRAVITY, pos, torch.zeros(8, dtype=torch.float64))
    with pytest.raises(P.P2PError):
        P._check_inputs(P.P2P_GRAVITY, pos, torch.zeros(7, dtype=torch.float32))
    with pytest.raises(P.P2PError):
        P._check_inputs(P.P2P_GRAVITY, torch.zeros(8, 2), torch.zeros(8))
    with pytest.raises(P.P2PError):
        P._check_inputs(P.P2P_HELMHOLTZ2D, torch.zeros(8, 2), torch.zeros(8))
    with pytest.raises(P.P2PError):
        P._check_inputs(P.P2P_GRAVITY, pos, torch.zeros(8), dtype=torch.float64)
    P._check_inputs(P.P2P_GRAVITY, pos, torch.zeros(8))
    P._check_inputs(P.P2P_HELMHOLTZ2D, torch.zeros(8, 2, dtype=torch.float64), torch.zeros(8, 2, dtype=torch.float64))


def test_build_stamp_records_the_flags(lib):
    """libp2p.so built with experiment flags is rebuilt when P2P_NVCC_FLAGS changes"""
    from paper_2511_21535_b200 import build as B
    assert os.path.exists(B.STAMP) and open(B.STAMP).read() == B._flag_stamp()
    old = os.environ.get("P2P_NVCC_FLAGS")
    os.environ["P2P_NVCC_FLAGS"] = "-DP2P_SOME_EXPERIMENT"
    try:
        assert B._flag_stamp() != open(B.STAMP).read()
    finally:
        if old is None:
            del os.environ["P2P_NVCC_FLAGS"]
        else:
            os.environ["P2P_NVCC_FLAGS"] = old
