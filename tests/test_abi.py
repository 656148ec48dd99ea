"""The C-ABI library loads and exports every symbol include/cntgw_b200.h
declares; argument validation works without a GPU (no compute calls). CPU."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cntgw_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cntgw_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_expected_surface():
    names = _declared()
    for must in ("cntgw_softmin", "cntgw_prep_cols", "cntgw_sweep_init", "cntgw_plan_reduce",
                 "cntgw_outer_reduce_rows", "cntgw_moments", "cntgw_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2602_06658_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding declares a signature for each of them
    assert set(_declared()) <= set(_native.SIGNATURES)


def test_abi_version_and_state_layout():
    from paper_2602_06658_b200 import _native

    assert _native.LIB.cntgw_abi_version() == _native.ABI_VERSION == 4
    assert _native.LIB.cntgw_sweep_state_size() == ctypes.sizeof(_native.SweepStateStruct)


@pytest.mark.parametrize("prec,kd,sq,stride", [
    (0, 1, 0, 4), (0, 3, 1, 8), (0, 4, 0, 8), (0, 16, 0, 20), (0, 32, 1, 36), (0, 64, 1, 68),
    (1, 1, 0, 4), (1, 3, 1, 6), (1, 4, 0, 6), (1, 4, 1, 8), (1, 16, 0, 18), (1, 32, 1, 36),
    (1, 64, 1, 68)])
def test_column_record_stride(prec, kd, sq, stride):
    from paper_2602_06658_b200 import _native

    assert _native.LIB.cntgw_col_stride(prec, kd, sq) == stride


def test_invalid_arguments_report_errors_without_gpu():
    from paper_2602_06658_b200 import _native

    assert _native.LIB.cntgw_col_stride(0, 5, 0) == -1
    assert b"kd=5" in _native.LIB.cntgw_last_error()
    assert _native.LIB.cntgw_col_stride(7, 4, 0) == -1
    rc = _native.LIB.cntgw_softmin(None, 0, 0, 3, 1, None, 3, None, None, None, 0, 0, None, None,
                                   None, None, 0, None)
    assert rc == -1 and b"softmin" in _native.LIB.cntgw_last_error()
    with pytest.raises(_native.NativeError, match="prep_cols"):
        _native.call("cntgw_prep_cols", None, 0, 3, 1, None, 3, None, None, None, 0, None, None)


def test_padding_helpers():
    from paper_2602_06658_b200 import _native, engine

    assert _native.LIB.cntgw_cols_padded(1) == 256
    assert _native.LIB.cntgw_cols_padded(257) == 512
    assert [engine.padded_kd(k) for k in (1, 2, 3, 5, 9, 17, 33, 64)] == [1, 2, 3, 8, 16, 32, 64, 64]
    with pytest.raises(ValueError):
        engine.padded_kd(65)


def test_no_cuda_means_loud_failure():
    import torch

    from paper_2602_06658_b200 import engine

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        engine.require_cuda()


def test_frontend_entry_points_validate_without_gpu():
    """k-means, cost-product and graph entry points reject bad arguments
    before touching the device (CNTGW_EINVAL / ENOSPACE + a message)."""
    from paper_2602_06658_b200 import _native

    L = _native.LIB
    assert L.cntgw_km_assign(None, 10, 3, None, 2, None, None, None) == -1
    assert b"km_assign" in L.cntgw_last_error()
    buf = (ctypes.c_double * 16)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    assert L.cntgw_km_assign(p, 10, 7 + 3, p, 2, p, p, None) == -1  # d = 10 unsupported
    assert b"dimension 10" in L.cntgw_last_error()
    assert L.cntgw_km_draw(p, None, 10, p, 1, p, p, 0, p, p, p, p, 8, None) == -3  # workspace
    assert L.cntgw_km_draw_workspace(10, 1) > 8
    assert L.cntgw_cost_product(9, 0.0, p, 10, 2, p, p, 8, p, None) == -1
    assert b"cost kind 9" in L.cntgw_last_error()
    assert L.cntgw_cost_product(0, 0.0, p, 10, 2, p, p, 12, p, None) == -1
    assert L.cntgw_km_centers(None, 3, None, None, None, 1, None, None, None, None) == -1
    assert L.cntgw_graph_launch(None, None) == -1
