"""ctypes binding of the C-ABI library ``libcntgw_b200.so`` (include/cntgw_b200.h).

There is no CPU fallback: if the library is missing, importing this module
raises, and every entry point requires CUDA device buffers. Tensors cross the
boundary as raw device pointers (``tensor.data_ptr()``) plus sizes; the
stream is torch's current CUDA stream, so launches are graph-capturable.
"""

from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libcntgw_b200.so")

c_int, c_double, c_float, c_size_t = ctypes.c_int, ctypes.c_double, ctypes.c_float, ctypes.c_size_t
c_i64, c_vp = ctypes.c_int64, ctypes.c_void_p


class SweepStateStruct(ctypes.Structure):
    """Host mirror of ``cntgw_sweep_state`` (include/cntgw_b200.h)."""

    _fields_ = [
        ("eps", c_double), ("anneal_from", c_double), ("threshold", c_double),
        ("eps_n", c_double), ("gap_r", c_double), ("gap_c", c_double),
        ("lam_d", c_double), ("sqrt_lam_d", c_double),
        ("lam", c_float), ("sqrt_lam", c_float),
        ("max_sweeps", ctypes.c_int32), ("mode", ctypes.c_int32), ("sweep", ctypes.c_int32),
        ("applied", ctypes.c_int32), ("done", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("check", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


class SolveConfigStruct(ctypes.Structure):
    """Host mirror of ``cntgw_solve_config`` (include/cntgw_b200.h)."""

    _fields_ = [
        ("eps", c_double), ("mode", c_int), ("n_inner", c_int), ("threshold", c_double),
        ("max_inner", c_int), ("anneal_from", c_double), ("max_outer", c_int),
        ("delta_outer", c_double), ("precision", c_int),
    ]


class OuterStateStruct(ctypes.Structure):
    """Host mirror of ``cntgw_outer_state`` (include/cntgw_b200.h)."""

    _fields_ = [
        ("constant", c_double), ("eps_outer", c_double), ("delta_outer", c_double),
        ("prev_objective", c_double), ("t0_ns", c_double),
        ("max_outer", ctypes.c_int32), ("step", ctypes.c_int32), ("ups", ctypes.c_int32),
        ("done", ctypes.c_int32), ("converged", ctypes.c_int32), ("error", ctypes.c_int32),
        ("has_prev", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


F32, F64, TF32X3, F32C, F64S = 0, 1, 2, 3, 4  # cntgw_precision
ABI_VERSION = 4  # CNTGW_ABI_VERSION

# name -> (restype, argtypes); every symbol include/cntgw_b200.h declares
SIGNATURES = {
    "cntgw_abi_version": (c_int, []),
    "cntgw_last_error": (ctypes.c_char_p, []),
    "cntgw_sweep_state_size": (c_int, []),
    "cntgw_col_stride": (c_int, [c_int, c_int, c_int]),
    "cntgw_locality_codes": (c_int, [c_vp, c_i64, c_int, c_i64, c_vp, c_vp, c_vp]),
    "cntgw_ctr_rows_bytes": (c_size_t, [c_i64, c_int, c_int]),
    "cntgw_ctr_cols_bytes": (c_size_t, [c_i64, c_int, c_int]),
    "cntgw_prep_rows_ctr": (c_int, [c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "cntgw_prep_cols_ctr": (c_int, [c_vp, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                    c_vp, c_vp]),
    "cntgw_cols_padded": (c_i64, [c_i64]),
    "cntgw_sweep_init": (c_int, [c_vp, c_double, c_double, c_double, c_int, c_int, c_vp]),
    "cntgw_sweep_begin": (c_int, [c_vp, c_vp]),
    "cntgw_gap_blocks": (c_int, [c_i64]),
    "cntgw_sweep_gap": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "cntgw_sweep_finish": (c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "cntgw_sweep_apply": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    "cntgw_prep_cols": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                c_vp, c_vp]),
    "cntgw_softmin_workspace": (c_size_t, [c_int, c_i64, c_i64, c_int, c_int]),
    "cntgw_softmin": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp,
                              c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_size_t, c_vp]),
    "cntgw_lse_finalize": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "cntgw_softmin_dense": (c_int, [c_vp, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64,
                                    c_vp, c_vp]),
    "cntgw_plan_reduce_workspace": (c_size_t, [c_i64, c_i64, c_int, c_int]),
    "cntgw_comm_available": (c_int, []),
    "cntgw_comm_nccl_version": (c_int, []),
    "cntgw_comm_id_bytes": (c_int, []),
    "cntgw_comm_unique_id": (c_int, [c_vp]),
    "cntgw_comm_init": (c_int, [c_vp, c_int, c_int, c_vp]),
    "cntgw_comm_destroy": (c_int, [c_vp]),
    "cntgw_comm_allreduce": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp]),
    "cntgw_lse_rescale": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "cntgw_comm_combine_lse": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "cntgw_solver_create": (c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp,
                                    c_vp, c_vp, c_i64, c_vp]),
    "cntgw_solver_destroy": (c_int, [c_vp]),
    "cntgw_solver_init_potentials": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cntgw_solver_run": (c_int, [c_vp, c_double, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cntgw_solver_results": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "cntgw_gw_constant": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_vp]),
    "cntgw_select_order": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "cntgw_f64s_rows_bytes": (c_size_t, [c_i64, c_int]),
    "cntgw_f64s_plan_density": (c_int, [c_int, c_int, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "cntgw_f64s_plan_layout": (c_int, [c_int, c_int, c_i64, c_i64, c_vp]),
    "cntgw_prep_rows_f64s": (c_int, [c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "cntgw_prep_cols_f64s": (c_int, [c_vp, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                     c_vp, c_vp]),
    "cntgw_update_cols_f64s": (c_int, [c_vp, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                     c_vp, c_vp]),
    "cntgw_plan_reduce_f64s": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp,
                                       c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_size_t, c_vp, c_size_t, c_vp]),
    "cntgw_plan_reduce_ctr_workspace": (c_size_t, [c_i64, c_int]),
    "cntgw_plan_reduce_ctr": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp,
                                      c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_size_t, c_vp, c_size_t, c_vp]),
    "cntgw_plan_reduce": (c_int, [c_vp, c_int, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_size_t, c_vp]),
    "cntgw_apply_operator": (c_int, [c_vp, c_int, c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64,
                                     c_vp]),
    "cntgw_outer_reduce_workspace": (c_size_t, [c_i64, c_int, c_int]),
    "cntgw_outer_reduce_rows": (c_int, [c_vp, c_i64, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp,
                                        c_vp, c_i64, c_vp, c_vp, c_size_t, c_vp]),
    "cntgw_outer_reduce_cols": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_size_t,
                                        c_vp]),
    "cntgw_moments_workspace": (c_size_t, [c_i64, c_int]),
    "cntgw_moments": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_size_t, c_vp]),
    "cntgw_outer_state_size": (c_int, []),
    "cntgw_outer_init": (c_int, [c_vp, c_double, c_double, c_double, c_int, c_vp]),
    "cntgw_outer_finish": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp]),
    "cntgw_graph_begin": (c_int, [c_vp]),
    "cntgw_graph_while_begin": (c_int, [c_vp, c_vp, ctypes.POINTER(ctypes.c_uint64)]),
    "cntgw_graph_while_end": (c_int, [c_vp]),
    "cntgw_graph_set_condition": (c_int, [ctypes.c_uint64, c_vp, c_vp]),
    "cntgw_graph_end": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "cntgw_graph_launch": (c_int, [c_vp, c_vp]),
    "cntgw_graph_destroy": (c_int, [c_vp]),
    "cntgw_cost_product": (c_int, [c_int, c_double, c_vp, c_i64, c_int, c_vp, c_vp, c_int, c_vp, c_vp]),
    "cntgw_km_draw_workspace": (c_size_t, [c_i64, c_int]),
    "cntgw_km_draw": (c_int, [c_vp, c_vp, c_i64, c_vp, c_int, c_vp, c_vp, c_int, c_vp, c_vp, c_vp,
                              c_vp, c_size_t, c_vp]),
    "cntgw_km_update_d2": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp]),
    "cntgw_km_assign": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "cntgw_km_centers": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
}


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero cntgw_status."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cntgw_abi_version() != ABI_VERSION:
        raise ImportError("libcntgw_b200.so ABI version mismatch; rebuild the extension")
    if lib.cntgw_sweep_state_size() != ctypes.sizeof(SweepStateStruct):
        raise ImportError("cntgw_sweep_state layout mismatch between header and host mirror")
    if lib.cntgw_outer_state_size() != ctypes.sizeof(OuterStateStruct):
        raise ImportError("cntgw_outer_state layout mismatch between header and host mirror")
    return lib


LIB = _load()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = LIB.cntgw_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'cntgw'} failed ({rc}): {msg}")


def call(name: str, *args):
    """Call an int-returning entry point and raise on a non-zero status."""
    rc = getattr(LIB, name)(*args)
    check(rc, name)
    return rc
