"""The solve-level C ABI (cntgw_solver_*, csrc/solve.cu) against the Python
package's solve and the reference's C1 golden values.

A caller without Python builds a handle from device features and weights,
gets the loss constant (cntgw_gw_constant) and the default interaction
potentials, and runs one graph-captured solve. It issues the same kernels in
the same order as solvers._DeviceSolve, so trajectories agree with the
package to rounding (the half squared norms are formed on the device here,
from numpy there) and with the reference to BASELINE's 1e-4.
"""

import ctypes

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _native_solve(x, a, y, b, eps, precision, n_inner=0, threshold=0.0, max_inner=10000, max_outer=20,
                  delta_outer=1e-5, order_x=None, order_y=None):
    import torch

    from paper_2602_06658_b200._native import SolveConfigStruct, call

    dev = torch.device("cuda", 0)
    X = torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=dev)
    Y = torch.as_tensor(np.ascontiguousarray(y), dtype=torch.float64, device=dev)
    A = torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    B = torch.as_tensor(np.ascontiguousarray(b), dtype=torch.float64, device=dev)
    (n, d), (m, e) = X.shape, Y.shape
    s = torch.cuda.current_stream().cuda_stream
    cfg = SolveConfigStruct(eps=eps, mode=1, n_inner=n_inner, threshold=threshold, max_inner=max_inner,
                            anneal_from=0.0, max_outer=max_outer, delta_outer=delta_outer, precision=precision)
    h = ctypes.c_void_p()
    ox = 0 if order_x is None else order_x.data_ptr()
    oy = 0 if order_y is None else order_y.data_ptr()
    call("cntgw_solver_create", ctypes.byref(h), X.data_ptr(), n, d, Y.data_ptr(), m, e, A.data_ptr(),
         B.data_ptr(), ox, oy, ctypes.byref(cfg), None, 0, s)
    try:
        const = ctypes.c_double()
        call("cntgw_gw_constant", X.data_ptr(), n, d, A.data_ptr(), Y.data_ptr(), m, e, B.data_ptr(),
             ctypes.byref(const), s)
        f = torch.empty(n, dtype=torch.float64, device=dev)
        g = torch.empty(m, dtype=torch.float64, device=dev)
        call("cntgw_solver_init_potentials", h, f.data_ptr(), g.data_ptr(), s)
        gamma = torch.zeros(d * e, dtype=torch.float64, device=dev)
        gprev = torch.zeros(d * e, dtype=torch.float64, device=dev)
        trace = (ctypes.c_double * (5 * max_outer))()
        status = (ctypes.c_int * 4)()
        call("cntgw_solver_run", h, const.value, gamma.data_ptr(), gprev.data_ptr(), f.data_ptr(),
             g.data_ptr(), trace, status, s)
        am = torch.empty(n, dtype=torch.int64, device=dev)
        eps_eff = ctypes.c_double()
        call("cntgw_solver_results", h, None, am.data_ptr(), ctypes.byref(eps_eff), s)
        am = am.cpu().numpy()
    finally:
        call("cntgw_solver_destroy", h)
    steps = status[0]
    rows = np.array(trace[: 5 * steps]).reshape(steps, 5)
    # reference-form potentials of the returned coupling (built on Gamma_t)
    f_ref = (f + (X * X).sum(1)).cpu().numpy()
    zy = Y @ gprev.view(d, e).t()
    g_ref = (g + (zy * zy).sum(1)).cpu().numpy()
    return dict(trace=rows, converged=bool(status[1]), error=bool(status[2]),
                gamma=gamma.view(d, e).cpu().numpy(), gamma_prev=gprev.view(d, e).cpu().numpy(),
                f=f_ref, g=g_ref, constant=const.value, eps_eff=eps_eff.value, argmax=am)


@pytest.fixture(scope="module")
def P(cuda):
    import paper_2602_06658_b200 as P

    return P


@pytest.mark.parametrize("prec_name", ["f64", "f32"])
def test_native_solve_c1_matches_package_and_reference(P, prec_name, monkeypatch):
    from paper_2602_06658_b200._native import F32, F64

    gold = golden("c1_solve")
    prec = {"f64": F64, "f32": F32}[prec_name]
    nat = _native_solve(gold["x_feat"], gold["a"], gold["y_feat"], gold["b"], 0.01, prec, threshold=1e-5,
                        max_inner=200, max_outer=20)
    monkeypatch.setenv("CNTGW_PRECISION", prec_name)
    src = P.EmbeddedMeasure(gold["x_feat"], gold["a"])
    tgt = P.EmbeddedMeasure(gold["y_feat"], gold["b"])
    res = P.solve_cnt_gw(src, tgt, P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20))
    assert nat["constant"] == pytest.approx(float(gold["constant"]), rel=1e-12)
    assert [int(v) for v in nat["trace"][:, 3]] == res.trace.inner_iters == gold["inner_iters"].tolist()
    assert nat["converged"] == res.converged and not nat["error"]
    # (fp64 path: the two drivers differ only in how the half squared norms
    # were rounded; the fp32 path carries that difference through fp32 terms)
    tol = 1e-9 if prec_name == "f64" else 1e-6
    assert _rel(nat["trace"][:, 0], res.trace.objectives) < tol
    assert _rel(nat["gamma"], res.gamma) < tol
    assert _rel(nat["f"], res.coupling.f) < tol and _rel(nat["g"], res.coupling.g) < tol
    assert nat["eps_eff"] == pytest.approx(res.coupling.eps_eff, rel=1e-15)
    # the reference's own values
    assert _rel(nat["f"], gold["f"]) < 1e-4 and _rel(nat["g"], gold["g"]) < 1e-4
    assert abs(nat["trace"][-1, 0] - float(gold["value"])) < 1e-4 * abs(float(gold["value"]))
    sure = gold["argmax_gap"] > 1e-3
    assert np.array_equal(nat["argmax"][sure], gold["argmax"][sure])


def test_native_solve_c5_law_on_the_measured_plan_path(P, monkeypatch):
    """C5 law (reduced N, 64/32-dim, fixed budget) on CNTGW_F64S with the
    package's cluster orders: the same trajectory as the package's solve and
    the reference golden's objectives."""
    import torch

    from paper_2602_06658_b200 import solvers
    from paper_2602_06658_b200._native import F64S

    gold = golden("c5law_solve")
    x, y, a, b = gold["x_feat"], gold["y_feat"], gold["a"], gold["b"]
    monkeypatch.setenv("CNTGW_PRECISION", "f64s")
    src, tgt = P.EmbeddedMeasure(x, a), P.EmbeddedMeasure(y, b)
    cfg = P.make_config(0.02, n_inner=200, max_outer=3, delta_outer=1e-12)
    st = solvers._CntGwState(src, tgt, cfg)
    objs = [st.step().objective for _ in range(3)]
    ox, oy = st.dev.src.locality(), st.dev.tgt.locality()
    nat = _native_solve(x, a, y, b, 0.02, F64S, n_inner=200, max_outer=3, delta_outer=1e-12,
                        order_x=ox, order_y=oy)
    assert nat["trace"].shape[0] == 3
    # cold law (|exponents| ~ 1e6 log2 units): rounding differences of the
    # half squared norms (device vs numpy) reach ~1e-8 of the objective
    assert _rel(nat["trace"][:, 0], objs) < 1e-6
    assert _rel(nat["trace"][:, 0], gold["objective"][:3]) < 1e-4
    assert _rel(nat["gamma"], st.gamma) < 1e-5
    torch.cuda.synchronize()
