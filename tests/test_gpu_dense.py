"""GPU parity of the dense-plan GW baselines and the coupling CSV formats
(reference solvers.py:384-665, measures.py:259-360)
against the reference's own outputs (tests/golden/dense.npz)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def env(cuda):
    import paper_2602_06658_b200 as P
    from paper_2602_06658_b200 import kernels as K

    gold = golden("dense")
    cx = K.cost_matrix(K.CostSpec("sq_euclidean"), P.DiscreteMeasure(gold["x"], gold["a"]))
    cy = K.cost_matrix(K.CostSpec("euclidean"), P.DiscreteMeasure(gold["y"], gold["b"]))
    return P, gold, cx, cy


@pytest.mark.parametrize("name", ["kgw", "egw"])
def test_dense_baselines_match_reference(env, name):
    P, gold, cx, cy = env
    fn = P.solve_kernel_gw if name == "kgw" else P.solve_entropic_gw
    cfg = P.make_config(0.05, n_inner=40, max_outer=6, delta_outer=1e-12)
    res = fn(cx, cy, gold["a"], gold["b"], cfg)
    assert res.gamma is None and isinstance(res.coupling, P.DenseCoupling)
    assert _rel(res.trace.objectives, gold[f"{name}__obj"]) < TOL
    assert _rel(res.trace.gamma_deltas, gold[f"{name}__delta"]) < 1e-3
    assert _rel(res.coupling.matrix, gold[f"{name}__pi"]) < TOL
    assert res.value == pytest.approx(float(gold[f"{name}__value"]), rel=TOL)


def test_adaptive_wrapper_around_kernel_solver(env):
    P, gold, cx, cy = env
    cfg = P.make_config(0.05, n_inner=3, max_outer=8, delta_outer=1e-12)
    res = P.solve_adaptive(P.solve_kernel_gw, cx, cy, gold["a"], gold["b"], cfg=cfg)
    assert list(res.schedule) == list(gold["ad__sched"])
    assert _rel(res.trace.objectives, gold["ad__obj"]) < TOL


def test_dense_guard_and_init(env):
    P, gold, cx, cy = env
    cfg = P.make_config(0.05, n_inner=5, max_outer=2, max_dense_entries=100)
    with pytest.raises(ValueError, match="memory guard"):
        P.solve_kernel_gw(cx, cy, gold["a"], gold["b"], cfg)
    cfg = P.make_config(0.05, n_inner=5, max_outer=2, init="gamma", init_gamma=np.eye(3))
    with pytest.raises(ValueError, match="not available for dense solvers"):
        P.solve_entropic_gw(cx, cy, gold["a"], gold["b"], cfg)


def test_coupling_csv_round_trip(env, tmp_path):
    P, gold, cx, cy = env
    cfg = P.make_config(0.05, n_inner=40, max_outer=2, delta_outer=1e-12)
    res = P.solve_kernel_gw(cx, cy, gold["a"], gold["b"], cfg)
    for dense in (False, True):
        path = tmp_path / f"c{int(dense)}.csv"
        P.save_coupling(path, res.coupling, dense=dense, header="kernel GW\nstep 2")
        back = P.load_coupling(path, gold["a"], gold["b"])
        keep = res.coupling.matrix >= 1e-12
        assert np.array_equal(back.matrix[keep], res.coupling.matrix[keep])
    pc = P.DiscreteMeasure(gold["x"], gold["a"])
    P.save_point_cloud(tmp_path / "p.csv", pc, header="c1")
    back = P.load_point_cloud(tmp_path / "p.csv")
    assert np.array_equal(back.points, pc.points) and np.array_equal(back.weights, pc.weights)
