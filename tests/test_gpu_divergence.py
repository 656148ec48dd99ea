"""GPU parity of the streaming plan reductions, loss decomposition, envelope
gradients, SGW and gradient flow (reference divergence.py:72-410, SURVEY.md
§8(f) row 1) against the reference's own outputs (tests/golden/gradients.npz,
made by tests/golden/make_golden.py on C1-law clouds).

Given the reference's plan factors, the device reductions are compared at
1e-6 (fp32 MUFU exponentials inside an fp64 pass); results that go through
our own solves at the BASELINE tolerance 1e-4."""

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
    from paper_2602_06658_b200 import divergence as D

    gold = golden("gradients")
    src = P.EmbeddedMeasure(gold["x_feat"], gold["a"])
    tgt = P.EmbeddedMeasure(gold["y_feat"], gold["b"])
    xbar = np.column_stack([gold["x_feat"], 0.5 * (gold["x_feat"] ** 2).sum(1)])
    coupling = P.ImplicitCoupling(gold["f"], gold["g"], P.SquaredEuclideanCost(xbar, gold["zbar"]),
                                  gold["a"], gold["b"], float(gold["eps_eff"]))
    return P, D, gold, src, tgt, coupling


def test_plan_reductions_both_sides(env):
    P, D, gold, src, tgt, coupling = env
    pi_y, pi_sy, pit_x, pit_sx, sigma_ss = D._plan_reductions(coupling, src, tgt)
    assert _rel(pi_y, gold["pi_y"]) < 1e-6
    assert _rel(pi_sy, gold["pi_sy"]) < 1e-6
    assert _rel(pit_x, gold["pit_x"]) < 1e-6
    assert _rel(pit_sx, gold["pit_sx"]) < 1e-6
    assert sigma_ss == pytest.approx(float(gold["sigma_ss"]), rel=1e-6)


def test_grad_constant_closed_form(env):
    P, D, gold, src, tgt, coupling = env
    got = D._grad_constant(src, tgt.trace_second_moment())
    assert _rel(got, gold["grad_const"]) < 1e-12


def test_feature_gradients_and_loss_decomposition(env):
    P, D, gold, src, tgt, coupling = env
    gsrc, gtgt = P.feature_gradients(src, tgt, gold["gamma"], coupling)
    assert _rel(gsrc, gold["gsrc"]) < 1e-6
    assert _rel(gtgt, gold["gtgt"]) < 1e-6
    rep = P.gw_value_report(gold["gamma"], coupling, src, tgt, 0.05)
    got = [rep.value, rep.constant, rep.gamma_sq, rep.kl_term, rep.cross_term, rep.sigma_ss]
    np.testing.assert_allclose(got, gold["report"], rtol=1e-6)
    assert P.quartic_loss(coupling, src, tgt) == pytest.approx(float(gold["quartic"]), rel=1e-6)


def test_egw_gradient_through_a_solve(env):
    P, D, gold, src, tgt, coupling = env
    cfg = P.make_config(0.05, n_inner=60, max_outer=6, delta_outer=1e-12)
    pg = P.egw_gradient(src, tgt, cfg)
    assert pg.value == pytest.approx(float(gold["value"]), rel=TOL)
    assert _rel(pg.source, gold["gsrc"]) < TOL
    assert _rel(pg.target, gold["gtgt"]) < TOL
    with pytest.raises(ValueError, match="configuration"):
        P.egw_gradient(src, tgt)


def test_sgw_three_solves(env):
    P, D, gold, src, tgt, coupling = env
    cfg = P.make_config(0.05, n_inner=60, max_outer=6, delta_outer=1e-12)
    with pytest.warns(RuntimeWarning, match="temperature heuristic"):
        res = P.sgw(src, tgt, cfg)
    assert res.value == pytest.approx(float(gold["sgw_value"]), rel=TOL)
    parts = [res.cross.value, res.self_src.value, res.self_tgt.value]
    np.testing.assert_allclose(parts, gold["sgw_parts"], rtol=TOL)
    # a measure against itself: one self solve, exactly zero
    with pytest.warns(RuntimeWarning):
        assert P.sgw(src, src, cfg).value == 0.0


def test_gradient_flow_trajectory(env):
    P, D, gold, src, tgt, coupling = env
    n, mt = gold["flow_points"].shape[0], gold["flow_tau"].shape[0]
    tau = P.embed_measure(P.DiscreteMeasure(gold["flow_tau"], np.full(mt, 1.0 / mt)),
                          P.CostSpec("sq_euclidean"), dim=3)
    cfg = P.make_config(0.1, n_inner=40, max_outer=4, delta_outer=1e-12)
    fl = P.gradient_flow(P.DiscreteMeasure(gold["flow_points"], np.full(n, 1.0 / n)), [(1.0, tau)],
                         cfg, steps=3, step_size=0.05)
    assert _rel(np.array(fl.positions), gold["flow_positions"]) < TOL
    assert _rel(fl.objectives, gold["flow_objectives"]) < TOL
    with pytest.raises(ValueError, match="positive weight"):
        P.gradient_flow(P.DiscreteMeasure(gold["flow_points"], np.full(n, 1.0 / n)), [(0.0, tau)],
                        cfg, steps=1)
