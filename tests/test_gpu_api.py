"""GPU parity of the building-block API and the plan consumers.

Golden vectors: tests/golden/c1_api.npz, written by the REFERENCE package
(tests/golden/make_golden.py gen_c1_api) on the C1 inputs: ``pi_step`` at the
reference's converged Gamma (solvers.py:199-224), ``gamma_step``
(:190-196) and ``egw_objective`` (:259-282) on its plan, and the plan
consumers ``row_marginal`` / ``col_marginal`` / ``marginal_error`` /
``kl_divergence`` (measures.py:197-256), ``transport_cost`` /
``eot_primal_value`` (sinkhorn.py:261-284).

Two kinds of checks:
  * end to end: our pi_step / gamma_step / egw_objective from the same
    inputs, within BASELINE's 1e-4 (the plans come from two solvers);
  * reductions only: an ImplicitCoupling built from the REFERENCE's
    potentials, so the device passes (plan.py) are compared with the
    reference's host block loops on the identical plan. The K4 pass is fp64
    throughout (exponents and their 2^x, common.cuh exp2_f64): 1e-10.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def P(cuda):
    import paper_2602_06658_b200 as P

    return P


@pytest.fixture(scope="module")
def api(P):
    gold = golden("c1_api")
    src = P.EmbeddedMeasure(gold["x_feat"], gold["a"])
    tgt = P.EmbeddedMeasure(gold["y_feat"], gold["b"])
    inner = P.SinkhornConfig(eps=0.01, threshold=1e-5, max_inner=200)
    pr = P.pi_step(gold["gamma"], src, tgt, 0.01, inner)
    return gold, src, tgt, pr


def test_pi_step_matches_reference(api):
    gold, src, tgt, pr = api
    cp = pr.coupling
    assert pr.iterations == int(gold["pi_iters"])
    assert pr.converged == bool(gold["pi_converged"])
    assert cp.eps_eff == pytest.approx(float(gold["pi_eps_eff"]), rel=1e-15)
    assert _rel(cp.f, gold["pi_f"]) < TOL
    assert _rel(cp.g, gold["pi_g"]) < TOL
    assert _rel(cp.cost._z, gold["pi_zbar"]) < 1e-12
    assert pr.marginal_err == pytest.approx(float(gold["pi_err"]), rel=1e-3)


def test_gamma_step_and_objective_match_reference(P, api):
    gold, src, tgt, pr = api
    gam = P.gamma_step(pr.coupling, src, tgt)
    assert _rel(gam, gold["gamma_next"]) < TOL
    obj = P.egw_objective(gold["gamma"], pr.coupling, src, tgt, 0.01)
    assert obj == pytest.approx(float(gold["obj"]), rel=TOL)
    obj2 = P.egw_objective(gold["gamma_next"], pr.coupling, src, tgt, 0.01)
    assert obj2 == pytest.approx(float(gold["obj_next"]), rel=TOL)


def test_plan_consumers_end_to_end(P, api):
    gold, src, tgt, pr = api
    cp = pr.coupling
    assert P.kl_divergence(cp) == pytest.approx(float(gold["pi_kl"]), rel=TOL)
    assert P.transport_cost(cp) == pytest.approx(float(gold["pi_tc"]), rel=TOL)
    assert P.eot_primal_value(cp) == pytest.approx(float(gold["pi_eot"]), rel=TOL)
    assert _rel(cp.row_marginal(), gold["pi_row"]) < 1e-3
    assert _rel(cp.col_marginal(), gold["pi_col"]) < 1e-3


@pytest.mark.parametrize("which", ["pi", "res"])
def test_reductions_on_the_reference_plan(P, which):
    """Same plan on both sides (the reference's potentials): the device
    passes reproduce the reference's block loops."""
    gold = golden("c1_api")
    pre = f"{which}_"
    cost = P.SquaredEuclideanCost(gold[pre + "xbar"], gold[pre + "zbar"])
    cp = P.ImplicitCoupling(gold[pre + "f"], gold[pre + "g"], cost, gold["a"], gold["b"],
                            float(gold[pre + "eps_eff"]))
    assert P.kl_divergence(cp) == pytest.approx(float(gold[pre + "kl"]), rel=1e-10)
    assert P.transport_cost(cp) == pytest.approx(float(gold[pre + "tc"]), rel=1e-10)
    assert P.marginal_error(cp) == pytest.approx(float(gold[pre + "me"]), rel=1e-9, abs=1e-14)
    assert _rel(cp.row_marginal(), gold[pre + "row"]) < 1e-10
    assert _rel(cp.col_marginal(), gold[pre + "col"]) < 1e-10
    if which == "pi":
        src = P.EmbeddedMeasure(gold["x_feat"], gold["a"])
        tgt = P.EmbeddedMeasure(gold["y_feat"], gold["b"])
        assert _rel(P.gamma_step(cp, src, tgt), gold["gamma_next"]) < 1e-10
        assert P.egw_objective(gold["gamma"], cp, src, tgt, 0.01) == pytest.approx(
            float(gold["obj"]), rel=1e-10)


def test_densify_blocks_and_marginals_of_a_dense_cost(P):
    """ImplicitCoupling over a DenseCost (no feature form: blocked fp64 device
    pass): densify, marginals and KL against the closed form, and the
    non-finite report of densify (measures.py:209-226)."""
    rng = np.random.default_rng(3)
    a = rng.random(7) + 0.5
    a /= a.sum()
    b = rng.random(5) + 0.5
    b /= b.sum()
    cost = P.DenseCost(rng.random((7, 5)))
    f, g = rng.standard_normal(7) * 0.1, rng.standard_normal(5) * 0.1
    mass = (np.outer(a, b) * np.exp((f[:, None] + g[None, :] - cost.full()) / 0.5)).sum()
    f = f - 0.5 * np.log(mass)
    cp = P.ImplicitCoupling(f, g, cost, a, b, 0.5)
    expect = np.outer(a, b) * np.exp((f[:, None] + g[None, :] - cost.full()) / 0.5)
    assert np.allclose(cp.densify().matrix, expect, rtol=1e-14, atol=0)
    assert np.allclose(np.vstack([blk for _, _, blk in cp.row_blocks(3)]), expect, rtol=1e-14, atol=0)
    assert np.allclose(cp.row_marginal(), expect.sum(1), rtol=1e-13)
    assert np.allclose(cp.col_marginal(), expect.sum(0), rtol=1e-13)
    assert P.kl_divergence(cp) == pytest.approx(P.kl_divergence(cp.densify()), rel=1e-12)
    assert P.transport_cost(cp) == pytest.approx(float((expect * cost.full()).sum()), rel=1e-13)
    bad = P.ImplicitCoupling(np.full(7, 400.0), np.full(5, 400.0), P.DenseCost(np.zeros((7, 5))),
                             a, b, 1.0)
    with pytest.raises(FloatingPointError, match=r"\(0, 0\)"):
        bad.densify()


def test_low_rank_coupling_reductions(P):
    """SeparableLowRankCost plans (the C2 cost form, no squared coordinate)
    through the same K4 identity against the oracle's explicit blocks."""
    from oracle import cntgw_oracle as O
    from paper_2602_06658_b200 import configs

    inst = configs.c2(seed=9, n=700, m=900, k=16)
    n, m = 700, 900
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    cost = P.SeparableLowRankCost(inst.u, inst.v, inst.row_sep, inst.col_sep)
    res = P.sinkhorn(a, b, cost, P.SinkhornConfig(eps=0.05, n_inner=30))
    cp = res.coupling
    ocost = O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep)
    row, col = O.marginals(cp.f, cp.g, ocost, a, b, cp.eps_eff)
    assert _rel(cp.row_marginal(), row) < 1e-10
    assert _rel(cp.col_marginal(), col) < 1e-10
    assert P.kl_divergence(cp) == pytest.approx(O.kl(cp.f, cp.g, ocost, a, b, cp.eps_eff), rel=1e-9)
    tc = sum(float((blk * ocost.rows(i0, i1)).sum())
             for i0, i1, blk in O.plan_blocks(cp.f, cp.g, ocost, a, b, cp.eps_eff))
    assert P.transport_cost(cp) == pytest.approx(tc, rel=1e-9)


def test_large_coupling_consumers_stay_on_device(P):
    """A 2^17 x 2^17 plan (1.7e10 entries, 137 GB dense): marginals, Err, KL
    and <C, pi> come back without any host block (plan.py passes)."""
    from paper_2602_06658_b200 import configs

    pc = configs.c4(seed=1, n=1 << 17)
    src = P.embed_measure(P.DiscreteMeasure(pc.x, pc.a), P.CostSpec("sq_euclidean"), dim=3)
    tgt = P.embed_measure(P.DiscreteMeasure(pc.y, pc.b), P.CostSpec("sq_euclidean"), dim=3)
    pr = P.pi_step(np.zeros((3, 3)), src, tgt, 0.5, P.SinkhornConfig(eps=0.5, n_inner=20))
    cp = pr.coupling
    row, col = cp.row_marginal(), cp.col_marginal()
    assert row.sum() == pytest.approx(col.sum(), rel=1e-10)  # both are the plan's total mass
    assert row.sum() == pytest.approx(1.0, abs=1e-2)
    me = float(np.abs(row - cp.source_weights).sum() + np.abs(col - cp.target_weights).sum())
    # the loop's Err comes from its tentatives, the pass's from explicit sums
    assert me == pytest.approx(pr.marginal_err, rel=1e-3)
    kl = P.kl_divergence(cp)
    assert np.isfinite(kl) and kl >= 0.0
    assert P.eot_primal_value(cp) == pytest.approx(P.transport_cost(cp) + cp.eps_eff * kl, rel=1e-14)
