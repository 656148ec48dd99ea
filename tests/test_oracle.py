"""Pin the CPU oracle (oracle/cntgw_oracle.py) to the reference's own outputs.

The golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py); here the oracle restatement must reproduce them
to fp64 round-off, plus the reference tests' known answers. CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import cntgw_oracle as O


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


CASES = ["dense_sym_fixed", "dense_std_fixed", "dense_sym_tau", "dense_std_tau", "dense_anneal",
         "dense_anneal_trunc", "dense_cap", "dense_big"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_sinkhorn_cases(name):
    g = golden("sinkhorn_cases")
    kw = eval(str(g[f"{name}__kw"]))
    eps = kw.pop("eps")
    res = O.sinkhorn(g[f"{name}__a"], g[f"{name}__b"], O.Dense(g[f"{name}__c"]), eps, **kw)
    assert _rel(res["f"], g[f"{name}__f"]) < 1e-12
    assert _rel(res["g"], g[f"{name}__g"]) < 1e-12
    assert res["iterations"] == int(g[f"{name}__iters"])
    assert res["converged"] == bool(g[f"{name}__conv"])
    assert res["eps_eff"] == float(g[f"{name}__eps_eff"])
    assert res["marginal_err"] == pytest.approx(float(g[f"{name}__err"]), rel=1e-9, abs=1e-15)


def test_oracle_sq_euclidean_case():
    g = golden("sinkhorn_cases")
    a, b = np.full(40, 1 / 40), np.full(33, 1 / 33)
    res = O.sinkhorn(a, b, O.SqEuclid(g["sqe__x"], g["sqe__z"]), 0.4, n_inner=21)
    assert _rel(res["f"], g["sqe__f"]) < 1e-12
    assert _rel(res["g"], g["sqe__g"]) < 1e-12


def test_oracle_c2_small():
    g = golden("c2_small")
    n = g["u"].shape[0]
    w = np.full(n, 1 / n)
    cost = O.LowRank(g["u"], g["v"], g["ra"], g["cb"])
    res = O.sinkhorn(w, w, cost, float(g["eps"]), mode="standard", n_inner=1,
                     warm=(np.zeros(n), g["g0"].astype(float)))
    assert _rel(res["f"], g["f"]) < 1e-12
    assert _rel(res["g"], g["g"]) < 1e-12


def test_oracle_c2_full_size_subsample():
    """Row-subsample f-update at N=M=2^20 against the reference's _softmin."""
    from paper_2602_06658_b200 import configs

    gold = golden("c2_subsample")
    inst = configs.c2(seed=int(gold["seed"]), n=int(gold["n"]), k=int(gold["k"]))
    cost = O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep)
    got = O.softmin(cost, inst.log_wb, inst.g.astype(float), inst.eps, row_idx=gold["rows"][:8])
    assert _rel(got, gold["f_rows"][:8]) < 1e-12


def test_oracle_c1_full_solve():
    gold = golden("c1_solve")
    x, y, a, b = gold["x_feat"], gold["y_feat"], gold["a"], gold["b"]
    res = O.solve_cnt_gw(x, a, y, b, 0.01, dict(threshold=1e-5, max_inner=200), max_outer=20)
    assert res["trace"]["inner_iters"] == gold["inner_iters"].tolist()
    assert _rel(res["trace"]["objective"], gold["objective"]) < 1e-10
    assert _rel(res["f"], gold["f"]) < 1e-10
    assert _rel(res["g"], gold["g"]) < 1e-10
    assert _rel(res["gamma"], gold["gamma"]) < 1e-10
    assert res["value"] == pytest.approx(float(gold["value"]), rel=1e-10)
    assert res["converged"] == bool(gold["converged"])
    assert res["constant"] == pytest.approx(float(gold["constant"]), rel=1e-12)
    cost = O.SqEuclid(res["xbar"], res["zbar"])
    idx, gap = O.plan_argmax(res["f"], res["g"], cost, b, res["eps_eff"])
    sure = gold["argmax_gap"] > 1e-9
    assert np.array_equal(idx[sure], gold["argmax"][sure])


def test_oracle_c5law_trajectory():
    gold = golden("c5law_solve")
    x, y, a, b = gold["x_feat"], gold["y_feat"], gold["a"], gold["b"]
    res = O.solve_cnt_gw(x, a, y, b, 0.02, dict(n_inner=200), max_outer=10, delta_outer=1e-300)
    # cold regime (Err ~ 1): fp64 summation-order differences grow ~1e-11 -> ~1e-8
    # over 2000 sweeps, so the oracle pin is 1e-7 here
    assert _rel(res["trace"]["objective"], gold["objective"]) < 1e-7
    assert _rel(res["f"], gold["f_steps"][-1]) < 1e-7


def test_oracle_closed_form_constant():
    """The device's O(N D^2) closed form equals the reference's O(N^2 D) sum."""
    gold = golden("c1_solve")
    for feat, w, key in ((gold["x_feat"], gold["a"], "fm_x"), (gold["y_feat"], gold["b"], "fm_y")):
        xc = feat - w @ feat
        nn = (xc * xc).sum(1)
        cov = xc.T @ (w[:, None] * xc)
        q = 2 * (w @ nn**2) + 2 * (w @ nn) ** 2 + 4 * (cov * cov).sum()
        assert q == pytest.approx(float(gold[key]), rel=1e-12)
        assert O.fourth_moment(feat, w) == pytest.approx(float(gold[key]), rel=1e-12)


class TestKnownAnswers:
    """Reference tests' known answers, restated against the oracle."""

    def test_single_point_splits_cost(self):
        res = O.sinkhorn(np.ones(1), np.ones(1), O.Dense([[1.7]]), 0.5, n_inner=80)
        assert res["f"][0] == pytest.approx(0.85, abs=1e-12)
        assert res["g"][0] == pytest.approx(0.85, abs=1e-12)

    def test_frozen_marginal_error(self):
        # all mass on one cell against uniform marginals: 1 + 1
        f = np.array([0.0, -1e9])
        g = np.array([0.0, -1e9])
        c = np.zeros((2, 2))
        err = O.marginal_error(f + np.log(2.0), g + np.log(2.0), O.Dense(c), np.full(2, .5),
                               np.full(2, .5), 1.0)
        assert err == pytest.approx(2.0)

    def test_product_plan_kl_zero(self):
        a, b = np.array([0.3, 0.7]), np.array([0.6, 0.4])
        assert O.kl(np.zeros(2), np.zeros(2), O.Dense(np.zeros((2, 2))), a, b, 1.0) == pytest.approx(
            0.0, abs=1e-15)

    def test_weighted_gap_cap(self):
        assert np.isfinite(O.weighted_gap(np.ones(2), np.array([1e6, 0]), np.zeros(2), 1e-3))


def test_oracle_plan_reductions_and_gradients():
    """Oracle restatement of divergence._plan_reductions / _grad_constant /
    feature_gradients against the reference's own outputs (golden 'gradients')."""
    gold = golden("gradients")
    x, y, a, b = gold["x_feat"], gold["y_feat"], gold["a"], gold["b"]
    cost = O.SqEuclid(O.augment(x), gold["zbar"])
    red = O.plan_reductions(gold["f"], gold["g"], cost, a, b, float(gold["eps_eff"]), x, y)
    for got, key in zip(red[:4], ("pi_y", "pi_sy", "pit_x", "pit_sx")):
        assert _rel(got, gold[key]) < 1e-10, key
    assert red[4] == pytest.approx(float(gold["sigma_ss"]), rel=1e-10)
    ty = float(b @ (y**2).sum(1))
    assert _rel(O.grad_constant(x, a, ty), gold["grad_const"]) < 1e-10
    gsrc, gtgt = O.feature_gradients(x, a, y, b, gold["gamma"], red)
    assert _rel(gsrc, gold["gsrc"]) < 1e-10
    assert _rel(gtgt, gold["gtgt"]) < 1e-10
