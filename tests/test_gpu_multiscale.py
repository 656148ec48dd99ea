"""GPU parity of the multiscale front end (reference solvers.py:668-763,
SURVEY.md §8(f) row 2) against the reference's own outputs
(tests/golden/multiscale.npz): the device weighted k-means reproduces the
reference's numpy k-means exactly (assignments, centres, masses — including
the empty-cluster path and D=64), and the two-stage solve matches at the
BASELINE tolerance."""

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


@pytest.mark.parametrize("case", ["c1", "dirichlet", "dupes", "d64", "bigclusters"])
def test_weighted_kmeans_is_the_references(P, case):
    from paper_2602_06658_b200 import solvers

    gold = golden("multiscale")
    x, w, k = gold[f"{case}__x"], gold[f"{case}__w"], int(gold[f"{case}__k"])
    assign, centers, cw = solvers._weighted_kmeans(x, w, k, np.random.default_rng(7))
    assert np.array_equal(assign, gold[f"{case}__assign"])
    assert np.array_equal(centers, gold[f"{case}__centers"])
    assert np.array_equal(cw, gold[f"{case}__cw"])


def test_solve_multiscale_matches_reference(P):
    gold = golden("multiscale")
    src = P.EmbeddedMeasure(gold["ms_x"], gold["ms_a"])
    tgt = P.EmbeddedMeasure(gold["ms_y"], gold["ms_b"])
    cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
    res = P.solve_multiscale(src, tgt, cfg, rho=0.1)
    assert res.coarse is not None
    assert res.coarse.value == pytest.approx(float(gold["ms_coarse_value"]), rel=TOL)
    assert _rel(res.coarse.gamma, gold["ms_coarse_gamma"]) < TOL
    assert res.value == pytest.approx(float(gold["ms_value"]), rel=TOL)
    assert _rel(res.gamma, gold["ms_gamma"]) < TOL
    assert _rel(res.coupling.f, gold["ms_f"]) < TOL
    assert _rel(res.coupling.g, gold["ms_g"]) < TOL
    for got, want in ((res.trace.inner_iters, gold["ms_inner"]),
                      (res.coarse.trace.inner_iters, gold["ms_coarse_inner"])):
        assert len(got) == len(want)
        assert np.abs(np.array(got) - want).max() <= 1
