"""GPU parity of the kernel-PCA embeddings (reference kernels.py:149-446,
SURVEY.md §8(f) row 3) against the reference's own outputs
(tests/golden/kpca.npz): every cost kind through the dense branch (N=300),
the matrix-free subspace branch (N=4500, costs streamed by
cntgw_cost_product), centred kernels, the CNT diagnostic, cost matrices and
cost gradients."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def K(cuda):
    from paper_2602_06658_b200 import kernels as K

    return K


@pytest.mark.parametrize("name", ["euclid", "pnorm", "exp", "sqlow", "embed", "matrix"])
def test_embedding_dense_branch(K, name):
    from paper_2602_06658_b200.measures import DiscreteMeasure

    gold = golden("kpca")
    meas = DiscreteMeasure(gold["pts"], gold["w"])
    specs = {
        "euclid": K.CostSpec("euclidean"),
        "pnorm": K.CostSpec("p_norm", p=1.5),
        "exp": K.CostSpec("exp_kernel", sigma=0.8),
        "sqlow": K.CostSpec("sq_euclidean"),
        "embed": K.CostSpec("precomputed_embedding", path="mem", payload=gold["emb6"]),
        "matrix": K.CostSpec("dense_matrix", path="mem",
                             payload=K.cost_matrix(K.CostSpec("euclidean"), meas)),
    }
    e = K.embed_measure(meas, specs[name], dim=int(gold[f"{name}__dim"]))
    assert _rel(e.eigenvalues, gold[f"{name}__vals"]) < 1e-10
    assert _rel(e.features, gold[f"{name}__f"]) < 1e-8
    assert e.explained_variance == pytest.approx(float(gold[f"{name}__ev"]), rel=1e-10)
    np.testing.assert_allclose(e.weights, gold["w"])


def test_embedding_streaming_subspace_branch(K):
    """N=4500 > the dense cutoff: matrix-free products with the streamed cost."""
    from paper_2602_06658_b200.measures import DiscreteMeasure

    gold = golden("kpca")
    n = gold["big"].shape[0]
    e = K.embed_measure(DiscreteMeasure(gold["big"], np.full(n, 1.0 / n)), K.CostSpec("euclidean"), dim=3)
    assert _rel(e.eigenvalues, gold["big__vals"]) < 1e-7
    assert _rel(e.features, gold["big__f"]) < 1e-5
    assert e.explained_variance == pytest.approx(float(gold["big__ev"]), rel=1e-7)


def test_kernels_diagnostics_costs_gradients(K):
    gold = golden("kpca")
    ws = np.full(40, 1.0 / 40)
    kern = K.kernel_from_cost(gold["c40"], ws, base_index=3)
    assert _rel(kern.matrix, gold["k40"]) < 1e-12
    d = K.cnt_diagnostic(gold["c40"], ws)
    assert d.is_cnt and d.max_abs_eigenvalue == pytest.approx(gold["diag"][1], rel=1e-10)
    d2 = K.cnt_diagnostic(gold["rnd"], ws)
    assert not d2.is_cnt
    assert d2.min_eigenvalue == pytest.approx(gold["diag2"][0], rel=1e-10)
    from paper_2602_06658_b200.measures import DiscreteMeasure

    small = gold["pts"][:40]
    assert _rel(K.cost_matrix(K.CostSpec("exp_kernel", sigma=0.8), DiscreteMeasure(small, ws)),
                gold["cexp"]) < 1e-12
    assert _rel(K.cost_gradients(K.CostSpec("exp_kernel", sigma=0.8), small[:20]), gold["gexp"]) < 1e-12
    assert _rel(K.cost_gradients(K.CostSpec("p_norm", p=1.5), small[:20]), gold["gpn"]) < 1e-12
    with pytest.raises(ValueError, match="not differentiable"):
        K.cost_gradients(K.CostSpec("euclidean"), small)


def test_streamed_cost_product_matches_dense(K):
    """cntgw_cost_product against the dense product for every point kind."""
    import torch

    from paper_2602_06658_b200._native import call

    rng = np.random.default_rng(3)
    x = rng.standard_normal((777, 4))
    v = rng.standard_normal((777, 16))
    dev = torch.device("cuda", 0)
    xt = torch.as_tensor(x, device=dev)
    sqn = (xt * xt).sum(1).contiguous()
    vt = torch.as_tensor(v, device=dev)
    from paper_2602_06658_b200.measures import DiscreteMeasure

    for kind, spec, par in ((0, K.CostSpec("sq_euclidean"), 0.0), (1, K.CostSpec("euclidean"), 0.0),
                            (2, K.CostSpec("p_norm", p=1.3), 1.3),
                            (3, K.CostSpec("exp_kernel", sigma=0.7), 0.7)):
        out = torch.empty_like(vt)
        call("cntgw_cost_product", kind, par, xt.data_ptr(), 777, 4, sqn.data_ptr(), vt.data_ptr(), 16,
             out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        c = K.cost_matrix(spec, DiscreteMeasure(x, np.full(777, 1 / 777)))
        assert _rel(out.cpu().numpy(), c @ v) < 1e-12, kind
