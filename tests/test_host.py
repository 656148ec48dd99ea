"""Host-side logic of the drop-in API (config validation, boundary types,
trace, embedding fast path, synthetic generators) — CPU only, mirroring the
reference's own config/measure tests (tests/test_sinkhorn.py:74-89,
tests/test_measures.py, tests/test_kernels.py:198-247)."""

import numpy as np
import pytest

import paper_2602_06658_b200 as P
from paper_2602_06658_b200 import configs


class TestSinkhornConfig:
    def test_requires_one_budget(self):
        with pytest.raises(ValueError, match="exactly one"):
            P.SinkhornConfig(eps=1.0, n_inner=10, threshold=1e-6)

    def test_default_budget_is_fixed_sweeps(self):
        cfg = P.SinkhornConfig(eps=1.0)
        assert cfg.n_inner == 100 and cfg.threshold is None

    @pytest.mark.parametrize("eps", [0.0, -1.0, float("inf"), float("nan")])
    def test_rejects_bad_eps(self, eps):
        with pytest.raises(ValueError, match="eps"):
            P.SinkhornConfig(eps=eps)

    def test_rejects_bad_mode(self):
        with pytest.raises(ValueError, match="mode"):
            P.SinkhornConfig(eps=1.0, mode="fast")

    def test_rejects_bad_budgets(self):
        with pytest.raises(ValueError, match="n_inner"):
            P.SinkhornConfig(eps=1.0, n_inner=0)
        with pytest.raises(ValueError, match="threshold"):
            P.SinkhornConfig(eps=1.0, threshold=-1.0)
        with pytest.raises(ValueError, match="max_inner"):
            P.SinkhornConfig(eps=1.0, threshold=1e-3, max_inner=0)
        with pytest.raises(ValueError, match="anneal_from"):
            P.SinkhornConfig(eps=1.0, anneal_from=0.0)

    def test_with_helpers(self):
        cfg = P.SinkhornConfig(eps=1.0).with_temperature(0.5).with_warm_start([1], [2])
        assert cfg.eps == 0.5 and cfg.warm_start == ([1], [2])
        lc = cfg.loop_config()
        assert lc.max_sweeps == 100 and lc.mode == "symmetrized"
        lc2 = P.SinkhornConfig(eps=1.0, threshold=1e-3, max_inner=7).loop_config()
        assert lc2.max_sweeps == 7


class TestEgwConfig:
    def test_make_config_bundles_inner(self):
        cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
        assert cfg.inner.threshold == 1e-5 and cfg.inner.max_inner == 200 and cfg.max_outer == 20

    @pytest.mark.parametrize("kw,msg", [
        (dict(max_outer=0), "max_outer"), (dict(delta_outer=0.0), "delta_outer"),
        (dict(init="bogus"), "init"), (dict(init="gamma"), "init_gamma"),
        (dict(init="coupling"), "init_coupling"), (dict(init="landmarks"), "init_pairs"),
        (dict(final_anneal=0.0), "final_anneal"), (dict(feasibility_tol=0.0), "feasibility_tol"),
    ])
    def test_validation(self, kw, msg):
        with pytest.raises(ValueError, match=msg):
            P.make_config(0.1, **kw)


class TestMeasures:
    def test_discrete_measure_validation(self):
        with pytest.raises(ValueError, match="non-finite"):
            P.DiscreteMeasure([[np.nan, 0.0]])
        with pytest.raises(ValueError, match="strictly positive"):
            P.DiscreteMeasure([[0.0], [1.0]], [1.0, 0.0])
        with pytest.raises(ValueError, match="sum to 1"):
            P.DiscreteMeasure([[0.0], [1.0]], [0.5, 0.6])
        m = P.DiscreteMeasure(np.zeros((4, 2)))
        assert np.allclose(m.weights, 0.25) and not m.points.flags.writeable

    def test_dense_coupling_frozen_examples(self):
        c = P.DenseCoupling(np.array([[1.0, 0.0], [0.0, 0.0]]), np.full(2, 0.5), np.full(2, 0.5))
        assert P.marginal_error(c) == pytest.approx(2.0)
        d = P.DenseCoupling(np.diag([0.5, 0.5]), np.full(2, 0.5), np.full(2, 0.5))
        assert P.kl_divergence(d) == pytest.approx(np.log(2.0))
        a, b = np.array([0.3, 0.7]), np.array([0.6, 0.4])
        assert P.kl_divergence(P.DenseCoupling(np.outer(a, b), a, b)) == pytest.approx(0, abs=1e-15)
        with pytest.raises(ValueError, match="mass"):
            P.DenseCoupling(np.full((2, 2), 0.5), np.full(2, 0.5), np.full(2, 0.5))

    def test_implicit_coupling_validation(self):
        """Construction-time validation (measures.py:160-179); the plan's
        arithmetic (densify, marginals, KL) runs on the GPU and is covered by
        tests/test_gpu_api.py."""
        rng = np.random.default_rng(3)
        a = np.full(7, 1 / 7)
        b = np.full(5, 1 / 5)
        cost = P.DenseCost(rng.random((7, 5)))
        f, g = rng.standard_normal(7) * 0.1, rng.standard_normal(5) * 0.1
        with pytest.raises(ValueError, match="non-finite"):
            P.ImplicitCoupling([np.inf] * 7, g, cost, a, b, 0.5)
        with pytest.raises(ValueError, match="eps_eff"):
            P.ImplicitCoupling(f, g, cost, a, b, 0.0)
        with pytest.raises(ValueError, match="potential shapes"):
            P.ImplicitCoupling(f[:6], g, cost, a, b, 0.5)

    def test_dense_cost_provider(self):
        c = np.arange(12.0).reshape(3, 4)
        p = P.DenseCost(c)
        assert np.array_equal(p.rows(1, 3), c[1:3])
        assert np.array_equal(p.transpose().full(), c.T) and p.transpose().transpose() is p
        with pytest.raises(ValueError, match="non-finite"):
            P.DenseCost(np.array([[np.inf]]))

    def test_sinkhorn_rejects_bad_shapes_before_touching_the_gpu(self):
        cost = P.DenseCost(np.ones((3, 2)))
        with pytest.raises(ValueError, match="weight shapes"):
            P.sinkhorn(np.ones(2) / 2, np.ones(2) / 2, cost, P.SinkhornConfig(eps=1.0))
        cfg = P.SinkhornConfig(eps=1.0).with_warm_start(np.zeros(2), np.zeros(2))
        with pytest.raises(ValueError, match="warm-start"):
            P.sinkhorn(np.ones(3) / 3, np.ones(2) / 2, cost, cfg)


class TestEmbedding:
    def test_fast_path_centres_and_half_norms(self):
        rng = np.random.default_rng(0)
        pts = rng.standard_normal((50, 3))
        w = rng.random(50)
        w /= w.sum()
        emb = P.embed_measure(P.DiscreteMeasure(pts, w), P.CostSpec("sq_euclidean"), dim=3)
        assert np.allclose(emb.features, pts - w @ pts)
        assert np.allclose(emb.half_sq_norms, 0.5 * (emb.features**2).sum(1))
        assert np.allclose(emb.augmented()[:, -1], emb.half_sq_norms)
        assert emb.trace_second_moment() == pytest.approx(float(np.trace(emb.covariance())))

    def test_kernel_pca_runs_on_the_device_only(self):
        """Kernel-PCA embeddings have no CPU fallback (the CPU suite has no GPU)."""
        m = P.DiscreteMeasure(np.random.default_rng(0).standard_normal((10, 5)))
        with pytest.raises(RuntimeError, match="CUDA device"):
            P.embed_measure(m, P.CostSpec("sq_euclidean"), dim=2)
        with pytest.raises(ValueError, match="exceeds support size"):
            P.embed_measure(m, P.CostSpec("euclidean"), dim=11)

    def test_cost_spec_grammar_and_validation(self):
        from paper_2602_06658_b200 import kernels as K

        assert K.parse_cost_spec("p_norm:1.5").p == 1.5
        assert K.parse_cost_spec("exp:0.3").sigma == 0.3
        assert K.parse_cost_spec(" euclidean ").kind == "euclidean"
        assert K.CostSpec("p_norm", p=1.5).differentiable and not K.CostSpec("euclidean").differentiable
        assert K.CostSpec("exp_kernel", sigma=2.0).describe() == "exp:2"
        for bad in ("p_norm:x", "exp:", "cosine", "foo:1"):
            with pytest.raises(ValueError):
                K.parse_cost_spec(bad)
        with pytest.raises(ValueError, match="exponent"):
            K.CostSpec("p_norm", p=2.5)
        with pytest.raises(ValueError, match="radius"):
            K.CostSpec("exp_kernel", sigma=0.0)
        with pytest.raises(ValueError, match="payload"):
            K.CostSpec("dense_matrix")

    def test_matrix_payload_checks(self, tmp_path):
        from paper_2602_06658_b200 import kernels as K

        good = tmp_path / "c.csv"
        good.write_text("0,1,2\n1,0,1\n2,1,0\n")
        assert K.parse_cost_spec(f"matrix:{good}").payload.shape == (3, 3)
        bad = tmp_path / "b.csv"
        bad.write_text("0,1\n2,0\n")
        with pytest.raises(ValueError, match="symmetric"):
            K.load_matrix_payload(bad)


def test_solve_trace_csv(tmp_path):
    tr = P.SolveTrace()
    tr.append(1, 0.5, 0.1, 1e-3, 7, 0.01)
    tr.append(2, 0.25, 0.05, 1e-4, 3, 0.02)
    path = tmp_path / "t.csv"
    tr.to_csv(path, header="run")
    lines = path.read_text().splitlines()
    assert lines[0] == "# run"
    assert lines[1] == "step,objective,gamma_delta,marginal_err,inner_iters,elapsed_s"
    assert lines[2].startswith("1,0.5,0.10000000000000001,") and len(tr) == 2


class TestGenerators:
    def test_c1_law(self):
        pc = configs.c1(seed=0, n=200)
        for p in (pc.x, pc.y):
            sq = (p**2).sum(1)
            d2 = sq[:, None] + sq[None, :] - 2 * p @ p.T
            assert d2.max() == pytest.approx(1.0, rel=1e-5)
            assert np.array_equal(p, p.astype(np.float32).astype(np.float64))

    def test_deterministic(self):
        a, b = configs.c4(seed=3, n=500), configs.c4(seed=3, n=500)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)

    def test_c5_weights_sum_to_one(self):
        pc = configs.c5(seed=0, n=1024)
        assert pc.x.shape == (1024, 64) and pc.y.shape == (1024, 32)
        assert abs(pc.a.sum() - 1) < 1e-12 and (pc.a > 0).all()
        P.DiscreteMeasure(pc.x, pc.a)

    def test_c2_shapes(self):
        inst = configs.c2(seed=0, n=4096, k=16)
        assert inst.u.shape == (4096, 16) and inst.u.dtype == np.float32
        assert inst.u.std() == pytest.approx(0.25, rel=0.05)


def test_coarsen_validation():
    """coarsen rejects rho outside (0, 1) and fewer than 2 clusters before
    touching the device (reference solvers.py:714-721)."""
    import pytest as _pt

    from paper_2602_06658_b200 import EmbeddedMeasure, coarsen

    m = EmbeddedMeasure(np.zeros((10, 2)), np.full(10, 0.1))
    rng = np.random.default_rng(0)
    with _pt.raises(ValueError, match="rho must lie"):
        coarsen(m, 1.0, rng)
    with _pt.raises(ValueError, match="need at least 2"):
        coarsen(m, 0.05, rng)
