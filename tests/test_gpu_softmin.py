"""GPU parity of the streaming half-update kernel (K1/K2) against the oracle.

Covers every supported feature width, the squared-difference coordinate,
ragged and degenerate shapes (1 row, 1 column, sizes off the 256-column tile
and the 128*R-row CTA tile), split-column planning, determinism, the lazy
rebase path under huge exponents, and the full-size C2 (N=M=2^20, K=16)
half-updates on row/column subsamples against the reference's own values.
Tolerance: |out - oracle|_inf <= 1e-4 * |oracle|_inf (BASELINE north_star),
tighter where noted."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def env(cuda):
    import torch

    import importlib

    import paper_2602_06658_b200 as P
    from paper_2602_06658_b200 import engine
    from oracle import cntgw_oracle as O

    S = importlib.import_module("paper_2602_06658_b200.sinkhorn")

    return P, engine, S, O, torch, cuda


def _half_update(env, cost, a, b, g, eps, prec=None):
    """GPU f-update S(g) through the device problem of ``cost`` (reference form)."""
    P, engine, S, O, torch, dev = env
    prob = S.device_problem(cost, a, b, dev)
    if prec is not None:
        prob.fwd.prec = prec
    st = engine.SweepState(dev)
    st.init(eps)
    gt = engine.to_dev64(np.asarray(g) - prob.col_sep, dev)
    out = torch.empty(len(a), dtype=torch.float64, device=dev)
    prob.fwd(st, gt, out, skip=False)
    return out.cpu().numpy() + prob.row_sep


# "f32c" runs the centred path's FFMA2 kernel (the default); "f32c_tc" its
# opt-in tcgen05 kernel where kd + sq <= 4 (CNTGW_CTR_TC=1)
PRECS = {"f32": 0, "f64": 1, "f32c": 3, "f32c_tc": 3, "f64s": 4}


def _prec(name, monkeypatch):
    monkeypatch.setenv("CNTGW_CTR_TC", "1" if name == "f32c_tc" else "0")
    return PRECS[name]


@pytest.mark.parametrize("pname", list(PRECS))
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8, 16, 17, 33, 64, 65])
@pytest.mark.parametrize("n,m", [(1, 1), (1, 300), (300, 1), (129, 257), (1000, 1000), (2049, 771)])
def test_sq_euclidean_half_update(env, k, n, m, pname, monkeypatch):
    P, engine, S, O, torch, dev = env
    prec = _prec(pname, monkeypatch)
    if prec == 3 and not engine.ctr_supported(engine.padded_kd(max(k - 1, 1)), True):
        pytest.skip("centred fp32 path: kd + sq <= 8")
    rng = np.random.default_rng(k * 1000 + n + m)
    x = rng.standard_normal((n, k)) * 0.5
    z = rng.standard_normal((m, k)) * 0.5
    a = rng.random(n) + 0.2
    a /= a.sum()
    b = rng.random(m) + 0.2
    b /= b.sum()
    g = rng.standard_normal(m) * 0.1 + (z * z).sum(1)
    eps = 0.05
    got = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, prec)
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    assert _rel(got, want) < (5e-7 if prec in (1, 4) else 1e-5)


@pytest.mark.parametrize("k", [4, 16])
def test_low_rank_half_update(env, k):
    P, engine, S, O, torch, dev = env
    inst = __import__("paper_2602_06658_b200.configs", fromlist=["c2"]).c2(seed=5, n=3000, m=2500, k=k)
    n, m = inst.u.shape[0], inst.v.shape[0]
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    cost = P.SeparableLowRankCost(inst.u, inst.v, inst.row_sep, inst.col_sep)
    got = _half_update(env, cost, a, b, inst.g, inst.eps)
    want = O.softmin(O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep), np.log(b),
                     inst.g.astype(float), inst.eps)
    assert _rel(got, want) < 1e-5


@pytest.mark.parametrize("pname", list(PRECS))
def test_rebase_path_under_huge_exponents(env, pname, monkeypatch):
    """Cold regime: |exponent| ~ 1e6 log2 units; exercises lazy rebasing."""
    P, engine, S, O, torch, dev = env
    prec = _prec(pname, monkeypatch)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((700, 4)) * 6.0
    z = rng.standard_normal((900, 4)) * 6.0
    a, b = np.full(700, 1 / 700), np.full(900, 1 / 900)
    g = rng.standard_normal(900) * 30.0 + (z * z).sum(1)
    eps = 1.25e-3
    got = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, prec)
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    assert _rel(got, want) < (5e-7 if prec in (1, 4) else 1e-5)


@pytest.mark.parametrize("tc", ["1", "0"], ids=["tcgen05", "ffma"])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("n,m", [(5000, 7000), (130, 100_000)])
def test_centred_path_cold_locality(env, k, n, m, tc, monkeypatch):
    """CNTGW_F32C on a cold clustered law (|exponent| ~ 1e5-1e6 log2 units,
    where plain fp32 loses ~0.1 log2 units per term): fp32 pair terms on
    Morton-ordered centred tiles match the fp64 oracle; outputs come back in
    the caller's (unsorted) order."""
    P, engine, S, O, torch, dev = env
    monkeypatch.setenv("CNTGW_CTR_TC", tc)
    rng = np.random.default_rng(10 * k + n % 7)
    cx = rng.standard_normal((8, k)) * 2.0
    x = cx[rng.integers(0, 8, n)] + rng.standard_normal((n, k)) * 0.7
    rot = np.linalg.qr(rng.standard_normal((k, k)))[0]
    z = cx[rng.integers(0, 8, m)] @ rot + rng.standard_normal((m, k)) * 0.7
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    g = rng.standard_normal(m) * 3.0 + (z * z).sum(1)
    eps = 1.25e-3
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    got = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, 3)
    plain = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, 0)
    lam = np.log2(np.e) / eps  # per-row errors in log2 units of the plan entries
    e_c, e_p = np.abs(got - want) * lam, np.abs(plain - want) * lam
    print(f"k={k} n={n} m={m}: rel f32c {_rel(got, want):.2e} f32 {_rel(plain, want):.2e}; "
          f"p99 log2 err f32c {np.percentile(e_c, 99):.2e} f32 {np.percentile(e_p, 99):.2e}")
    assert _rel(got, want) < 1e-5
    if n >= 5000:  # local row groups (130 rows are one group spanning the cloud)
        assert np.percentile(e_c, 99) < 0.75 * np.percentile(e_p, 99)


# the centred kernel's opt-in variants (csrc/cntgw_b200.cu pick_ctr): row
# groups per CTA (CNTGW_CTR_R), lazy-rebase group width (CNTGW_CTR_G) and the
# FMA-pipe exp2 share (CNTGW_CTR_POLY); "default" is R=4, G=4, no polynomial
CTR_VARIANTS = {"default": {}, "r2": {"CNTGW_CTR_R": "2"}, "r8": {"CNTGW_CTR_R": "8"},
                "g8": {"CNTGW_CTR_G": "8"}, "poly": {"CNTGW_CTR_POLY": "1"}}


@pytest.mark.parametrize("variant", list(CTR_VARIANTS))
def test_centred_block_sparse_skip(env, variant, monkeypatch):
    """The centred kernel's block-sparse plan (tiles that cannot hold a term
    within 2^-64 of a row's maximum are skipped) on a cold clustered law large
    enough for most tiles to be skipped: equal to the dense sweep to 1e-9 and
    to the fp64 oracle on sampled rows — for every shipped kernel variant."""
    P, engine, S, O, torch, dev = env
    for key, val in CTR_VARIANTS[variant].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(11)
    n = m = 1 << 16
    cx = rng.standard_normal((8, 3)) * 2.0
    x = cx[rng.integers(0, 8, n)] + rng.standard_normal((n, 3)) * 0.7
    z = cx[rng.integers(0, 8, m)] + rng.standard_normal((m, 3)) * 0.7
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    g = rng.standard_normal(m) * 0.1 + (z * z).sum(1)
    eps = 1.25e-3
    cost = P.SquaredEuclideanCost(x, z)
    monkeypatch.setenv("CNTGW_CTR_SKIP", "1")
    sparse = _half_update(env, cost, a, b, g, eps, 3)
    monkeypatch.setenv("CNTGW_CTR_SKIP", "0")
    dense = _half_update(env, cost, a, b, g, eps, 3)
    assert _rel(sparse, dense) < 1e-9
    rows = rng.choice(n, 512, replace=False)
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps, row_idx=rows)
    assert _rel(sparse[rows], want) < 1e-5


@pytest.mark.parametrize("pname", list(PRECS))
def test_zero_weight_region(env, pname, monkeypatch):
    """Zero column weights (the reference's sinkhorn accepts them: log 0 =
    -inf terms) on a whole spatial region, so that entire Morton tiles (and
    column groups of the other kernels) carry no mass: zero weight, not NaN."""
    P, engine, S, O, torch, dev = env
    prec = _prec(pname, monkeypatch)
    rng = np.random.default_rng(5)
    n, m = 2000, 6000
    x = rng.standard_normal((n, 3)) * 2.0
    z = rng.standard_normal((m, 3)) * 2.0
    a = np.full(n, 1 / n)
    b = np.where(z[:, 0] > 0.5, 0.0, 1.0)
    b /= b.sum()
    g = rng.standard_normal(m) + (z * z).sum(1)
    eps = 2.5e-3
    with np.errstate(divide="ignore"):
        want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    got = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, prec)
    assert np.all(np.isfinite(got))
    assert _rel(got, want) < 1e-5


@pytest.mark.parametrize("tc", ["1", "0"], ids=["tcgen05", "ffma"])
@pytest.mark.parametrize("limit", ["0", "2000"])
def test_centred_path_fp64_tile_fallback(env, limit, tc, monkeypatch):
    """Tile pairs whose fp32 pair-term bound exceeds CNTGW_CTR_TILE_LIMIT are
    taken in fp64 inside the kernel: with limit 0 every pair is (fp64-exact,
    the fp64 path's tolerance), with a mid limit the two kinds mix."""
    P, engine, S, O, torch, dev = env
    rng = np.random.default_rng(3)
    n, m, k = 3000, 2600, 3
    x = rng.standard_normal((n, k)) * 2.5
    z = rng.standard_normal((m, k)) * 2.5
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    g = rng.standard_normal(m) * 3.0 + (z * z).sum(1)
    eps = 1.25e-3
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    monkeypatch.setenv("CNTGW_CTR_TC", tc)
    monkeypatch.setenv("CNTGW_CTR_TILE_LIMIT", limit)
    got = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, 3)
    assert _rel(got, want) < (5e-7 if limit == "0" else 1e-5)


@pytest.mark.parametrize("k", [1, 3, 4, 8, 16, 33, 64])
def test_dmma_path_matches_dfma_path_cold(env, k, monkeypatch):
    """fp64 half-update: the DMMA (m8n8k4 f64) kernel and the DFMA
    kernel agree with the oracle and with each other in the cold regime
    (exponents ~1e5 log2 units, lazy rebases), including ragged shapes."""
    P, engine, S, O, torch, dev = env
    rng = np.random.default_rng(k)
    n, m = 531, 777
    x = rng.standard_normal((n, k)) * 1.5
    z = rng.standard_normal((m, k)) * 1.5
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    g = rng.standard_normal(m) * 30.0 + (z * z).sum(1)
    eps = 2.5e-3
    want = O.softmin(O.SqEuclid(x, z), np.log(b), g, eps)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CNTGW_F64_DMMA", flag)
        outs.append(_half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, eps, 1))
        assert _rel(outs[-1], want) < 5e-7, flag
    assert _rel(outs[0], outs[1]) < 1e-9


def test_deterministic_reruns(env):
    P, engine, S, O, torch, dev = env
    rng = np.random.default_rng(1)
    x, z = rng.standard_normal((5000, 3)), rng.standard_normal((7000, 3))
    a, b = np.full(5000, 1 / 5000), np.full(7000, 1 / 7000)
    g = rng.standard_normal(7000)
    r1 = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, 0.02)
    r2 = _half_update(env, P.SquaredEuclideanCost(x, z), a, b, g, 0.02)
    assert np.array_equal(r1, r2)


@pytest.fixture(scope="module")
def c2_full(env):
    """The full-size C2 instance (N=M=2^20, K=16), one GPU rep (f then g)."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200 import configs

    inst = configs.c2(seed=0)
    n = inst.u.shape[0]
    w = np.full(n, 1.0 / n)
    cost = P.SeparableLowRankCost(inst.u, inst.v, inst.row_sep, inst.col_sep)
    cfg = P.SinkhornConfig(eps=inst.eps, mode="standard", n_inner=1).with_warm_start(
        np.zeros(n), inst.g.astype(np.float64))
    res = P.sinkhorn(w, w, cost, cfg)
    return inst, res


def test_c2_full_size_f_update_matches_reference(env, c2_full):
    """Rows sampled at full M; reference values from the reference's _softmin."""
    inst, res = c2_full
    gold = golden("c2_subsample")
    assert int(gold["n"]) == inst.u.shape[0]
    rows = gold["rows"]
    assert _rel(res.coupling.f[rows], gold["f_rows"]) < 1e-5


def test_c2_full_size_g_update_given_gpu_f(env, c2_full):
    """g-update on a column subsample at full N, given the GPU's own f."""
    P, engine, S, O, torch, dev = env
    inst, res = c2_full
    n = inst.u.shape[0]
    cols = np.sort(np.random.default_rng(7).choice(n, size=32, replace=False))
    cost_t = O.LowRank(inst.v, inst.u, inst.col_sep, inst.row_sep)
    want = O.softmin(cost_t, np.full(n, -np.log(n)), res.coupling.f, inst.eps, row_idx=cols)
    assert _rel(res.coupling.g[cols], want) < 1e-5


@pytest.mark.parametrize("prec,kind", [(0, None), (2, "f16"), (2, "tf32")], ids=["f32", "tc-f16", "tc-tf32"])
@pytest.mark.parametrize("k", [8, 16])
@pytest.mark.parametrize("n,m", [(1, 1), (129, 257), (1000, 1000), (2049, 771), (300, 5000)])
def test_low_rank_paths(env, prec, kind, k, n, m, monkeypatch):
    """fp32 FFMA2 and tcgen05 split-precision half-updates (fp16 operands, the
    default, and tf32 operands) on the C2 cost form."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200 import configs

    if kind:
        monkeypatch.setenv("CNTGW_TC_KIND", kind)

    inst = configs.c2(seed=n + m + k, n=n, m=m, k=k)
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    cost = P.SeparableLowRankCost(inst.u, inst.v, inst.row_sep, inst.col_sep)
    got = _half_update(env, cost, a, b, inst.g.astype(float) + inst.col_sep, inst.eps, prec)
    want = O.softmin(O.LowRank(inst.u, inst.v, inst.row_sep, inst.col_sep), np.log(b),
                     inst.g.astype(float) + inst.col_sep, inst.eps)
    assert _rel(got, want) < 1e-5


@pytest.mark.parametrize("k", [8, 16])
@pytest.mark.parametrize("shift", [0, 30, -30])
@pytest.mark.parametrize("poly", ["0", "3", "6"])
def test_tc_fp16_operand_ranges(env, k, shift, poly, monkeypatch):
    """The fp16-operand tcgen05 split scales both sides into fp16's exponent
    range from the absmax of the column features: the same scores with the
    features scaled by 2^s / 2^-s, features 2^-20 / 2^-25 below the side's
    largest (values below fp16's normal range after scaling), zero-weight columns
    (log2 w = -inf) and a large bias all match the oracle; every split of the
    exponentials between MUFU and the FMA pipe."""
    P, engine, S, O, torch, dev = env
    monkeypatch.setenv("CNTGW_TC_KIND", "f16")
    monkeypatch.setenv("CNTGW_TC_POLY", poly)
    rng = np.random.default_rng(100 + k + shift)
    n, m = 700, 1500
    u = (rng.standard_normal((n, k)) * 0.25 * 2.0 ** shift).astype(np.float32)
    v = (rng.standard_normal((m, k)) * 0.25 * 2.0 ** -shift).astype(np.float32)
    v[:, k // 2:] *= np.float32(2.0 ** -20)  # half of the products vanish against the rest
    u[:, :k // 4] *= np.float32(2.0 ** -25)
    a = np.full(n, 1 / n)
    b = np.where(np.arange(m) % 7 == 3, 0.0, 1.0)
    b /= b.sum()
    g = rng.standard_normal(m) * 40.0  # |bias| ~ 1e3 log2 units at eps = 0.05
    zero_n, zero_m = np.zeros(n), np.zeros(m)
    cost = P.SeparableLowRankCost(u, v, zero_n, zero_m)
    with np.errstate(divide="ignore"):
        want = O.softmin(O.LowRank(u, v, zero_n, zero_m), np.log(b), g, 0.05)
    got = _half_update(env, cost, a, b, g, 0.05, 2)
    assert np.all(np.isfinite(got))
    assert _rel(got, want) < 1e-5


@pytest.mark.parametrize("anneal", [None, 0.05], ids=["fixed", "annealed"])
def test_centred_plan_reuse_across_sweeps(env, anneal, monkeypatch):
    """A Sinkhorn loop on the centred path reuses its block-sparse plan across
    sweeps while no column record moved by more than the plan's margin: the
    potentials equal those of replanning every half-update (to 1e-9) and of
    the dense sweep. With sqrt annealing (anneal_from) lam changes every
    sweep, which rescales the whole record: the plan key forces a replan."""
    P, engine, S, O, torch, dev = env
    rng = np.random.default_rng(21)
    n = m = 1 << 15
    cx = rng.standard_normal((8, 3)) * 2.0
    x = cx[rng.integers(0, 8, n)] + rng.standard_normal((n, 3)) * 0.7
    z = cx[rng.integers(0, 8, m)] + rng.standard_normal((m, 3)) * 0.7
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    monkeypatch.setenv("CNTGW_PRECISION", "f32c")
    cfg = P.SinkhornConfig(eps=2e-3, n_inner=30, anneal_from=anneal)
    out = {}
    for tag, env_vars in (("reuse", {}), ("replan", {"CNTGW_CTR_REUSE": "0"}),
                          ("dense", {"CNTGW_CTR_SKIP": "0"})):
        for key in ("CNTGW_CTR_REUSE", "CNTGW_CTR_SKIP"):
            monkeypatch.delenv(key, raising=False)
        for key, val in env_vars.items():
            monkeypatch.setenv(key, val)
        res = P.sinkhorn(a, b, P.SquaredEuclideanCost(x, z), cfg)
        out[tag] = (res.coupling.f, res.coupling.g)
    for tag in ("replan", "dense"):
        assert _rel(out["reuse"][0], out[tag][0]) < 1e-9, tag
        assert _rel(out["reuse"][1], out[tag][1]) < 1e-9, tag


@pytest.mark.parametrize("anneal", [None, 0.05], ids=["fixed", "annealed"])
@pytest.mark.parametrize("k", [3, 32])
def test_f64s_measured_plan_matches_dense_loop(env, k, anneal, monkeypatch):
    """CNTGW_F64S: fp64 DMMA sweeps on cluster-ordered rows/columns that skip
    the (row group, stage) pairs a measured plan found below 2^-80 of every
    row's maximum. A whole Sinkhorn loop (plan reused across sweeps, replanned
    when a column record drifts or lam changes under annealing) equals the
    dense fp64 loop; outputs come back in the caller's order."""
    P, engine, S, O, torch, dev = env
    rng = np.random.default_rng(31 + k)
    n, m = 1 << 14, 3 << 12
    cx = rng.standard_normal((16, k)) * 2.0
    x = cx[rng.integers(0, 16, n)] + rng.standard_normal((n, k)) * 0.5
    z = cx[rng.integers(0, 16, m)] @ np.linalg.qr(rng.standard_normal((k, k)))[0] \
        + rng.standard_normal((m, k)) * 0.5
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    cost = P.SquaredEuclideanCost(x, z)
    cfg = P.SinkhornConfig(eps=2.5e-3, n_inner=30, anneal_from=anneal)
    out = {}
    for prec in ("f64s", "f64"):
        monkeypatch.setenv("CNTGW_PRECISION", prec)
        res = P.sinkhorn(a, b, cost, cfg)
        out[prec] = (res.coupling.f, res.coupling.g)
    # (the two paths visit columns in different orders, and both sum
    # 2^(fp64 offset truncated to fp32) per term: ~1e-9 relative apart)
    assert _rel(out["f64s"][0], out["f64"][0]) < 5e-8
    assert _rel(out["f64s"][1], out["f64"][1]) < 5e-8
    rows = np.sort(rng.choice(n, 64, replace=False))
    want = O.softmin(O.SqEuclid(x, z), np.log(b), out["f64s"][1], res.coupling.eps_eff, row_idx=rows)
    got = _half_update(env, cost, a, b, out["f64s"][1], res.coupling.eps_eff, 4)
    assert _rel(got[rows], want) < 5e-7


@pytest.mark.parametrize("anneal", [None, 0.05], ids=["fixed", "annealed"])
def test_f64s_hoisted_loop_equals_per_call_packing(env, anneal):
    """A driver that owns a loop gathers the F64S rows block once and lets
    pack() rewrite only the bias column after the first sweep
    (cntgw_update_cols_f64s; every sweep packs everything when lam is
    annealed): bit-identical to gathering and packing on every half-update."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200._native import F64S

    rng = np.random.default_rng(17)
    n, m, k = 1800, 2600, 8
    src = engine.Side.make(rng.standard_normal((n, k)) * 0.6, rng.random(n) * 4.0, np.full(n, 1 / n), dev, k)
    tgt = engine.Side.make(rng.standard_normal((m, k)) * 0.6, rng.random(m) * 4.0, np.full(m, 1 / m), dev, k)
    pots = [engine.to_dev64(rng.standard_normal(m) * (2.0 + s), dev) for s in range(4)]
    outs = {}
    for hoist in (False, True):
        op = engine.HalfUpdate(src, tgt, True)
        op.prec = F64S
        st = engine.SweepState(dev)
        st.init(2.5e-3, anneal, None, 8, "symmetrized")
        if hoist:
            op.hoist_rows()
        res = []
        for pot in pots:
            st.begin()
            out = torch.empty(n, dtype=torch.float64, device=dev)
            op(st, pot, out, skip=False)
            res.append(out.cpu().numpy())
        outs[hoist] = res
    for a_, b_ in zip(outs[False], outs[True]):
        assert np.array_equal(a_, b_)


def test_f64s_probe_stands_down_on_extreme_scales(env):
    """Row features of magnitude 1e-37 would need a power-of-two scale beyond
    fp32's normal range in the tcgen05 probe: it stands down and the sweep
    measures in fp64 instead, with the dense path's results."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200._native import F64, F64S

    rng = np.random.default_rng(5)
    n, m, k = 900, 1300, 3
    src = engine.Side.make(rng.standard_normal((n, k)) * 1e-37, rng.random(n) * 1e-37, np.full(n, 1 / n), dev, k)
    tgt = engine.Side.make(rng.standard_normal((m, k)), rng.random(m) * 3.0, np.full(m, 1 / m), dev, k)
    pot = engine.to_dev64(rng.standard_normal(m) * 5.0, dev)
    outs = {}
    for name, prec in (("f64s", F64S), ("f64", F64)):
        op = engine.HalfUpdate(src, tgt, True)
        op.prec = prec
        st = engine.SweepState(dev)
        st.init(2.5e-3, None, None, 4, "symmetrized")
        st.begin()
        out = torch.empty(n, dtype=torch.float64, device=dev)
        op(st, pot, out, skip=False)
        outs[name] = out.cpu().numpy()
    assert np.all(np.isfinite(outs["f64s"]))
    assert _rel(outs["f64s"], outs["f64"]) < 5e-9


@pytest.mark.parametrize("k", [3, 32])
@pytest.mark.parametrize("zero_side", ["rows", "cols", "none"])
def test_f64s_vanishing_dot_term(env, k, zero_side, monkeypatch):
    """At Gamma = 0 one side's dot features are all zero and the F64S sweep
    takes q_ij = -beta_j + s_i c_sj with one DFMA per pair instead of the DMMA
    k-steps (decided per call on the device): a loop of sweeps equals the
    dense fp64 DMMA path whichever side vanishes, and the generic case is
    untouched."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200._native import F64, F64S

    rng = np.random.default_rng(3 + k)
    n, m = 2100, 2900
    x = rng.standard_normal((n, k)) * (0.0 if zero_side == "rows" else 0.6)
    z = rng.standard_normal((m, k)) * (0.0 if zero_side == "cols" else 0.6)
    sx, sz = rng.random(n) * 6.0, rng.random(m) * 6.0
    src = engine.Side.make(x, sx, np.full(n, 1 / n), dev, k)
    tgt = engine.Side.make(z, sz, np.full(m, 1 / m), dev, k)
    pot = engine.to_dev64(rng.standard_normal(m) * 5.0, dev)
    outs = {}
    for name, prec in (("f64s", F64S), ("f64", F64)):
        op = engine.HalfUpdate(src, tgt, True)
        op.prec = prec
        st = engine.SweepState(dev)
        st.init(2.5e-3, None, None, 8, "symmetrized")
        res = []
        for _ in range(3):  # a probe sweep, then re-voted / measuring sweeps
            st.begin()
            out = torch.empty(n, dtype=torch.float64, device=dev)
            op(st, pot, out, skip=False)
            res.append(out.cpu().numpy())
        outs[name] = res
    for a_, b_ in zip(outs["f64s"], outs["f64"]):
        assert np.all(np.isfinite(a_))
        assert _rel(a_, b_) < 5e-9


@pytest.mark.parametrize("k,kind", [(3, "tc"), (3, "ffma"), (8, "tc"), (32, "tc"), (64, "tc")])
@pytest.mark.parametrize("zero_w", [False, True])
def test_f64s_probe_bounds(env, k, kind, zero_w, monkeypatch):
    """The probes store LOWER bounds of every row's minimum exponent q_ij =
    beta_j + sum_k a_ik b_jk over every column stage, a few log2 units (the
    published error bound) below the exact minima: read back from the plan
    workspace after a first sweep and compared with minima recomputed in
    fp64 from the device's own row block and column records."""
    P, engine, S, O, torch, dev = env
    from paper_2602_06658_b200._native import LIB

    monkeypatch.setenv("CNTGW_F64S_PROBE_TC", "1" if kind == "tc" else "0")
    monkeypatch.setenv("CNTGW_F64S_REMEASURE", "2.0")  # the exact sweep must not overwrite tmin
    rng = np.random.default_rng(7 + k)
    n, m = 1500, 2900
    cx = rng.standard_normal((16, k)) * (2.0 if k <= 8 else 0.5)
    x = cx[rng.integers(0, 16, n)] + rng.standard_normal((n, k)) * 0.5
    z = cx[rng.integers(0, 16, m)] + rng.standard_normal((m, k)) * 0.5
    a = np.full(n, 1 / n)
    b = np.where(np.arange(m) % 5 == 2, 0.0, 1.0) if zero_w else np.ones(m)
    b /= b.sum()
    g = rng.standard_normal(m) * 3.0 + (z * z).sum(1)
    eps = 2.5e-3
    prob = S.device_problem(P.SquaredEuclideanCost(x, z), a, b, dev)
    op = prob.fwd
    op.prec = 4
    st = engine.SweepState(dev)
    st.init(eps)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    op(st, engine.to_dev64(g - prob.col_sep, dev), out, skip=False)
    torch.cuda.synchronize()
    lay = np.zeros(3, dtype=np.int64)
    assert LIB.cntgw_f64s_plan_layout(op.kd, 1, n, m, lay.ctypes.data) == 0
    off, stages, td = (int(v) for v in lay)
    tmin = op.ws[off:off + 4 * n * stages].view(torch.float32).reshape(n, stages).cpu().numpy().astype(np.float64)
    kd = op.kd
    stride = LIB.cntgw_col_stride(4, kd, 1)
    mpad = stages * td
    rec = op.rec[:mpad * stride].reshape(mpad, stride).cpu().numpy()
    rows = op.f64s_rows.cpu().numpy()
    a256 = lambda v: (v + 255) // 256 * 256
    feat = rows[a256(8 * n):a256(8 * n) + 8 * n * kd].view(np.float64).reshape(n, kd)
    sq = rows[a256(8 * n) + a256(8 * n * kd):a256(8 * n) + a256(8 * n * kd) + 8 * n].view(np.float64)
    arow = np.concatenate([feat, sq[:, None]], axis=1)
    q = arow @ rec[:, :kd + 1].T + rec[None, :, kd + 1]
    q[:, m:] = np.inf  # padding columns
    exact = q.reshape(n, stages, td).min(axis=2)
    finite = np.isfinite(exact)
    assert np.all(np.isinf(tmin[~finite]) & (tmin[~finite] > 0))
    gap = exact[finite] - tmin[finite]
    assert gap.min() >= 0.0, f"probe value above the exact stage minimum by {-gap.min():.3e}"
    # ... and not uselessly loose: within a few units of the bound's own size
    scale = np.abs(rec[:m, kd + 1]).max() + np.linalg.norm(arow, axis=1).max() * np.linalg.norm(
        np.abs(rec[:m, :kd + 1]).max(axis=0))
    kp = (3 * (kd + 1) + 3 + 15) // 16 * 16
    bound = ((2 * kp + 32) if kind == "tc" else (kd + 5)) * 2.0 ** -24 * scale
    assert gap.max() <= 2.5 * bound + 1e-3, (gap.max(), bound)


@pytest.mark.parametrize("anneal", [None, 0.05], ids=["fixed", "annealed"])
@pytest.mark.parametrize("k,kind", [(3, "tc"), (4, "tc"), (3, "ffma"), (4, "ffma"), (8, "tc"), (16, "tc"),
                                    (32, "tc"), (64, "tc")])
def test_f64s_probe_matches_fp64_measurement(env, k, kind, anneal, monkeypatch):
    """CNTGW_F64S with a probe (the dense measurement of each loop's first
    sweep as stage minima minus a rigorous error bound: the tcgen05 probe,
    softmin_f64s_tcprobe.cuh, at every width, and the fp32 FFMA2 probe,
    softmin_f64s_probe.cuh, up to kd + sq = 8) against the fp64 measuring
    sweep (CNTGW_F64S_PROBE=0): every plan skips only terms below 2^-48 of
    their rows' maxima, so the loops agree to fp64 rounding; and both equal
    the dense fp64 loop. (A probe value above the true stage minimum would
    drop needed stages and show up here.)"""
    P, engine, S, O, torch, dev = env
    monkeypatch.setenv("CNTGW_F64S_PROBE_TC", "1" if kind == "tc" else "0")
    rng = np.random.default_rng(41 + k)
    n, m = (1 << 14, 3 << 12) if k <= 4 else (1 << 12, 3 << 11)
    cx = rng.standard_normal((16, k)) * 2.0
    x = cx[rng.integers(0, 16, n)] + rng.standard_normal((n, k)) * 0.5
    z = cx[rng.integers(0, 16, m)] @ np.linalg.qr(rng.standard_normal((k, k)))[0] \
        + rng.standard_normal((m, k)) * 0.5
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    cost = P.SquaredEuclideanCost(x, z)
    cfg = P.SinkhornConfig(eps=2.5e-3, n_inner=30, anneal_from=anneal)
    out = {}
    for tag, prec, probe in (("probe", "f64s", "1"), ("fp64", "f64s", "0"), ("dense", "f64", "1")):
        monkeypatch.setenv("CNTGW_PRECISION", prec)
        monkeypatch.setenv("CNTGW_F64S_PROBE", probe)
        res = P.sinkhorn(a, b, cost, cfg)
        out[tag] = (res.coupling.f, res.coupling.g)
    # (the walks differ in which stages they visit, so the lazy reference of
    # each row rebases at other points and the fp32 exponent arguments round
    # differently: ~1e-9 relative; the skipped mass itself is < 2^-64)
    assert _rel(out["probe"][0], out["fp64"][0]) < 5e-9
    assert _rel(out["probe"][1], out["fp64"][1]) < 5e-9
    assert _rel(out["probe"][0], out["dense"][0]) < 5e-8
    assert _rel(out["probe"][1], out["dense"][1]) < 5e-8
