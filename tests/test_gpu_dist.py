"""Row-sharded CNT-GW solve on the GPU: 2 ranks (gloo collectives, both on
cuda:0 — the ranks never wait on each other on the device, the collectives are
host-mediated) must reproduce the single-process solve and the reference's C1
golden values. Covers the sharded f-update, the partial-LSE g-update combine,
the gap reduction and the all-reduced outer-step reductions end to end."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results, precision="auto"):
    import torch
    import torch.distributed as dist

    os.environ["CNTGW_PRECISION"] = precision

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_06658_b200 as P

    g = golden("c1_solve")
    src = P.EmbeddedMeasure(g["x_feat"], g["a"])
    tgt = P.EmbeddedMeasure(g["y_feat"], g["b"])
    cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
    res = P.solve_cnt_gw(src, tgt, cfg)
    results[rank] = (res.value, np.array(res.coupling.f), np.array(res.coupling.g),
                     list(res.trace.inner_iters), np.array(res.gamma), np.array(res.argmax))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["auto", "f32c"])
def test_two_rank_sharded_solve_matches_reference(precision):
    """auto: the fp64/fp32 kernels the problem selects; f32c: the centred
    kernel forced, whose per-shard locality orders and scattered partial-LSE
    outputs must combine like the unsharded ones."""
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results, precision), nprocs=world, join=True)
    g = golden("c1_solve")
    v0, f0, g0, it0, gam0, am0 = results[0]
    v1, f1, g1, it1, gam1, am1 = results[1]
    assert v0 == v1 and np.array_equal(f0, f1) and np.array_equal(g0, g1)
    assert it0 == g["inner_iters"].tolist()
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()  # noqa: E731
    assert rel(f0, g["f"]) < 1e-4 and rel(g0, g["g"]) < 1e-4
    assert abs(v0 - float(g["value"])) < 1e-4 * abs(float(g["value"]))
    sure = g["argmax_gap"] > 1e-3
    assert np.array_equal(am0[sure], g["argmax"][sure])


# ---------------------------------------------------------------------------
# partial-LSE outputs of every kernel path, combined across row shards
# ---------------------------------------------------------------------------
def _sharded_g_update(prec, row_feat, row_sq, col_feat, col_sq, a, b, f_ref, row_sep, eps, shards=2):
    """The g-update of a row-sharded run, simulated in one process: each shard's
    bwd operator writes per-column partial (max, sum) pairs over its own rows,
    the pairs are merged with the library's rescale kernel (the step the NCCL
    exchange runs between ranks) and finalised."""
    import torch

    from paper_2602_06658_b200 import dist as D
    from paper_2602_06658_b200 import engine
    from paper_2602_06658_b200._native import call
    from paper_2602_06658_b200.sinkhorn import feature_problem

    dev = torch.device("cuda", 0)
    n = row_feat.shape[0]
    m = col_feat.shape[0]
    st = engine.SweepState(dev)
    st.init(eps)
    parts = []
    for r in range(shards):
        lo, hi = D.shard_range(n, r, shards)
        _, _, _, bwd = feature_problem(row_feat[lo:hi], None if row_sq is None else row_sq[lo:hi],
                                       col_feat, col_sq, a[lo:hi], b, dev)
        bwd.prec = prec
        mx = torch.empty(m, dtype=torch.float64, device=dev)
        sm = torch.empty(m, dtype=torch.float64, device=dev)
        f_t = engine.to_dev64(f_ref[lo:hi] - row_sep[lo:hi], dev)
        bwd.partials(st, f_t, mx, sm, skip=False)
        parts.append((mx, sm, bwd))
    mg = torch.stack([p[0] for p in parts]).amax(0)
    total = torch.zeros(m, dtype=torch.float64, device=dev)
    for mx, sm, _ in parts:
        call("cntgw_lse_rescale", mx.data_ptr(), mg.data_ptr(), sm.data_ptr(), m,
             torch.cuda.current_stream().cuda_stream)
        total += sm
    out = torch.empty(m, dtype=torch.float64, device=dev)
    parts[0][2].finalize(st, mg, total, out, skip=False)
    return out.cpu().numpy()


@pytest.mark.parametrize("prec_name", ["tc", "f32"])
def test_partial_lse_c2_shape_two_shards(cuda, prec_name):
    """C2 cost form (K=16, no squared coordinate) on the tcgen05 3xTF32 and
    fp32 kernels: sharded g-update = the oracle's full-N g-update on sampled
    columns."""
    from oracle import cntgw_oracle as O
    from paper_2602_06658_b200 import configs
    from paper_2602_06658_b200._native import F32, TF32X3

    n = m = 1 << 15
    inst = configs.c2(seed=4, n=n, k=16)
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    f = np.random.default_rng(1).standard_normal(n) + inst.row_sep
    prec = TF32X3 if prec_name == "tc" else F32
    got = _sharded_g_update(prec, inst.u, None, inst.v, None, a, b, f, inst.row_sep.astype(float),
                            inst.eps) + inst.col_sep
    cols = np.sort(np.random.default_rng(2).choice(m, 96, replace=False))
    want = O.softmin(O.LowRank(inst.v, inst.u, inst.col_sep, inst.row_sep), np.log(a), f, inst.eps,
                     row_idx=cols)
    assert np.abs(got[cols] - want).max() / np.abs(want).max() < 1e-5


@pytest.mark.parametrize("prec_name", ["dmma", "f64s", "f32c"])
def test_partial_lse_c5_and_c4_shapes_two_shards(cuda, prec_name, monkeypatch):
    """C5 shape (E-side projection: 32 dot features + the squared coordinate)
    on the fp64 DMMA kernel and on CNTGW_F64S (ordered rows, measured plan),
    and the C4 shape (3 + sq) on the centred kernel (partials scattered back
    to the caller's order), cold regime: sharded g-update = the oracle on
    sampled columns."""
    from oracle import cntgw_oracle as O
    from paper_2602_06658_b200._native import F32C, F64, F64S

    rng = np.random.default_rng(5)
    n = m = 1 << 14
    k = 3 if prec_name == "f32c" else 32
    cx = rng.standard_normal((8, k)) * 2.0
    x = cx[rng.integers(0, 8, n)] + rng.standard_normal((n, k)) * 0.6
    z = cx[rng.integers(0, 8, m)] + rng.standard_normal((m, k)) * 0.6
    xs, zs = 0.5 * (x * x).sum(1), 0.5 * (z * z).sum(1)
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    eps = 1.25e-3 if prec_name == "f32c" else 2.5e-3
    row_sep, col_sep = (x * x).sum(1), (z * z).sum(1)
    f = rng.standard_normal(n) * 3.0 + row_sep + xs * xs
    monkeypatch.setenv("CNTGW_F64_DMMA", "1")
    prec = {"dmma": F64, "f64s": F64S, "f32c": F32C}[prec_name]
    got = _sharded_g_update(prec, x, xs, z, zs, a, b, f, row_sep, eps) + col_sep
    cols = np.sort(rng.choice(m, 96, replace=False))
    cost = O.SqEuclid(np.column_stack([x, xs]), np.column_stack([z, zs]))
    want = O.softmin(cost.T(), np.log(a), f, eps, row_idx=cols)
    assert np.abs(got[cols] - want).max() / np.abs(want).max() < 1e-5


@pytest.mark.parametrize("precision", ["auto", "f32c"])
def test_native_nccl_sharded_solve_single_rank(cuda, precision, monkeypatch):
    """The row-sharded solve with the library's own NCCL communicator
    (cntgw_comm_*, a single-rank communicator here): every exchange — the
    partial-LSE combine, the gap partials, the outer-step reductions — is an
    NCCL collective enqueued on the compute stream and captured inside the
    solve's CUDA graph (nested conditional WHILE nodes). Same trajectory as
    the unsharded solve and the reference's C1 values."""
    import paper_2602_06658_b200 as P
    from paper_2602_06658_b200 import solvers

    g = golden("c1_solve")
    src = P.EmbeddedMeasure(g["x_feat"], g["a"])
    tgt = P.EmbeddedMeasure(g["y_feat"], g["b"])
    cfg = P.make_config(0.01, threshold=1e-5, max_inner=200, max_outer=20)
    monkeypatch.setenv("CNTGW_PRECISION", precision)
    plain = P.solve_cnt_gw(src, tgt, cfg)
    monkeypatch.setenv("CNTGW_FORCE_SHARDED", "1")
    st = solvers._CntGwState(src, tgt, cfg)
    assert st.dev.comm is not None and st.dev.comm.capturable
    res = P.solve_cnt_gw(src, tgt, cfg)
    assert res.trace.inner_iters == plain.trace.inner_iters == g["inner_iters"].tolist()
    np.testing.assert_allclose(res.trace.objectives, plain.trace.objectives, rtol=1e-12)
    assert np.abs(res.coupling.f - plain.coupling.f).max() <= 1e-12 * np.abs(plain.coupling.f).max()
    assert abs(res.value - float(g["value"])) < 1e-4 * abs(float(g["value"]))
    sure = g["argmax_gap"] > 1e-3
    assert np.array_equal(res.argmax[sure], g["argmax"][sure])
