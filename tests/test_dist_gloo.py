"""Row-sharded multi-process logic (dist.py) on CPU with the gloo backend,
world size 2. The local half-update operators are replaced by oracle-backed
CPU stand-ins with the same interface (``partials`` / ``finalize``); what is
tested is the sharding, the partial-LSE all-reduce combine, the gap reduction
and that every rank ends with the full, identical g."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_06658_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _OracleColumnOp:
    """CPU stand-in for HalfUpdate over local rows: per-column partial LSE."""

    def __init__(self, cost_local, log_a_local, eps):
        self.c = cost_local  # local rows x M
        self.la = log_a_local
        self.lam = np.log2(np.e) / eps

    def partials(self, state, f_local, mx, sm, skip=True):
        t = (self.la[:, None] / np.log(2.0)) + self.lam * (f_local.numpy()[:, None] - self.c)
        m = t.max(axis=0)
        mx.copy_(torch.from_numpy(m))
        sm.copy_(torch.from_numpy(np.exp2(t - m[None, :]).sum(axis=0)))

    def finalize(self, state, mx, sm, out, skip=True, row_add=None):
        out.copy_(-(mx + torch.log2(sm)) / self.lam)


class _Loop:
    def __init__(self, op, pr):
        self.bwd = op
        self.state = None
        self.pr = pr
        self.gap_n = 1


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    info = D.init_from_env("gloo")
    rng = np.random.default_rng(0)
    n, m, eps = 37, 23, 0.3
    cost = rng.random((n, m))
    a = rng.random(n) + 0.5
    a /= a.sum()
    f = rng.standard_normal(n) * 0.1
    lo, hi = D.shard_range(n, info.rank, info.world)
    comm = D.RowShardComm(info)
    # g-update over all ranks' rows
    op = _OracleColumnOp(cost[lo:hi], np.log(a[lo:hi]), eps)
    pr = torch.zeros(4, dtype=torch.float64)
    pr[:2] = torch.tensor([0.25 * (rank + 1), 0.5])
    loop = _Loop(op, pr)
    out = torch.zeros(m, dtype=torch.float64)
    comm.g_update(loop, torch.from_numpy(f[lo:hi]), out)
    comm.reduce_gap_partials(loop)
    tot = comm.all_sum(torch.tensor([float(hi - lo)], dtype=torch.float64))
    results[rank] = (out.numpy().copy(), float(loop.pr.sum()), float(tot), (lo, hi))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_g_update_matches_oracle():
    from oracle import cntgw_oracle as O

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    rng = np.random.default_rng(0)
    n, m, eps = 37, 23, 0.3
    cost = rng.random((n, m))
    a = rng.random(n) + 0.5
    a /= a.sum()
    f = rng.standard_normal(n) * 0.1
    want = O.softmin(O.Dense(cost.T), np.log(a), f, eps)
    g0, gap0, n0, s0 = results[0]
    g1, gap1, n1, s1 = results[1]
    assert np.array_equal(g0, g1)  # identical on every rank, no broadcast needed
    assert np.abs(g0 - want).max() < 1e-12
    assert gap0 == pytest.approx(0.25 + 0.5 + 0.5 + 0.5) and gap1 == gap0
    assert n0 == n1 == n
    assert s0 == (0, 19) and s1 == (19, 37)


@pytest.mark.parametrize("n,world", [(10, 3), (1, 2), (1 << 20, 8), (7, 7)])
def test_shard_range_partitions(n, world):
    spans = [D.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
    sizes = [h - l for l, h in spans]
    assert max(sizes) - min(sizes) <= 1
