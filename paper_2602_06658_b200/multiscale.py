"""Multiscale front end (reference solvers.py:668-726 and 729-763; SURVEY.md
§8(f) row 2): weighted k-means coarsening on the GPU, a coarse solve, and a
fine solve warm-started from cluster-constant upsampled potentials.

The reference builds a dense N x k x D distance tensor per Lloyd sweep
(infeasible at N = 1e6); here the assignment streams the centres through
shared memory (``cntgw_km_assign``) and the k-means++ draws run on the device
(``cntgw_km_draw``), bit-compatible with the reference's numpy arithmetic so
the coarse problems — and hence the multiscale results — are the reference's
own (see csrc/kmeans.cu for the exact ordering rules). Only the uniforms come
from the host ``numpy.random.Generator`` (the same stream ``choice`` draws).
"""

from __future__ import annotations

import heapq
import math
import os
import time
from dataclasses import replace

import numpy as np
import torch

from . import engine
from ._native import LIB, call
from .kernels import EmbeddedMeasure

_TREES: dict = {}


def _pw_tree(n: int, device):
    """numpy's pairwise-summation tree of n values: leaf offsets (blocks <= 128,
    halves rounded down to multiples of 8) and the internal nodes as
    (node, left, right) ordered by height, so a level only reads finished
    children."""
    key = (n, str(device))
    if key not in _TREES:
        offs, nodes = [], []  # nodes: (height, left, right) with child ids

        def build(off, m):  # returns (node id or ('leaf', k), height)
            if m <= 128:
                offs.append(off)
                return ("L", len(offs) - 1), 0
            m2 = m // 2
            m2 -= m2 % 8
            left, hl = build(off, m2)
            right, hr = build(off + m2, m - m2)
            nodes.append((max(hl, hr) + 1, left, right))
            return ("I", len(nodes) - 1), max(hl, hr) + 1

        import sys

        sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
        build(0, n)
        nleaves = len(offs)
        order = sorted(range(len(nodes)), key=lambda t: (nodes[t][0], t))
        ident = {t: nleaves + r for r, t in enumerate(order)}

        def ref(c):
            return c[1] if c[0] == "L" else ident[c[1]]

        tree, hoff, cur = [], [0], 1
        for t in order:
            h = nodes[t][0]
            while h > cur:
                hoff.append(len(tree) // 3)
                cur += 1
            tree += [ident[t], ref(nodes[t][1]), ref(nodes[t][2])]
        hoff.append(len(tree) // 3)
        if not nodes:
            hoff = [0]
        offs.append(n)
        _TREES[key] = (torch.tensor(offs, dtype=torch.int64, device=device),
                       torch.tensor(tree or [0, 0, 0], dtype=torch.int32, device=device),
                       torch.tensor(hoff, dtype=torch.int32, device=device), len(hoff) - 1)
    return _TREES[key]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _centers_from(x, w, assign, counts, centers, ids=None, masses=None):
    """Centres (or masses) of the clusters of ``assign`` from a stable CSR."""
    k = counts.numel()
    perm = torch.sort(assign, stable=True).indices
    offsets = torch.zeros(k + 1, dtype=torch.int64, device=x.device)
    offsets[1:] = torch.cumsum(counts, 0)
    call("cntgw_km_centers", x.data_ptr(), x.shape[1], w.data_ptr(), perm.data_ptr(),
         offsets.data_ptr(), k, 0, 0 if masses is not None else centers.data_ptr(),
         masses.data_ptr() if masses is not None else 0, _stream())
    return perm, offsets


def _fill_empty(x, assign, own, counts, centers):
    """The reference's in-order handling of empty clusters (solvers.py:689-697):
    cluster j empty at its turn takes the point farthest from its centre.
    Returns the moves (j, point, previous cluster) in processing order."""
    empty = (counts == 0).nonzero().flatten().tolist()
    if not empty:
        return []
    heap = list(empty)
    heapq.heapify(heap)
    moves = []
    while heap:
        j = heapq.heappop(heap)
        far = int(torch.argmax(own))  # first maximum, like numpy
        orig = int(assign[far])
        assign[far] = j
        own[far] = 0.0
        counts[orig] -= 1
        counts[j] += 1
        moves.append((j, far, orig))
        if orig > j and int(counts[orig]) == 0:  # emptied before its own turn
            heapq.heappush(heap, orig)
    return moves


def _refresh_robbed(x, w, perm, offsets, moves, centers):
    """Clusters that lost a point to a LATER empty cluster computed their
    centre (at their turn) with that point still a member."""
    extra: dict[int, list[int]] = {}
    for j, far, orig in moves:
        if orig < j:
            extra.setdefault(orig, []).append(far)
    if not extra:
        return
    ids, segs = [], []
    off = offsets.cpu().numpy()
    for c, pts in sorted(extra.items()):
        members = perm[off[c]:off[c + 1]].cpu().numpy().tolist()
        segs.append(sorted(set(members) | set(pts)))
        ids.append(c)
    lens = np.cumsum([0] + [len(s) for s in segs])
    dev = x.device
    mem = torch.tensor([i for s in segs for i in s], dtype=torch.int64, device=dev)
    offs = torch.tensor(lens, dtype=torch.int64, device=dev)
    idt = torch.tensor(ids, dtype=torch.int64, device=dev)
    call("cntgw_km_centers", x.data_ptr(), x.shape[1], w.data_ptr(), mem.data_ptr(), offs.data_ptr(),
         len(ids), idt.data_ptr(), centers.data_ptr(), 0, _stream())


def _weighted_kmeans(features, weights, k, rng, sweeps: int = 100):
    """Seeded weighted k-means (reference solvers.py:668-705) on the GPU.
    Returns (assignments, centers, center_weights) as numpy arrays."""
    dev = engine.require_cuda()
    x = engine.to_dev64(np.ascontiguousarray(features, dtype=np.float64), dev)
    w = engine.to_dev64(weights, dev)
    n, d = x.shape
    k = int(k)
    # k-means++: one Generator.choice per centre = one uniform each
    us = torch.as_tensor(rng.random(k), dtype=torch.float64, device=dev)
    leaves, tree, hoff, nh = _pw_tree(n, dev)
    nl = leaves.numel() - 1
    ws_bytes = int(LIB.cntgw_km_draw_workspace(n, nl))
    ws = torch.empty((ws_bytes + 7) // 8, dtype=torch.float64, device=dev)
    idx = torch.empty(1, dtype=torch.int64, device=dev)
    jdev = torch.zeros(1, dtype=torch.int32, device=dev)  # draw index, advanced on the device
    centers = torch.empty((k, d), dtype=torch.float64, device=dev)
    d2 = torch.empty(n, dtype=torch.float64, device=dev)

    def draw(first):
        st = _stream()
        call("cntgw_km_draw", w.data_ptr(), 0 if first else d2.data_ptr(), n, leaves.data_ptr(), nl,
             tree.data_ptr(), hoff.data_ptr(), nh, us.data_ptr(), jdev.data_ptr(), idx.data_ptr(),
             ws.data_ptr(), ws_bytes, st)
        call("cntgw_km_update_d2", x.data_ptr(), n, d, idx.data_ptr(), centers.data_ptr(),
             jdev.data_ptr(), d2.data_ptr(), 1 if first else 0, st)

    timing = os.environ.get("CNTGW_KM_TIMING") == "1"
    if timing:
        t_start = time.perf_counter()
    draw(True)
    # the k-1 sequential draws replay a captured chunk of draws (the index
    # lives on the device), one graph launch per chunk
    chunk = int(os.environ.get("CNTGW_KM_CHUNK", "64"))
    reps, rest = divmod(k - 1, chunk) if chunk > 0 else (0, k - 1)
    if reps:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                for _ in range(chunk):
                    draw(False)
        torch.cuda.current_stream().wait_stream(side)
        # capture does not execute: replay all chunks
        for _ in range(reps):
            g.replay()
    for _ in range(rest):
        draw(False)
    if timing:
        torch.cuda.synchronize()
        print(f"[km] {k} k-means++ draws: {time.perf_counter() - t_start:.3f} s", flush=True)
        t_start = time.perf_counter()
    s = _stream()
    assign = torch.zeros(n, dtype=torch.int64, device=dev)
    new = torch.empty_like(assign)
    own = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(sweeps):
        call("cntgw_km_assign", x.data_ptr(), n, d, centers.data_ptr(), k, new.data_ptr(),
             own.data_ptr(), s)
        counts = torch.bincount(new, minlength=k)
        moves = _fill_empty(x, new, own, counts, centers)
        perm, offsets = _centers_from(x, w, new, counts, centers)
        if moves:
            _refresh_robbed(x, w, perm, offsets, moves, centers)
        done = torch.equal(new, assign)
        assign.copy_(new)
        if done:
            break
    if timing:
        torch.cuda.synchronize()
        print(f"[km] Lloyd sweeps: {time.perf_counter() - t_start:.3f} s", flush=True)
    counts = torch.bincount(assign, minlength=k)
    masses = torch.zeros(k, dtype=torch.float64, device=dev)
    _centers_from(x, w, assign, counts, centers, masses=masses)
    return assign.cpu().numpy(), centers.cpu().numpy(), masses.cpu().numpy()


def coarsen(measure, rho: float, rng):
    """Cluster an embedded measure into ceil(rho n) weighted centroids
    (solvers.py:708-726). Returns the coarse measure and the assignment."""
    if not (0.0 < rho < 1.0):
        raise ValueError(f"rho must lie in (0, 1), got {rho!r}")
    k = math.ceil(rho * measure.n)
    if k < 2:
        raise ValueError(
            f"rho={rho} gives {k} cluster(s) for {measure.n} points; need at least 2")
    assign, centers, center_weights = _weighted_kmeans(measure.features, measure.weights, k, rng)
    coarse = EmbeddedMeasure(centers, center_weights,
                             explained_variance=getattr(measure, "explained_variance", 1.0))
    return coarse, assign


def solve_multiscale(src, tgt, cfg, rho: float = 0.1):
    """Two-stage solve (solvers.py:729-763): coarse solve on weighted k-means
    centroids, then the fine solve from the coarse operator and the
    cluster-constant upsampled potentials (separable parts swapped for the
    fine problem's own)."""
    from .solvers import solve_cnt_gw

    rng = np.random.default_rng(cfg.seed)
    coarse_src, assign_src = coarsen(src, rho, rng)
    coarse_tgt, assign_tgt = coarsen(tgt, rho, rng)
    coarse_result = solve_cnt_gw(coarse_src, coarse_tgt, cfg)
    gamma_c = coarse_result.gamma
    phi_c = (coarse_src.augmented() ** 2).sum(axis=1)
    psi_c = (np.column_stack([coarse_tgt.features @ gamma_c.T, coarse_tgt.half_sq_norms]) ** 2).sum(axis=1)
    phi_f = (np.column_stack([src.features, src.half_sq_norms]) ** 2).sum(axis=1)
    psi_f = (np.column_stack([np.asarray(tgt.features) @ gamma_c.T, tgt.half_sq_norms]) ** 2).sum(axis=1)
    f_up = (coarse_result.coupling.f - phi_c)[assign_src] + phi_f
    g_up = (coarse_result.coupling.g - psi_c)[assign_tgt] + psi_f
    fine_cfg = replace(cfg, init="gamma", init_gamma=gamma_c)
    fine_result = solve_cnt_gw(src, tgt, fine_cfg, _warm_potentials=(f_up, g_up))
    fine_result.coarse = coarse_result
    return fine_result
