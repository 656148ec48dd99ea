"""CPU oracle for the CNT-GW hot path — TEST INFRASTRUCTURE ONLY.

A float64 numpy/scipy restatement of the reference package ``cntgw``'s hot
path (arXiv 2602.06658, ``/root/reference/pkg/src/cntgw``). It exists to CHECK
the B200 path: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it. The
product package never imports it and has no CPU fallback.

Pinning: every function is checked against golden vectors produced by the
reference itself in the build container (``tests/golden/make_golden.py``
imports ``/root/reference`` read-only and commits the outputs as fixtures;
``tests/test_oracle.py`` replays them). Third-party arithmetic at the
boundary: ``scipy.special.logsumexp`` (reference pin ``scipy>=1.10``,
``pyproject.toml:13``; 1.18.1 installed) and numpy's BLAS ``@``.

Each routine cites the reference lines it restates.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import logsumexp

BLOCK = 1024  # reference row-block size, measures.py:19


# ----------------------------------------------------------------------------
# cost rows (sinkhorn.py:59-109)
# ----------------------------------------------------------------------------
class SqEuclid:
    """Squared-Euclidean rows max(|x|^2+|z|^2-2x.z, 0) (sinkhorn.py:83-85)."""

    def __init__(self, x, z):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.z = np.ascontiguousarray(z, dtype=np.float64)
        self.nx = np.einsum("ij,ij->i", self.x, self.x)
        self.nz = np.einsum("ij,ij->i", self.z, self.z)
        self.shape = (self.x.shape[0], self.z.shape[0])

    def rows(self, i0, i1):
        c = self.nx[i0:i1, None] + self.nz[None, :]
        c -= 2.0 * (self.x[i0:i1] @ self.z.T)
        return np.maximum(c, 0.0)

    def T(self):
        return SqEuclid(self.z, self.x)


class Dense:
    """Explicit cost matrix rows (sinkhorn.py:30-56)."""

    def __init__(self, c):
        self.c = np.ascontiguousarray(c, dtype=np.float64)
        self.shape = self.c.shape

    def rows(self, i0, i1):
        return self.c[i0:i1]

    def T(self):
        return Dense(self.c.T)


class LowRank:
    """C2 micro-benchmark cost a_i + b_j - 2 u_i.v_j, no clip."""

    def __init__(self, u, v, ra, cb):
        self.u = np.asarray(u, dtype=np.float64)
        self.v = np.asarray(v, dtype=np.float64)
        self.ra = np.asarray(ra, dtype=np.float64)
        self.cb = np.asarray(cb, dtype=np.float64)
        self.shape = (self.u.shape[0], self.v.shape[0])

    def rows(self, i0, i1):
        return self.ra[i0:i1, None] + self.cb[None, :] - 2.0 * (self.u[i0:i1] @ self.v.T)

    def T(self):
        return LowRank(self.v, self.u, self.cb, self.ra)


# ----------------------------------------------------------------------------
# half-update and gaps (sinkhorn.py:166-188)
# ----------------------------------------------------------------------------
def softmin(cost, log_w, pot, eps, row_idx=None, threads=1, block=BLOCK):
    """out_i = -eps * logsumexp_j(log_w_j + (pot_j - C_ij)/eps)  (sinkhorn.py:166-176).

    ``row_idx`` restricts the evaluation to a subset of rows (used for the
    full-size subsample parity checks); ``threads`` splits the row blocks over
    a thread pool (numpy/BLAS release the GIL), which is how the CPU baseline
    uses the host's cores; ``block`` (default the reference's 1024 rows) bounds
    the per-block memory (block x M doubles) when many threads run at once.
    """
    bias = np.asarray(log_w, dtype=np.float64) + np.asarray(pot, dtype=np.float64) / eps
    n = cost.shape[0]
    if row_idx is None:
        spans = [(i0, min(i0 + block, n)) for i0 in range(0, n, block)]
        out = np.empty(n)

        def run(span):
            i0, i1 = span
            out[i0:i1] = -eps * logsumexp(bias[None, :] - cost.rows(i0, i1) / eps, axis=1)
    else:
        row_idx = np.asarray(row_idx)
        out = np.empty(row_idx.size)
        spans = [(k, min(k + block, row_idx.size)) for k in range(0, row_idx.size, block)]

        def run(span):
            k0, k1 = span
            blk = np.vstack([cost.rows(int(i), int(i) + 1) for i in row_idx[k0:k1]])
            out[k0:k1] = -eps * logsumexp(bias[None, :] - blk / eps, axis=1)

    if threads > 1 and len(spans) > 1:
        with ThreadPoolExecutor(threads) as pool:
            list(pool.map(run, spans))
    else:
        for s in spans:
            run(s)
    return out


def weighted_gap(w, pot, tent, eps):
    """sum w_i^2 |exp(min((pot-tent)/eps, 700)) - 1|  (sinkhorn.py:179-188)."""
    r = np.minimum((pot - tent) / eps, 700.0)
    return float(np.sum(w * w * np.abs(np.exp(r) - 1.0)))


# ----------------------------------------------------------------------------
# plan marginals and diagnostics (measures.py:185-256)
# ----------------------------------------------------------------------------
def plan_blocks(f, g, cost, a, b, eps):
    """Yield (i0, i1, pi block) with pi = a b exp((f+g-C)/eps) (measures.py:185-195)."""
    la = np.log(a) + f / eps
    lb = np.log(b) + g / eps
    n = cost.shape[0]
    for i0 in range(0, n, BLOCK):
        i1 = min(i0 + BLOCK, n)
        yield i0, i1, np.exp(la[i0:i1, None] + lb[None, :] - cost.rows(i0, i1) / eps)


def marginals(f, g, cost, a, b, eps):
    r = np.empty(cost.shape[0])
    c = np.zeros(cost.shape[1])
    for i0, i1, p in plan_blocks(f, g, cost, a, b, eps):
        r[i0:i1] = p.sum(axis=1)
        c += p.sum(axis=0)
    return r, c


def marginal_error(f, g, cost, a, b, eps):
    """||row - a||_1 + ||col - b||_1 (measures.py:229-235)."""
    r, c = marginals(f, g, cost, a, b, eps)
    return float(np.abs(r - a).sum() + np.abs(c - b).sum())


def kl(f, g, cost, a, b, eps):
    """KL(pi | a x b) via the potentials' log-ratio (measures.py:245-252)."""
    tot = 0.0
    for i0, i1, p in plan_blocks(f, g, cost, a, b, eps):
        tot += float((p * ((f[i0:i1, None] + g[None, :] - cost.rows(i0, i1)) / eps)).sum())
    return tot


# ----------------------------------------------------------------------------
# Sinkhorn loop (sinkhorn.py:112-258)
# ----------------------------------------------------------------------------
def sinkhorn(a, b, cost, eps, mode="symmetrized", n_inner=None, threshold=None,
             max_inner=10000, anneal_from=None, warm=None):
    """Log-domain Sinkhorn with the reference's control semantics.

    Budget: ``n_inner`` (default 100 when neither is given) xor ``threshold``
    (+ ``max_inner``), sinkhorn.py:137-140. Annealing eps_n = max(a0/sqrt(n), eps)
    (:223-226); the threshold is checked on tentatives only at eps_n == eps,
    before averaging, and the breaking sweep is not counted (:228-251).
    Returns dict(f, g, iterations, converged, eps_eff, marginal_err).
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if n_inner is None and threshold is None:
        n_inner = 100
    la, lb = np.log(a), np.log(b)
    n, m = cost.shape
    if warm is None:
        f, g = np.zeros(n), np.zeros(m)
    else:
        f = np.array(warm[0], dtype=np.float64)
        g = np.array(warm[1], dtype=np.float64)
    ct = cost.T()
    use_tau = threshold is not None
    sweeps = max_inner if use_tau else n_inner
    applied, converged, eps_eff = 0, not use_tau, eps
    for k in range(1, sweeps + 1):
        e = eps if anneal_from is None else max(anneal_from / np.sqrt(k), eps)
        eps_eff = e
        check = use_tau and e == eps
        if mode == "symmetrized":
            ft = softmin(cost, lb, g, e)
            gt = softmin(ct, la, f, e)
            if check and weighted_gap(a, f, ft, e) < threshold and weighted_gap(b, g, gt, e) < threshold:
                converged = True
                break
            f, g = 0.5 * (f + ft), 0.5 * (g + gt)
        else:
            ft = softmin(cost, lb, g, e)
            if check and weighted_gap(a, f, ft, e) < threshold:
                converged = True
                break
            f = ft
            g = softmin(ct, la, f, e)
        applied = k
    return dict(f=f, g=g, iterations=applied, converged=converged, eps_eff=eps_eff,
                marginal_err=marginal_error(f, g, cost, a, b, eps_eff))


# ----------------------------------------------------------------------------
# CNT-GW outer solver (solvers.py:190-339, 556-632; divergence.py:28-47)
# ----------------------------------------------------------------------------
def center(points, w):
    """Weighted-mean centering of the sq-Euclidean fast path (kernels.py:400-418)."""
    p = np.asarray(points, dtype=np.float64)
    return p - (w @ p)[None, :]


def fourth_moment(x, w):
    """Q = sum_ik w_i w_k |x_i - x_k|^4 in row blocks (divergence.py:28-38)."""
    sq = np.einsum("ij,ij->i", x, x)
    tot = 0.0
    for i0 in range(0, x.shape[0], BLOCK):
        d2 = np.maximum(sq[i0:i0 + BLOCK, None] + sq[None, :] - 2.0 * x[i0:i0 + BLOCK] @ x.T, 0.0)
        tot += float(w[i0:i0 + BLOCK] @ (d2 * d2) @ w)
    return tot


def constant(x, a, y, b):
    """C = Q_x + Q_y - 4 T_x T_y with T = sum w |x|^2 (divergence.py:41-47, kernels.py:392)."""
    tx = float(a @ np.einsum("ij,ij->i", x, x))
    ty = float(b @ np.einsum("ij,ij->i", y, y))
    return fourth_moment(x, a) + fourth_moment(y, b) - 4.0 * tx * ty


def augment(feat):
    """[features, |x|^2/2] (kernels.py:371, 385-387)."""
    return np.column_stack([feat, 0.5 * np.einsum("ij,ij->i", feat, feat)])


def zbar_of(gamma, y):
    """[Y Gamma^T, s_y] (solvers.py:219, 311-313)."""
    return np.column_stack([y @ gamma.T, 0.5 * np.einsum("ij,ij->i", y, y)])


def cnt_reductions(f, g, cost, x, a, y, b, eps):
    """One pass: (pi Y, sigma_ss, KL, Err) (solvers.py:227-256)."""
    sx = 0.5 * np.einsum("ij,ij->i", x, x)
    sy = 0.5 * np.einsum("ij,ij->i", y, y)
    pi_y = np.zeros((x.shape[0], y.shape[1]))
    col = np.zeros(y.shape[0])
    sig = klv = rerr = 0.0
    for i0, i1, p in plan_blocks(f, g, cost, a, b, eps):
        lr = (f[i0:i1, None] + g[None, :] - cost.rows(i0, i1)) / eps
        pi_y[i0:i1] = p @ y
        rs = p.sum(axis=1)
        col += p.sum(axis=0)
        sig += float(sx[i0:i1] @ (p @ sy))
        klv += float((p * lr).sum())
        rerr += float(np.abs(rs - a[i0:i1]).sum())
    return pi_y, sig, klv, rerr + float(np.abs(col - b).sum())


def plan_reductions(f, g, cost, a, b, eps, x, y):
    """(pi Y, pi s_y, pi^T X, pi^T s_x, sigma_ss) in one blocked pass
    (divergence.py:72-86)."""
    sx = 0.5 * np.einsum("ij,ij->i", x, x)
    sy = 0.5 * np.einsum("ij,ij->i", y, y)
    pi_y = np.empty((x.shape[0], y.shape[1]))
    pi_sy = np.empty(x.shape[0])
    pit_x = np.zeros((y.shape[0], x.shape[1]))
    pit_sx = np.zeros(y.shape[0])
    for i0, i1, p in plan_blocks(f, g, cost, a, b, eps):
        pi_y[i0:i1] = p @ y
        pi_sy[i0:i1] = p @ sy
        pit_x += p.T @ x[i0:i1]
        pit_sx += p.T @ sx[i0:i1]
    return pi_y, pi_sy, pit_x, pit_sx, float(sx @ pi_sy)


def grad_constant(x, a, other_trace):
    """Per-point gradient of Q - 4 T T_other, O(N^2 D) blocks (divergence.py:138-150)."""
    sq_norms = (x**2).sum(axis=1)
    out = np.empty_like(x)
    for i0 in range(0, x.shape[0], BLOCK):
        i1 = min(i0 + BLOCK, x.shape[0])
        diff = x[i0:i1, None, :] - x[None, :, :]
        sq = np.maximum(sq_norms[i0:i1, None] + sq_norms[None, :] - 2.0 * (x[i0:i1] @ x.T), 0.0)
        out[i0:i1] = 8.0 * a[i0:i1, None] * np.einsum("mk,mkd->md", sq * a[None, :], diff)
    out -= 8.0 * other_trace * a[:, None] * x
    return out


def feature_gradients(x, a, y, b, gamma, red):
    """Envelope gradients from the plan reductions (divergence.py:153-172)."""
    pi_y, pi_sy, pit_x, pit_sx, _ = red
    tx = float(a @ (x**2).sum(1))
    ty = float(b @ (y**2).sum(1))
    gsrc = grad_constant(x, a, ty) - 16.0 * (pi_y @ gamma.T + x * pi_sy[:, None])
    gtgt = grad_constant(y, b, tx) - 16.0 * (pit_x @ gamma + y * pit_sx[:, None])
    return gsrc, gtgt


def solve_cnt_gw(x, a, y, b, eps, inner, max_outer=200, delta_outer=1e-5,
                 gamma0=None, warm=None, final_anneal=None):
    """Feature-space EGW alternate minimisation (solvers.py:285-350, 556-632).

    ``x``/``y`` are centered features. ``inner`` is a dict of sinkhorn kwargs
    (mode, n_inner / threshold, max_inner). Returns a dict with the result
    pairing of the reference: ``gamma`` = Gamma_{t+1}, coupling factors
    (f, g, zbar, eps_eff) built on Gamma_t (Appendix A.1 item 11).
    Raises RuntimeError (the SolverError analogue) after 5 increases.
    """
    d, e_dim = x.shape[1], y.shape[1]
    gamma = np.zeros((d, e_dim)) if gamma0 is None else np.array(gamma0, dtype=np.float64)
    xbar = augment(x)
    psi = np.einsum("ij,ij->i", zbar_of(gamma, y), zbar_of(gamma, y))
    if warm is None:
        f = np.einsum("ij,ij->i", xbar, xbar)
        g = psi.copy()
    else:
        f, g = np.array(warm[0], dtype=np.float64), np.array(warm[1], dtype=np.float64)
    const = constant(x, a, y, b)
    trace = dict(objective=[], gamma_delta=[], marginal_err=[], inner_iters=[])
    state = {}

    def step(anneal=None):
        nonlocal gamma, psi, f, g
        zb = zbar_of(gamma, y)
        psi_now = np.einsum("ij,ij->i", zb, zb)
        g = g + (psi_now - psi)
        psi = psi_now
        cost = SqEuclid(xbar, zb)
        kw = dict(inner)
        if anneal is not None:
            kw["anneal_from"] = anneal
        res = sinkhorn(a, b, cost, eps / 8.0, warm=(f, g), **kw)
        f, g = res["f"], res["g"]
        pi_y, sig, klv, err = cnt_reductions(f, g, cost, x, a, y, b, res["eps_eff"])
        new_gamma = x.T @ pi_y
        obj = const + 8.0 * (-float((new_gamma**2).sum()) + (eps / 8.0) * klv - 2.0 * sig)
        delta = float(np.linalg.norm(new_gamma - gamma))
        state.update(zbar=zb, eps_eff=res["eps_eff"], f=f, g=g)
        gamma = new_gamma
        for key, val in (("objective", obj), ("gamma_delta", delta),
                         ("marginal_err", err), ("inner_iters", res["iterations"])):
            trace[key].append(val)
        return obj

    prev, ups, converged = None, 0, False
    for _ in range(max_outer):
        obj = step()
        if prev is not None:
            change = prev - obj
            if abs(change) < delta_outer:
                converged = True
                break
            if change < 0.0:
                ups += 1
                if ups >= 5:
                    raise RuntimeError("objective increased 5 outer steps in a row")
            else:
                ups = 0
        prev = obj
    if final_anneal is not None:
        step(anneal=final_anneal)
    return dict(gamma=gamma, f=state["f"], g=state["g"], zbar=state["zbar"], xbar=xbar,
                eps_eff=state["eps_eff"], trace=trace, value=trace["objective"][-1],
                converged=converged, constant=const)


def plan_argmax(f, g, cost, b, eps):
    """argmax_j pi_ij with numpy's first-max rule, and the top-2 log-score gap (nats).

    score_ij = log b_j + (g_j - C_ij)/eps (row constants dropped), SURVEY.md §7.3e.
    """
    lb = np.log(b) + g / eps
    n = cost.shape[0]
    idx = np.empty(n, dtype=np.int64)
    gap = np.empty(n)
    for i0 in range(0, n, BLOCK):
        i1 = min(i0 + BLOCK, n)
        s = lb[None, :] - cost.rows(i0, i1) / eps
        j = np.argmax(s, axis=1)
        idx[i0:i1] = j
        top = s[np.arange(i1 - i0), j]
        s[np.arange(i1 - i0), j] = -np.inf
        gap[i0:i1] = top - s.max(axis=1) if s.shape[1] > 1 else np.inf
    return idx, gap


def default_threads():
    return max(1, os.cpu_count() or 1)


__all__ = [
    "SqEuclid", "Dense", "LowRank", "softmin", "weighted_gap", "plan_blocks", "marginals",
    "marginal_error", "kl", "sinkhorn", "center", "fourth_moment", "constant", "augment",
    "zbar_of", "cnt_reductions", "solve_cnt_gw", "plan_argmax", "default_threads", "math",
]
