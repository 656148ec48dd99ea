"""CNT-GW outer solver on the GPU (reference ``solvers.py``).

Public surface kept from the reference: ``EgwConfig`` / ``make_config``
(solvers.py:44-110), ``SolveTrace`` (:113-151), ``EgwResult`` (:154-172),
``SolverError`` (:40), ``random_gamma`` (:183), ``gamma_step`` (:190),
``pi_step`` (:199), ``egw_objective`` (:259), ``solve_cnt_gw`` (:628) and
``solve_adaptive`` (:652, feature-space solver only).

One outer step (``_GwDevice.step``) is, entirely on the device:
  K5  operator application  -> dot features for Gamma_t (E-side projection
                               X_i.Gamma Y_j = (Gamma^T X_i).Y_j when D > E)
  K1-K3 Sinkhorn loop at eps/8 with carried interaction potentials
  K2  column tentative (only when the loop did not already produce it)
  K4  fused plan pass: row masses, pi Y, pi s, argmax
  K7  fp64 row/column reductions -> Gamma_{t+1}, KL terms, Err(pi)
followed by one small device->host read of the reduced scalars (the stop rule
and divergence guard of solvers.py:579-612 run on the host, as in the
reference). The objective uses the potentials identity:
  sum pi (f + g - C) = sum f~ r + sum g~ c + 2<Gamma_t, Gamma_{t+1}> - sum s^2 r
                       - sum t^2 c + 2 sigma_ss
with f~ = f - |X_i|^2 and g~ = g - |Gamma Y_j|^2 carried on device.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

import torch.distributed as tdist

from . import dist, divergence, engine
from ._native import F32, F32C, F64, F64S, LIB, call
from .measures import DenseCoupling, ImplicitCoupling
from .sinkhorn import SinkhornConfig, SquaredEuclideanCost, sinkhorn

MAX_DENSE_ENTRIES = 25_000_000
ADAPTIVE_CAP = 2**14
_DIVERGENCE_PATIENCE = 5
INIT_KINDS = ("product", "random", "gamma", "coupling", "landmarks")


class SolverError(RuntimeError):
    """An outer solve failed (divergence, budget cap, degenerate state)."""


@dataclass(frozen=True)
class EgwConfig:
    """Outer-loop configuration (reference solvers.py:44-94)."""

    eps: float
    inner: SinkhornConfig
    max_outer: int = 200
    delta_outer: float = 1e-5
    init: str = "product"
    init_gamma: np.ndarray | None = field(default=None, repr=False)
    init_coupling: np.ndarray | None = field(default=None, repr=False)
    init_pairs: np.ndarray | None = field(default=None, repr=False)
    init_scale: float = 1.0
    seed: int = 0
    final_anneal: float | None = None
    record_iterates: bool = False
    max_dense_entries: int = MAX_DENSE_ENTRIES
    feasibility_tol: float = 1e-4

    def __post_init__(self):
        checks = (
            (self.eps > 0.0 and np.isfinite(self.eps), f"eps must be positive and finite, got {self.eps!r}"),
            (self.max_outer >= 1, f"max_outer must be >= 1, got {self.max_outer!r}"),
            (self.delta_outer > 0.0, f"delta_outer must be positive, got {self.delta_outer!r}"),
            (self.init in INIT_KINDS, f"init must be one of {INIT_KINDS}, got {self.init!r}"),
            (not (self.init == "gamma" and self.init_gamma is None), "init='gamma' needs init_gamma"),
            (not (self.init == "coupling" and self.init_coupling is None),
             "init='coupling' needs init_coupling"),
            (not (self.init == "landmarks" and self.init_pairs is None),
             "init='landmarks' needs init_pairs"),
            (self.final_anneal is None or self.final_anneal > 0.0,
             f"final_anneal must be positive, got {self.final_anneal!r}"),
            (self.feasibility_tol > 0.0, f"feasibility_tol must be positive, got {self.feasibility_tol!r}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


def make_config(eps: float, *, mode: str = "symmetrized", n_inner: int | None = None,
                threshold: float | None = None, max_inner: int = 10000, **kwargs) -> EgwConfig:
    """Bundle the inner Sinkhorn configuration (reference solvers.py:97-110)."""
    inner = SinkhornConfig(eps=eps, mode=mode, n_inner=n_inner, threshold=threshold,
                           max_inner=max_inner)
    return EgwConfig(eps=eps, inner=inner, **kwargs)


_TRACE_COLS = ("steps", "objectives", "gamma_deltas", "marginal_errs", "inner_iters", "elapsed_s")


@dataclass
class SolveTrace:
    """Per-outer-step log with the reference's CSV columns (solvers.py:113-151)."""

    steps: list = field(default_factory=list)
    objectives: list = field(default_factory=list)
    gamma_deltas: list = field(default_factory=list)
    marginal_errs: list = field(default_factory=list)
    inner_iters: list = field(default_factory=list)
    elapsed_s: list = field(default_factory=list)

    def append(self, step, objective, gamma_delta, marginal_err, inner, elapsed):
        vals = (int(step), float(objective), float(gamma_delta), float(marginal_err), int(inner),
                float(elapsed))
        for col, v in zip(_TRACE_COLS, vals):
            getattr(self, col).append(v)

    def __len__(self):
        return len(self.steps)

    def to_csv(self, path, header=None) -> None:
        lines = [f"# {ln}" for ln in str(header).splitlines()] if header else []
        lines.append("step,objective,gamma_delta,marginal_err,inner_iters,elapsed_s")
        for s, o, d, e, k, t in zip(*(getattr(self, c) for c in _TRACE_COLS)):
            lines.append(f"{s},{o:.17g},{d:.17g},{e:.17g},{k},{t:.6f}")
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(lines) + "\n")


@dataclass
class EgwResult:
    """Outcome of an outer solve (solvers.py:154-172); ``argmax`` is the new
    per-row argmax_j pi_ij of the returned coupling (lowest j on ties)."""

    gamma: np.ndarray | None
    coupling: object
    trace: SolveTrace
    value: float
    converged: bool
    iterates: list | None = None
    schedule: list | None = None
    coarse: "EgwResult | None" = None
    argmax: np.ndarray | None = None


@dataclass
class _StepStats:
    objective: float
    gamma_delta: float
    marginal_err: float
    inner_iters: int


def random_gamma(src, tgt, rng, scale: float = 1.0) -> np.ndarray:
    """Gaussian operator at the canonical scale (solvers.py:183-187)."""
    d, e = src.features.shape[1], tgt.features.shape[1]
    tx = float(src.weights @ np.einsum("ij,ij->i", src.features, src.features))
    ty = float(tgt.weights @ np.einsum("ij,ij->i", tgt.features, tgt.features))
    return rng.standard_normal((d, e)) * (math.sqrt(tx * ty / (d * e)) * scale)


def _half_sq(measure) -> np.ndarray:
    h = getattr(measure, "half_sq_norms", None)
    return 0.5 * np.einsum("ij,ij->i", measure.features, measure.features) if h is None else h


def _stream():
    return torch.cuda.current_stream().cuda_stream


class _GwDevice:
    """Device buffers and kernels of the feature-space CNT-GW step.

    With torch.distributed initialised at world size > 1 the source rows are
    sharded (dist.py): this rank holds rows [lo, hi) of X, f and the plan
    reductions; Y, g and Gamma are replicated; the g-update and the row
    reductions go through NCCL all-reduces.
    """

    def __init__(self, src, tgt, device, info=None):
        self.device = device
        self.info = info if info is not None else dist.DistInfo()
        x = np.asarray(src.features, dtype=np.float64)
        y = np.asarray(tgt.features, dtype=np.float64)
        self.n_total = x.shape[0]
        self.comm = None
        # CNTGW_FORCE_SHARDED=1 runs the sharded code path at world size 1 (a
        # single-rank native NCCL communicator): the same captured collectives
        # as a multi-GPU solve, on one GPU
        forced = os.environ.get("CNTGW_FORCE_SHARDED", "0") == "1"
        if self.info.enabled or forced:
            native = dist.NativeComm(self.info) if (dist.native_comm_wanted() or not self.info.enabled) \
                else None
            spans = [dist.shard_range(self.n_total, r, self.info.world) for r in range(self.info.world)]
            self.comm = dist.RowShardComm(self.info, native=native,
                                          n_rows_max=max(h - l for l, h in spans))
        self.lo, self.hi = dist.shard_range(self.n_total, self.info.rank, self.info.world)
        x = x[self.lo:self.hi]
        self.n, self.d = x.shape
        self.m, self.e = y.shape
        self.x = engine.to_dev64(x, device)
        self.y = engine.to_dev64(y, device)
        self.sx = engine.to_dev64(_half_sq(src)[self.lo:self.hi], device)
        self.ty = engine.to_dev64(_half_sq(tgt), device)
        self.a = engine.to_dev64(np.asarray(src.weights)[self.lo:self.hi], device)
        self.b = engine.to_dev64(tgt.weights, device)
        self.proj_rows = self.d > self.e  # E-side projection
        self.k = min(self.d, self.e)
        self.kd = engine.padded_kd(self.k)
        if self.proj_rows:
            rows_feat = torch.zeros(self.n, self.kd, dtype=torch.float64, device=device)
            cols_feat = engine.to_dev64(y, device, self.kd)
        else:
            rows_feat = engine.to_dev64(x, device, self.kd)
            cols_feat = torch.zeros(self.m, self.kd, dtype=torch.float64, device=device)
        # locality orders of the point clouds (CNTGW_F32C tiles); the Gamma-dependent
        # features stay coherent along them (|Gamma dY| <= |Gamma| |dY|)
        self.src = engine.Side(rows_feat, self.sx, self.a, order=self._order(self.x, self.sx))
        self.tgt = engine.Side(cols_feat, self.ty, self.b, order=self._order(self.y, self.ty))
        # CNTGW_F64S visits the points in the squared-coordinate order while
        # Gamma = 0 (the cost is then a function of s_i - t_j) and in the
        # geometric order otherwise, switched on the device per loop (K5)
        self._orders = []
        for side in (self.src, self.tgt):
            cur = side.locality().clone()
            self._orders.append((torch.sort(side.sq64, stable=True).indices, side.locality(), cur))
            side.f64s_order = cur
        self.fwd = engine.HalfUpdate(self.src, self.tgt, True)
        self.bwd = engine.HalfUpdate(self.tgt, self.src, True)
        self.loop = engine.SinkhornLoop(self.fwd, self.bwd, self.a, self.b, device, comm=self.comm)
        if self.comm is not None:
            self.comm.prepare(self.m, self.loop.pr.numel(), device)
        # K4 / K7 buffers
        self.r = torch.empty(self.n, dtype=torch.float64, device=device)
        self.pi_y = torch.empty(self.n * self.e, dtype=torch.float64, device=device)
        self.pi_s = torch.empty(self.n, dtype=torch.float64, device=device)
        self.argmax = torch.empty(self.n, dtype=torch.int64, device=device)
        self.ws_plan = torch.empty(max(int(LIB.cntgw_plan_reduce_workspace(self.n, self.m, self.kd, self.e)),
                                       int(LIB.cntgw_plan_reduce_ctr_workspace(self.m, self.e))),
                                   dtype=torch.uint8, device=device)
        self.acc = torch.zeros(16 + self.d * self.e + 8, dtype=torch.float64, device=device)
        ows = max(int(LIB.cntgw_outer_reduce_workspace(self.n, self.d, self.e)),
                  int(LIB.cntgw_outer_reduce_workspace(self.m, 1, 1)))
        self.ws_outer = torch.empty(ows, dtype=torch.uint8, device=device)
        self.prec = F32

    @staticmethod
    def _order(pts: torch.Tensor, sq: torch.Tensor) -> torch.Tensor:
        """Locality order of a point cloud for the block-sparse paths: Morton
        codes of low-dimensional points (CNTGW_F32C tiles; the Gamma-dependent
        features stay coherent along them, |Gamma dY| <= |Gamma| |dY|), a
        k-means order by (cluster, s) above (CNTGW_F64S)."""
        mode = os.environ.get("CNTGW_ORDER", "auto")
        if mode == "morton" or (mode == "auto" and pts.shape[1] <= 3) or pts.shape[1] > 64:
            return engine.locality_order(pts)
        if pts.shape[1] not in (4, 8, 16, 32, 64):  # the k-means kernels' widths
            pts = torch.nn.functional.pad(pts, (0, engine.padded_kd(pts.shape[1]) - pts.shape[1]))
            if pts.shape[1] < 4:
                pts = torch.nn.functional.pad(pts, (0, 4 - pts.shape[1]))
        return engine.cluster_order(pts.contiguous(), sq)

    # -- K5 -----------------------------------------------------------------
    def set_gamma(self, gamma: np.ndarray):
        g = torch.as_tensor(np.ascontiguousarray(gamma, dtype=np.float64), device=self.device)
        if self.proj_rows:  # rows: Gamma^T X_i  (op = Gamma^T, E x D)
            op, side, feat, count, din, dout = g.t().contiguous(), self.src, self.x, self.n, self.d, self.e
        else:  # cols: Gamma Y_j  (op = Gamma, D x E)
            op, side, feat, count, din, dout = g.contiguous(), self.tgt, self.y, self.m, self.e, self.d
        self._op = op  # keep alive until the launch completes
        call("cntgw_apply_operator", op.data_ptr(), dout, din, feat.data_ptr(), din, count,
             side.feat64.data_ptr(), 0, self.kd, _stream())
        side.refresh32()
        self._gamma_h = g  # (alive until the launch completes)
        self._select_orders(g)

    def _select_orders(self, gamma_dev: torch.Tensor):
        self.loop.unhoist_rows()  # new features (and maybe a new order): the rows blocks are stale
        for sq_order, geo, cur in self._orders:
            call("cntgw_select_order", gamma_dev.data_ptr(), self.d * self.e, sq_order.data_ptr(),
                 geo.data_ptr(), cur.numel(), cur.data_ptr(), _stream())

    def set_gamma_dev(self, gamma_dev: torch.Tensor, gamma_t: torch.Tensor):
        """K5 from a device-resident Gamma (d*e fp64); graph-capturable (no
        allocation: ``gamma_t`` is a preallocated e x d buffer)."""
        if self.proj_rows:  # rows: Gamma^T X_i
            gamma_t.copy_(gamma_dev.view(self.d, self.e).t())
            op, side, feat, count, din, dout = gamma_t, self.src, self.x, self.n, self.d, self.e
        else:  # cols: Gamma Y_j
            op, side, feat, count, din, dout = gamma_dev, self.tgt, self.y, self.m, self.e, self.d
        call("cntgw_apply_operator", op.data_ptr(), dout, din, feat.data_ptr(), din, count,
             side.feat64.data_ptr(), 0, self.kd, _stream())
        side.refresh32()
        self._select_orders(gamma_dev)

    def plan_pass(self, f, g):
        """K4 for the final pair: r, pi Y, pi t and argmax per (local) row.

        On the centred path (CNTGW_F32C) the pass reuses the f-half-update's
        block-sparse plan (cntgw_plan_reduce_ctr: rows and columns in locality
        order, tiles that cannot hold a term within 2^-64 of a row's maximum
        skipped), on CNTGW_F64S its measured plan (cntgw_plan_reduce_f64s)
        while it holds; otherwise it is the dense fp64 pass (cntgw_plan_reduce).
        CNTGW_K4_SPARSE=0 forces the dense pass."""
        st = self.loop.state
        stream = _stream()
        fwd = self.fwd
        if self.prec == F32C and os.environ.get("CNTGW_K4_SPARSE", "1") != "0":
            src = self.src
            call("cntgw_prep_rows_ctr", fwd.kd, 1, src.feat64.data_ptr(), fwd.kd, src.sq64.data_ptr(),
                 src.locality().data_ptr(), src.n, fwd.ctr_rows.data_ptr(), stream)
            fwd.pack(st, g, prec=F32C)
            call("cntgw_plan_reduce_ctr", st.ptr, fwd.kd, 1, self.e, fwd.ctr_rows.data_ptr(),
                 fwd.ctr_cols.data_ptr(), self.tgt.locality().data_ptr(), src.feat64.data_ptr(),
                 fwd.kd, self.sx.data_ptr(), f.data_ptr(), src.log2w.data_ptr(), self.y.data_ptr(),
                 self.e, self.ty.data_ptr(), self.n, self.m, self.r.data_ptr(), self.pi_y.data_ptr(),
                 self.pi_s.data_ptr(), self.argmax.data_ptr(), fwd.ws.data_ptr(), fwd.ws.numel(),
                 self.ws_plan.data_ptr(), self.ws_plan.numel(), stream)
            return
        if self.prec == F64S and os.environ.get("CNTGW_K4_SPARSE", "1") != "0":
            src = self.src
            call("cntgw_prep_rows_f64s", fwd.kd, 1, src.feat64.data_ptr(), fwd.kd, src.sq64.data_ptr(),
                 src.plan_order().data_ptr(), src.n, fwd.f64s_rows.data_ptr(), stream)
            fwd.pack(st, g, prec=F64S)
            call("cntgw_plan_reduce_f64s", st.ptr, fwd.kd, 1, self.e, fwd.f64s_rows.data_ptr(),
                 fwd.rec.data_ptr(), self.tgt.plan_order().data_ptr(), src.feat64.data_ptr(), fwd.kd,
                 self.sx.data_ptr(), f.data_ptr(), src.log2w.data_ptr(), self.y.data_ptr(), self.e,
                 self.ty.data_ptr(), self.n, self.m, self.r.data_ptr(), self.pi_y.data_ptr(),
                 self.pi_s.data_ptr(), self.argmax.data_ptr(), fwd.ws.data_ptr(), fwd.ws.numel(),
                 self.ws_plan.data_ptr(), self.ws_plan.numel(), stream)
            return
        fwd.pack(st, g, prec=F64)
        call("cntgw_plan_reduce", st.ptr, self.kd, self.e, self.src.feat64.data_ptr(), self.kd,
             self.sx.data_ptr(), f.data_ptr(), self.src.log2w.data_ptr(), fwd.rec.data_ptr(),
             self.y.data_ptr(), self.e, self.ty.data_ptr(), self.n, self.m, self.r.data_ptr(),
             self.pi_y.data_ptr(), self.pi_s.data_ptr(), self.argmax.data_ptr(),
             self.ws_plan.data_ptr(), self.ws_plan.numel(), stream)

    def reductions(self, f, g, skip_g: int):
        """K2 tentative (skipped after a symmetrized threshold break), K4, K7."""
        st = self.loop.state
        self.loop.tentatives_g(f, skip=skip_g)
        self.plan_pass(f, g)
        stream = _stream()
        nrow = 16 + self.d * self.e
        call("cntgw_outer_reduce_rows", self.x.data_ptr(), self.d, self.d, self.pi_y.data_ptr(),
             self.e, self.r.data_ptr(), self.pi_s.data_ptr(), f.data_ptr(), self.sx.data_ptr(),
             self.a.data_ptr(), self.n, self.acc.data_ptr(), self.ws_outer.data_ptr(),
             self.ws_outer.numel(), stream)
        if self.comm is not None:  # row-side sums and Gamma_{t+1} over all shards
            self.comm.allreduce_(self.acc[:nrow])
        call("cntgw_outer_reduce_cols", st.ptr, g.data_ptr(), self.loop.gt.data_ptr(),
             self.ty.data_ptr(), self.b.data_ptr(), self.m, self.acc[nrow:].data_ptr(),
             self.ws_outer.data_ptr(), self.ws_outer.numel(), stream)
        return nrow

    def col_sep(self, gamma) -> torch.Tensor:
        """|Gamma Y_j|^2 in fp64 (reference separable column part)."""
        g = torch.as_tensor(np.ascontiguousarray(gamma, dtype=np.float64), device=self.device)
        return ((self.y @ g.t()) ** 2).sum(1)

    def row_sep(self) -> torch.Tensor:
        return (self.x ** 2).sum(1)

    def gather_rows(self, t: torch.Tensor) -> torch.Tensor:
        """Full-length copy of a row-sharded vector (all ranks)."""
        if self.info.world == 1:
            return t
        sizes = [dist.shard_range(self.n_total, r, self.info.world) for r in range(self.info.world)]
        width = max(h - l for l, h in sizes)
        buf = torch.zeros(width, dtype=t.dtype, device=t.device)
        buf[: t.numel()] = t
        parts = [torch.empty_like(buf) for _ in sizes]
        tdist.all_gather(parts, buf)
        return torch.cat([p[: h - l] for p, (l, h) in zip(parts, sizes)])

    def choose_precision(self, f, g, eps_min, reachable: bool = False):
        """Pick the half-update path from the exponent scale of the current
        operator, or — ``reachable`` — of every operator the solve can reach
        (the graph-captured solve fixes its path for all outer steps)."""
        fmax = f.abs().max()
        if self.comm is not None:
            self.comm.allmax_(fmax)
        pot = float(torch.maximum(fmax, g.abs().max()))
        if reachable:
            scale = self.reachable_scale(eps_min, pot)
        else:
            scale = engine.exponent_scale(eps_min, self.src.feat64, self.sx, self.tgt.feat64, self.ty, pot)
        self.prec = engine.choose_precision(
            scale, self.kd, True, ctr_deferred=lambda: self._ctr_deferred(eps_min),
            pairs=float(self.n_total) * float(self.m))
        self.loop.set_precision(self.prec)

    def reachable_scale(self, eps: float, pot_abs: float) -> float:
        """Upper bound of the exponent scale over every reachable operator.

        Gamma_{t+1} = X^T pi Y with pi >= 0 of marginals (a, b), so by
        Cauchy-Schwarz ||Gamma||_2 <= ||Gamma||_F <= sqrt(T_x T_y), T = sum
        w |x|^2; the dot term 2 |<x_i, z_j>| of any step is at most
        2 sqrt(T_x T_y) max|X| max|Y|, and at a Sinkhorn fixed point the
        interaction potentials are bounded by the interaction cost, |f~|,
        |g~| <~ dot + sq."""
        lam = math.log2(math.e) / eps
        tx = (self.a * (self.x * self.x).sum(1)).sum().reshape(1)
        xm = torch.stack([(self.x * self.x).sum(1).max().sqrt(), self.sx.abs().max()])
        if self.comm is not None:  # every rank must take the same path
            self.comm.allreduce_(tx)
            self.comm.allmax_(xm)
        ty = float((self.b * (self.y * self.y).sum(1)).sum())
        ym = float((self.y * self.y).sum(1).max().sqrt())
        dot = 2.0 * math.sqrt(max(float(tx), 0.0) * max(ty, 0.0)) * float(xm[0]) * ym
        sq = (float(xm[1]) + float(self.ty.abs().max())) ** 2
        return lam * (max(pot_abs, dot + sq) + dot + sq)

    def _ctr_deferred(self, eps_min):
        if float(self.n_total) * float(self.m) < engine.CTR_MIN_PAIRS:
            return 1.0
        s = max(engine.centred_deferred_fraction(eps_min, self.src, self.tgt),
                engine.centred_deferred_fraction(eps_min, self.tgt, self.src))
        if self.comm is not None:  # every rank must pick the same path
            t = torch.tensor([s], dtype=torch.float64, device=self.device)
            self.comm.allmax_(t)
            s = float(t)
        return s

    # -- one outer step ------------------------------------------------------
    def step(self, f, g, gamma: np.ndarray, loop_cfg: engine.LoopConfig, eps_outer: float,
             const: float, use_graph: bool):
        self.set_gamma(gamma)
        self.choose_precision(f, g, loop_cfg.eps)
        self.loop.hoist_rows()
        stats = self.loop.run(f, g, loop_cfg, use_graph=use_graph)
        # g-tentative (skipped on the device after a symmetrized threshold
        # break, whose tentatives are already the final ones), K4, K7
        nrow = self.reductions(f, g, skip_g=2)
        acc = self.acc.cpu().numpy()  # the one host read per outer step
        rows, cols = acc[:16], acc[nrow:]
        gamma_next = acc[16:nrow].reshape(self.d, self.e).copy()
        sigma_ss = rows[3]
        cross = float((gamma * gamma_next).sum())
        plan_lin = rows[0] + cols[0] + 2.0 * cross - rows[1] - cols[1] + 2.0 * sigma_ss
        kl = plan_lin / stats.eps_eff
        objective = const + 8.0 * (-float((gamma_next**2).sum()) + (eps_outer / 8.0) * kl
                                   - 2.0 * sigma_ss)
        err = rows[2] + cols[2]
        delta = float(np.linalg.norm(gamma_next - gamma))
        return gamma_next, _StepStats(objective, delta, err, stats.iterations), stats


def _initial_gamma(src, tgt, cfg: EgwConfig) -> np.ndarray:
    """Gamma_0 for each init kind (reference solvers.py:353-381)."""
    x, y = np.asarray(src.features), np.asarray(tgt.features)
    d, e = x.shape[1], y.shape[1]
    if cfg.init == "product":
        return np.zeros((d, e))
    if cfg.init == "random":
        return random_gamma(src, tgt, np.random.default_rng(cfg.seed), cfg.init_scale)
    if cfg.init == "gamma":
        gamma = np.asarray(cfg.init_gamma, dtype=np.float64)
        if gamma.shape != (d, e):
            raise ValueError(f"init_gamma shape {gamma.shape} does not match ({d}, {e})")
        return np.array(gamma)
    if cfg.init == "coupling":
        pi = np.asarray(getattr(cfg.init_coupling, "matrix", cfg.init_coupling), dtype=np.float64)
        if pi.shape != (x.shape[0], y.shape[0]):
            raise ValueError(f"init_coupling shape {pi.shape} does not match ({x.shape[0]}, {y.shape[0]})")
        dev = engine.require_cuda()
        xt = torch.as_tensor(x, device=dev)
        out = xt.t() @ (torch.as_tensor(pi, device=dev) @ torch.as_tensor(y, device=dev))
        return out.cpu().numpy()
    pairs = np.asarray(cfg.init_pairs)
    if pairs.ndim != 2 or pairs.shape[1] != 2:
        raise ValueError("init_pairs must be an array of (source, target) index pairs")
    gamma = np.zeros((d, e))
    for i, j in pairs:
        if not (0 <= i < x.shape[0] and 0 <= j < y.shape[0]):
            raise ValueError(f"landmark pair ({i}, {j}) out of range")
        gamma += np.outer(x[int(i)], y[int(j)])
    return gamma


class _CntGwState:
    """Feature-space alternate minimisation with device-resident plans
    (reference solvers.py:285-350)."""

    def __init__(self, src, tgt, cfg: EgwConfig, warm_potentials=None):
        self.src, self.tgt, self.cfg = src, tgt, cfg
        n, m = src.features.shape[0], tgt.features.shape[0]
        if cfg.record_iterates and n * m > cfg.max_dense_entries:
            raise ValueError(
                f"recording iterates would densify {n * m} entries per step, "
                f"beyond the memory guard ({cfg.max_dense_entries})"
            )
        self.device = engine.require_cuda()
        info = dist.DistInfo()
        if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
            info = dist.DistInfo(rank=tdist.get_rank(), world=tdist.get_world_size(),
                                 local_rank=self.device.index)
        self.dev = _GwDevice(src, tgt, self.device, info)
        self.gamma = _initial_gamma(src, tgt, cfg)
        if warm_potentials is None:
            # interaction potentials 0 (solvers.py:297-301): f~ = s^2, g~ = t^2
            self.f = self.dev.sx ** 2
            self.g = self.dev.ty ** 2
        else:
            f0 = np.asarray(warm_potentials[0], dtype=np.float64)[self.dev.lo:self.dev.hi]
            f0 = engine.to_dev64(f0, self.device)
            g0 = engine.to_dev64(np.asarray(warm_potentials[1], dtype=np.float64), self.device)
            self.f = f0 - self.dev.row_sep()
            self.g = g0 - self.dev.col_sep(self.gamma)
        mx = divergence.moments(np.asarray(src.features, dtype=np.float64),
                                np.asarray(src.weights, dtype=np.float64), self.device).cpu().numpy()
        my = divergence.moments(self.dev.y, self.dev.b, self.device).cpu().numpy()
        self.constant = divergence.constant_from_moments(mx, self.dev.d, my, self.dev.e)
        self.coupling_gamma = None
        self.eps_eff = None
        self.record = []
        comm = self.dev.comm
        self.use_graph = self.dev.n * self.dev.m <= (1 << 24) and (comm is None or comm.capturable)

    def step(self, inner_budget=None, anneal_from=None) -> _StepStats:
        inner = self.cfg.inner
        if inner_budget is not None:
            inner = replace(inner, n_inner=inner_budget, threshold=None)
        if anneal_from is not None:
            inner = replace(inner, anneal_from=anneal_from)
        loop_cfg = inner.with_temperature(self.cfg.eps / 8.0).loop_config()
        gamma_t = self.gamma
        gamma_next, stats, lstats = self.dev.step(self.f, self.g, gamma_t, loop_cfg, self.cfg.eps,
                                                   self.constant, self.use_graph)
        self.coupling_gamma = gamma_t
        self.eps_eff = lstats.eps_eff
        self.gamma = gamma_next
        if self.cfg.record_iterates:
            self.record.append(self.coupling().densify().matrix)
        return stats

    def coupling(self) -> ImplicitCoupling:
        """The last plan (built on Gamma_t, solvers.py:326-336) in reference form."""
        dev = self.dev
        gt = self.coupling_gamma
        f = dev.gather_rows(self.f + dev.row_sep()).cpu().numpy()
        g = (self.g + dev.col_sep(gt)).cpu().numpy()
        src, tgt = self.src, self.tgt
        xbar = np.column_stack([src.features, _half_sq(src)])
        zbar = np.column_stack([np.asarray(tgt.features) @ gt.T, _half_sq(tgt)])
        cp = ImplicitCoupling(f, g, SquaredEuclideanCost(xbar, zbar), src.weights, tgt.weights,
                              self.eps_eff, device=(self.f, self.g, dev))
        return cp

    def result(self, trace, converged, schedule=None) -> EgwResult:
        coupling = self.coupling() if self.coupling_gamma is not None else None
        return EgwResult(
            gamma=self.gamma, coupling=coupling, trace=trace,
            value=trace.objectives[-1] if len(trace) else math.nan, converged=converged,
            iterates=self.record if self.cfg.record_iterates else None, schedule=schedule,
            argmax=self.dev.gather_rows(self.dev.argmax).cpu().numpy() if coupling is not None else None,
        )


class _DeviceSolve:
    """The whole outer loop as ONE CUDA graph (single GPU).

    Captured once: an outer conditional WHILE node whose body is K5 (operator
    from the device-resident Gamma), the Sinkhorn loop (n_inner sweeps, or an
    inner conditional WHILE node that exits on the device-side threshold
    decision), the final tentative, K4/K7 and ``cntgw_outer_finish`` (objective,
    trace row, stop rule and divergence guard on the device), which sets the
    outer condition. The host launches it once and reads the trace at the end.
    """

    def __init__(self, state: "_CntGwState"):
        import ctypes

        from ._native import OuterStateStruct

        self.state = state
        dev, cfg = state.dev, state.cfg
        self.loop_cfg = cfg.inner.with_temperature(cfg.eps / 8.0).loop_config()
        device = state.device
        self.gamma = torch.as_tensor(np.ascontiguousarray(state.gamma).ravel(), device=device).clone()
        self.gamma_prev = torch.zeros_like(self.gamma)
        self.gamma_t = torch.zeros(dev.e * dev.d, dtype=torch.float64, device=device)
        self.trace = torch.zeros(5 * cfg.max_outer, dtype=torch.float64, device=device)
        self.os = torch.zeros(ctypes.sizeof(OuterStateStruct), dtype=torch.uint8, device=device)
        self._struct = OuterStateStruct
        # features and precision for the first step, fixed for the captured solve
        dev.set_gamma(state.gamma)
        # one path for the whole captured solve: safe for every reachable Gamma
        dev.choose_precision(state.f, state.g, self.loop_cfg.eps, reachable=True)
        self.exec = None

    def _capture(self):
        st, dev, cfg, lc = self.state, self.state.dev, self.state.cfg, self.loop_cfg
        loop = dev.loop
        s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        s0.wait_stream(torch.cuda.current_stream())
        import ctypes

        h1, h2 = ctypes.c_uint64(0), ctypes.c_uint64(0)
        done_sweep = loop.state.ptr + _native_offset("done")
        done_outer = self.os.data_ptr() + self._struct.done.offset
        with torch.cuda.stream(s0):
            call("cntgw_graph_begin", s0.cuda_stream)
            call("cntgw_outer_init", self.os.data_ptr(), float(st.constant), float(cfg.eps),
                 float(cfg.delta_outer), int(cfg.max_outer), s0.cuda_stream)
            call("cntgw_graph_while_begin", s0.cuda_stream, s1.cuda_stream, ctypes.byref(h1))
            with torch.cuda.stream(s1):
                dev.set_gamma_dev(self.gamma, self.gamma_t)
                loop.hoist_rows()
                loop.state.init(lc.eps, lc.anneal_from, lc.threshold, lc.max_sweeps, lc.mode)
                if lc.threshold is None:
                    for _ in range(lc.max_sweeps):
                        loop.sweep(st.f, st.g, lc.mode)
                else:
                    call("cntgw_graph_while_begin", s1.cuda_stream, s2.cuda_stream, ctypes.byref(h2))
                    with torch.cuda.stream(s2):
                        loop.sweep(st.f, st.g, lc.mode)
                        call("cntgw_graph_set_condition", h2.value, done_sweep, s2.cuda_stream)
                    call("cntgw_graph_while_end", s2.cuda_stream)
                loop.state.begin()  # a fully used budget is marked done
                nrow = dev.reductions(st.f, st.g, skip_g=2)
                call("cntgw_outer_finish", self.os.data_ptr(), loop.state.ptr, dev.acc.data_ptr(),
                     dev.acc[nrow:].data_ptr(), self.gamma.data_ptr(), self.gamma_prev.data_ptr(),
                     dev.d * dev.e, self.trace.data_ptr(), s1.cuda_stream)
                call("cntgw_graph_set_condition", h1.value, done_outer, s1.cuda_stream)
            call("cntgw_graph_while_end", s1.cuda_stream)
            exec_ptr = ctypes.c_void_p()
            call("cntgw_graph_end", s0.cuda_stream, ctypes.byref(exec_ptr))
        self.exec = exec_ptr.value
        self.stream = s0

    def run(self):
        """Launch the captured solve; returns (trace rows, converged, error)."""
        self._capture()
        try:
            call("cntgw_graph_launch", self.exec, self.stream.cuda_stream)
            self.stream.synchronize()
        finally:
            call("cntgw_graph_destroy", self.exec)
        torch.cuda.current_stream().wait_stream(self.stream)
        os_ = self._struct.from_buffer_copy(self.os.cpu().numpy().tobytes())
        rows = self.trace.view(-1, 5)[: os_.step].cpu().numpy()
        st, dev = self.state, self.state.dev
        st.gamma = self.gamma.view(dev.d, dev.e).cpu().numpy().copy()
        st.coupling_gamma = self.gamma_prev.view(dev.d, dev.e).cpu().numpy().copy()
        st.eps_eff = float(dev.loop.state.read().eps_n)
        return rows, bool(os_.converged), bool(os_.error)


def _native_offset(field: str) -> int:
    from ._native import SweepStateStruct

    return getattr(SweepStateStruct, field).offset


def _run_outer_device(state, cfg: EgwConfig) -> EgwResult:
    """Graph-captured outer loop (same semantics as _run_outer, single GPU)."""
    rows, converged, error = _DeviceSolve(state).run()
    if error:
        raise SolverError(
            f"objective increased {_DIVERGENCE_PATIENCE} outer steps in a "
            "row; raise n_inner or use the adaptive wrapper"
        )
    trace = SolveTrace()
    for k, (obj, delta, err, iters, t) in enumerate(rows, start=1):
        trace.append(k, obj, delta, err, int(iters), t)
    if cfg.final_anneal is not None:
        t0 = time.perf_counter()
        stats = state.step(anneal_from=cfg.final_anneal)
        last = trace.elapsed_s[-1] if len(trace) else 0.0
        trace.append(len(trace) + 1, stats.objective, stats.gamma_delta, stats.marginal_err,
                     stats.inner_iters, last + time.perf_counter() - t0)
    return state.result(trace, converged)


def _run_outer(state, cfg: EgwConfig, adaptive: bool = False) -> EgwResult:
    """Outer control: trace, |dobj| stop, 5-increase guard, adaptive doubling,
    optional final annealed step (reference solvers.py:556-625)."""
    trace = SolveTrace()
    start = time.perf_counter()
    prev, schedule, budget = None, [], None
    if adaptive:
        if cfg.inner.n_inner is None:
            raise ValueError("the adaptive wrapper needs a fixed-budget inner configuration")
        budget = cfg.inner.n_inner
    ups, converged = 0, False
    for k in range(1, cfg.max_outer + 1):
        stats = state.step(inner_budget=budget)
        schedule.append(budget if adaptive else stats.inner_iters)
        trace.append(k, stats.objective, stats.gamma_delta, stats.marginal_err, stats.inner_iters,
                     time.perf_counter() - start)
        if prev is not None:
            change = prev - stats.objective
            if abs(change) < cfg.delta_outer and not (adaptive and stats.marginal_err > cfg.feasibility_tol):
                converged = True
                prev = stats.objective
                break
            if change < 0.0:
                if adaptive:
                    budget *= 2
                    if budget > ADAPTIVE_CAP:
                        raise SolverError(
                            f"adaptive inner budget exceeded the cap ({ADAPTIVE_CAP}); "
                            "the objective keeps increasing, likely a non-CNT cost or "
                            "a temperature too small for this instance"
                        )
                    prev = stats.objective
                    continue
                ups += 1
                if ups >= _DIVERGENCE_PATIENCE:
                    raise SolverError(
                        f"objective increased {_DIVERGENCE_PATIENCE} outer steps in a "
                        "row; raise n_inner or use the adaptive wrapper"
                    )
            else:
                ups = 0
        prev = stats.objective
    if cfg.final_anneal is not None:
        stats = state.step(inner_budget=budget, anneal_from=cfg.final_anneal)
        trace.append(len(trace) + 1, stats.objective, stats.gamma_delta, stats.marginal_err,
                     stats.inner_iters, time.perf_counter() - start)
        if adaptive:
            schedule.append(budget)
    return state.result(trace, converged, schedule=schedule if adaptive else None)


def solve_cnt_gw(src, tgt, cfg: EgwConfig, _warm_potentials=None) -> EgwResult:
    """Feature-space EGW solve (reference solvers.py:628-632).

    The whole outer loop runs as a single CUDA graph (``_DeviceSolve``) on
    one GPU and on every rank of a row-sharded NCCL run (the exchanges are
    the library's own NCCL collectives, captured in the graph, dist.py);
    gloo-backed runs and ``record_iterates`` use the host-driven loop over the
    same device kernels. CNTGW_DEVICE_LOOP=0 forces the host-driven loop.
    """
    state = _CntGwState(src, tgt, cfg, warm_potentials=_warm_potentials)
    comm = state.dev.comm
    if ((comm is None or comm.capturable) and not cfg.record_iterates
            and os.environ.get("CNTGW_DEVICE_LOOP", "1") != "0"):
        return _run_outer_device(state, cfg)
    return _run_outer(state, cfg)


def solve_adaptive(solver, *args, cfg: EgwConfig) -> EgwResult:
    """Inner-budget doubling wrapper (reference solvers.py:652-665) around
    solve_cnt_gw, solve_kernel_gw or solve_entropic_gw."""
    from .dense_solvers import _EntropicGwState, _KernelGwState, solve_entropic_gw, solve_kernel_gw

    states = {solve_cnt_gw: _CntGwState, solve_kernel_gw: _KernelGwState,
              solve_entropic_gw: _EntropicGwState}
    try:
        state_cls = states[solver]
    except (TypeError, KeyError):
        raise ValueError("solver must be one of the solve_* functions of this module") from None
    return _run_outer(state_cls(*args, cfg), cfg, adaptive=True)


# ---------------------------------------------------------------------------
# building blocks exposed by the reference API
# ---------------------------------------------------------------------------
def pi_step(gamma, src, tgt, eps: float, inner: SinkhornConfig):
    """Plan update: EOT between augmented features at eps/8 (solvers.py:199-224)."""
    zbar = np.column_stack([np.asarray(tgt.features) @ np.asarray(gamma).T, _half_sq(tgt)])
    xbar = np.column_stack([src.features, _half_sq(src)])
    cost = SquaredEuclideanCost(xbar, zbar)
    if inner.warm_start is None:
        inner = inner.with_warm_start((xbar**2).sum(axis=1), (zbar**2).sum(axis=1))
    return sinkhorn(src.weights, tgt.weights, cost, inner.with_temperature(eps / 8.0))


def _plan_pass(coupling, src, tgt, transpose: bool = False):
    """Fused K4 pass over an ImplicitCoupling on a SquaredEuclideanCost
    (augmented features): returns device (r, pi Y, pi s_y, argmax) — or, with
    ``transpose``, the same pass over pi^T: (c, pi^T X, pi^T s_x, argmax_i),
    the column-side reductions of divergence._plan_reductions (plan.row_pass)."""
    from . import plan

    if not isinstance(coupling.cost, SquaredEuclideanCost):
        raise TypeError("fused plan reductions need a SquaredEuclideanCost coupling")
    dev = engine.require_cuda()
    form = plan.feature_form(coupling.cost, dev)
    f, g, a_w, b_w = plan._coupling_tensors(coupling, dev)
    f_t, g_t = f - form.row_sep, g - form.col_sep
    acc, acc_s = tgt.features, _half_sq(tgt)
    if transpose:
        form, f_t, g_t, a_w, b_w = form.transpose(), g_t, f_t, b_w, a_w
        acc, acc_s = src.features, _half_sq(src)
    e = np.asarray(acc).shape[1]
    # K4 accumulates at least as many features as it dots (padded widths)
    acc_d = engine.to_dev64(acc, dev, max(e, form.kd))
    r, pi_acc, pi_s, am = plan.row_pass(form, f_t, g_t, a_w, b_w, coupling.eps_eff, acc_d,
                                        engine.to_dev64(acc_s, dev))
    return r, pi_acc[:, :e].contiguous(), pi_s, am


def gamma_step(coupling, src, tgt) -> np.ndarray:
    """Gamma = X^T pi Y with the plan kept implicit (solvers.py:190-196)."""
    if isinstance(coupling, DenseCoupling):
        dev = engine.require_cuda()
        pi = torch.as_tensor(coupling.matrix, device=dev)
        xt = torch.as_tensor(np.asarray(src.features), device=dev)
        return (xt.t() @ (pi @ torch.as_tensor(np.asarray(tgt.features), device=dev))).cpu().numpy()
    _, pi_y, _, _ = _plan_pass(coupling, src, tgt)
    x = torch.as_tensor(np.asarray(src.features), device=pi_y.device)
    return (x.t() @ pi_y).cpu().numpy()


def egw_objective(gamma, coupling, src, tgt, eps: float) -> float:
    """C + 8 F(Gamma, pi) for any operator/plan pair (solvers.py:259-282)."""
    from .measures import kl_divergence

    gamma = np.asarray(gamma, dtype=np.float64)
    if isinstance(coupling, ImplicitCoupling):
        # _cnt_reductions (solvers.py:227-256) as device passes: pi Y and pi s_y
        # from K4, KL from the potentials identity (plan.plan_sums)
        r, pi_y, pi_s, _ = _plan_pass(coupling, src, tgt)
        x = torch.as_tensor(np.array(src.features, dtype=np.float64), device=pi_y.device)
        xt_pi_y = (x.t() @ pi_y).cpu().numpy()
        sigma_ss = float((torch.as_tensor(_half_sq(src), device=pi_y.device) * pi_s).sum())
        kl = kl_divergence(coupling)
    else:
        pi = coupling.matrix
        xt_pi_y = np.asarray(src.features).T @ (pi @ np.asarray(tgt.features))
        sigma_ss = float(_half_sq(src) @ pi @ _half_sq(tgt))
        kl = kl_divergence(coupling)
    cross = float((gamma * xt_pi_y).sum()) + sigma_ss
    const = divergence.constant_value(src, tgt)
    return const + 8.0 * (float((gamma**2).sum()) + (eps / 8.0) * kl - 2.0 * cross)


# multiscale front end (reference solvers.py:668-763), device k-means
from .multiscale import _weighted_kmeans, coarsen, solve_multiscale  # noqa: E402,F401
# dense-plan baselines (reference solvers.py:384-553, 629-638)
from .dense_solvers import solve_entropic_gw, solve_kernel_gw  # noqa: E402,F401
