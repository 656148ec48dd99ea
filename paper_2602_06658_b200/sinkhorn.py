"""Drop-in ``sinkhorn`` entry point and cost providers (reference ``sinkhorn.py``).

Same public surface as the reference module: ``SinkhornConfig`` (validation
of sinkhorn.py:112-155), ``SinkhornResult`` (:158-163), the cost-provider
protocol (``shape``, ``rows``, ``transpose``, ``full``) with ``DenseCost`` and
``SquaredEuclideanCost``, and ``sinkhorn(a, b, cost, config)`` (:191-258).
The loop itself runs on the GPU (engine.py): both half-updates are the
streaming kernels of libcntgw_b200.so, the control logic is device-resident,
and only the final potentials come back to the host in float64.

Additionally ``SeparableLowRankCost`` (C_ij = a_i + b_j - 2 u_i.v_j) is the
provider of the C2 micro-benchmark; any other duck-typed
provider is materialised once (``full()``) and streamed by the dense kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import engine
from .measures import ImplicitCoupling, kl_divergence

CACHE_ENTRIES = 2**22
_GRAPH_MAX_PAIRS = 1 << 24  # below this size, sweep chunks are replayed as CUDA graphs
_DENSE_MAX_ENTRIES = 1 << 28


def _on_device(x) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64,
                           device=engine.require_cuda())


# ---------------------------------------------------------------------------
# cost providers
# ---------------------------------------------------------------------------
class DenseCost:
    """Explicit cost matrix (reference sinkhorn.py:30-56)."""

    def __init__(self, matrix):
        self._dev = None
        if isinstance(matrix, torch.Tensor):  # device-resident (dense GW baselines)
            if matrix.ndim != 2:
                raise ValueError("cost matrix must be 2-dimensional")
            if not bool(torch.isfinite(matrix).all()):
                raise ValueError("cost matrix contains non-finite entries")
            self._dev = matrix.to(torch.float64).contiguous()
            self._m = None
            self._shape = tuple(self._dev.shape)
            self._t = None
            return
        m = np.ascontiguousarray(matrix, dtype=np.float64)
        if m.ndim != 2:
            raise ValueError("cost matrix must be 2-dimensional")
        if not np.isfinite(m).all():
            raise ValueError("cost matrix contains non-finite entries")
        self._m = m
        self._shape = m.shape
        self._t = None

    shape = property(lambda self: self._shape)

    def _host(self):
        if self._m is None:
            self._m = self._dev.cpu().numpy()
        return self._m

    def rows(self, i0, i1):
        return self._host()[i0:i1]

    def _rows_dev(self, i0, i1, device):
        src = self._dev if self._dev is not None else self._m[i0:i1]
        if self._dev is not None:
            return src[i0:i1].to(device)
        return torch.as_tensor(np.ascontiguousarray(src), device=device)

    def full(self):
        return self._host()

    def transpose(self) -> "DenseCost":
        if self._t is None:
            self._t = DenseCost(self._dev.t() if self._dev is not None else self._m.T)
            self._t._t = self
        return self._t


class SquaredEuclideanCost:
    """|x_i - z_j|^2 between feature arrays (reference sinkhorn.py:59-109).

    Row blocks (off the hot path, e.g. for ``densify``) are evaluated on the
    GPU in float64 with the reference's clip at 0. The Sinkhorn kernels never
    read blocks: they rebuild costs from the features, treating the last
    coordinate as a squared difference (exact re-expression of the same cost,
    better conditioned when that coordinate is the large augmentation s).
    ``cache_entries`` is accepted for signature compatibility; caching is
    value-neutral in the reference (sinkhorn.py:87-93).
    """

    def __init__(self, x, z, cache_entries: int = CACHE_ENTRIES):
        self._x = np.ascontiguousarray(x, dtype=np.float64)
        self._z = np.ascontiguousarray(z, dtype=np.float64)
        if self._x.ndim != 2 or self._z.ndim != 2 or self._x.shape[1] != self._z.shape[1]:
            raise ValueError("coordinate arrays must be 2-d with a common feature dimension")
        self._cache_entries = int(cache_entries)
        self._t = None
        self._dev = None

    shape = property(lambda self: (self._x.shape[0], self._z.shape[0]))

    def _device(self):
        if self._dev is None:
            x, z = _on_device(self._x), _on_device(self._z)
            self._dev = (x, z, (x * x).sum(1), (z * z).sum(1))
        return self._dev

    def _rows_dev(self, i0, i1, device=None):
        x, z, sx, sz = self._device()
        blk = sx[i0:i1, None] + sz[None, :] - 2.0 * (x[i0:i1] @ z.T)
        return blk.clamp_min_(0.0)

    def rows(self, i0, i1):
        return self._rows_dev(i0, i1).cpu().numpy()

    def full(self):
        return self.rows(0, self.shape[0])

    def transpose(self) -> "SquaredEuclideanCost":
        if self._t is None:
            self._t = SquaredEuclideanCost(self._z, self._x, self._cache_entries)
            self._t._t = self
        return self._t


class SeparableLowRankCost:
    """C_ij = a_i + b_j - 2 u_i.v_j (no clip): the C2 micro-benchmark cost form."""

    def __init__(self, u, v, row_sep, col_sep):
        self._u = np.ascontiguousarray(u, dtype=np.float64)
        self._v = np.ascontiguousarray(v, dtype=np.float64)
        self._ra = np.ascontiguousarray(row_sep, dtype=np.float64)
        self._cb = np.ascontiguousarray(col_sep, dtype=np.float64)
        n, k = self._u.shape
        m, k2 = self._v.shape
        if k != k2 or self._ra.shape != (n,) or self._cb.shape != (m,):
            raise ValueError("low-rank factors and separable terms have inconsistent shapes")
        self._t = None

    shape = property(lambda self: (self._u.shape[0], self._v.shape[0]))

    def _rows_dev(self, i0, i1, device=None):
        if getattr(self, "_dev", None) is None:
            self._dev = tuple(_on_device(t) for t in (self._u, self._v, self._ra, self._cb))
        u, v, ra, cb = self._dev
        return ra[i0:i1, None] + cb[None, :] - 2.0 * (u[i0:i1] @ v.T)

    def rows(self, i0, i1):
        return self._rows_dev(i0, i1).cpu().numpy()

    def full(self):
        return self.rows(0, self.shape[0])

    def transpose(self) -> "SeparableLowRankCost":
        if self._t is None:
            self._t = SeparableLowRankCost(self._v, self._u, self._cb, self._ra)
            self._t._t = self
        return self._t


# ---------------------------------------------------------------------------
# configuration / result (reference sinkhorn.py:112-163)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SinkhornConfig:
    """Inner-loop policy: fixed ``n_inner`` sweeps (default 100) xor a weighted
    ``threshold`` with a ``max_inner`` cap; optional sqrt annealing from
    ``anneal_from``; optional warm start (f, g)."""

    eps: float
    mode: str = "symmetrized"
    n_inner: int | None = None
    threshold: float | None = None
    max_inner: int = 10000
    anneal_from: float | None = None
    warm_start: tuple | None = None

    def __post_init__(self):
        if not (self.eps > 0.0 and np.isfinite(self.eps)):
            raise ValueError(f"eps must be positive and finite, got {self.eps!r}")
        if self.mode not in ("standard", "symmetrized"):
            raise ValueError(f"mode must be 'standard' or 'symmetrized', got {self.mode!r}")
        fixed, tau = self.n_inner, self.threshold
        if fixed is None and tau is None:
            object.__setattr__(self, "n_inner", 100)
            fixed = 100
        if fixed is not None and tau is not None:
            raise ValueError("exactly one of n_inner and threshold must be set")
        if fixed is not None and fixed < 1:
            raise ValueError(f"n_inner must be >= 1, got {fixed!r}")
        if tau is not None and not (tau > 0.0):
            raise ValueError(f"threshold must be positive, got {tau!r}")
        if tau is not None and self.max_inner < 1:
            raise ValueError(f"max_inner must be >= 1, got {self.max_inner!r}")
        if self.anneal_from is not None and not (self.anneal_from > 0.0):
            raise ValueError(f"anneal_from must be positive, got {self.anneal_from!r}")

    def with_temperature(self, eps: float) -> "SinkhornConfig":
        return replace(self, eps=eps)

    def with_warm_start(self, f, g) -> "SinkhornConfig":
        return replace(self, warm_start=(f, g))

    def loop_config(self) -> engine.LoopConfig:
        return engine.LoopConfig(eps=self.eps, mode=self.mode, n_inner=self.n_inner,
                                 threshold=self.threshold, max_inner=self.max_inner,
                                 anneal_from=self.anneal_from)


@dataclass
class SinkhornResult:
    coupling: ImplicitCoupling
    iterations: int
    marginal_err: float
    converged: bool


# ---------------------------------------------------------------------------
# device problems
# ---------------------------------------------------------------------------
@dataclass
class DeviceProblem:
    """Both half-update operators of one cost plus its separable parts (fp64)."""

    fwd: object
    bwd: object
    row_sep: np.ndarray
    col_sep: np.ndarray


def feature_problem(row_feat, row_sq, col_feat, col_sq, a, b, device) -> tuple:
    """Sides + operators for C = sep - 2<xf, zf> (+ (xs - zs)^2)."""
    k = row_feat.shape[1]
    kd = engine.padded_kd(max(k, 1))
    sq = row_sq is not None
    src = engine.Side.make(row_feat, row_sq, a, device, kd)
    tgt = engine.Side.make(col_feat, col_sq, b, device, kd)
    return src, tgt, engine.HalfUpdate(src, tgt, sq), engine.HalfUpdate(tgt, src, sq)


def _set_precision(problem, eps, f0, g0):
    """Pick fp32/fp64 exponent assembly from the problem's scales (engine.py)."""
    fwd = problem.fwd
    if not isinstance(fwd, engine.HalfUpdate):
        return
    pot = max(float(np.abs(f0 - problem.row_sep).max(initial=0.0)),
              float(np.abs(g0 - problem.col_sep).max(initial=0.0)))
    scale = engine.exponent_scale(eps, fwd.rows.feat64, fwd.rows.sq64, fwd.cols.feat64,
                                  fwd.cols.sq64, pot)
    prec = engine.choose_precision(scale, fwd.kd, fwd.sq,
                                   ctr_deferred=lambda: engine.centred_choice_fraction(
                                       eps, fwd.rows, fwd.cols),
                                   pairs=float(fwd.rows.n) * float(fwd.cols.n))
    problem.fwd.prec = prec
    problem.bwd.prec = prec


def device_problem(cost, a, b, device) -> DeviceProblem:
    if isinstance(cost, SquaredEuclideanCost):
        x, z = cost._x, cost._z
        xf, zf = x[:, :-1], z[:, :-1]
        if xf.shape[1] == 0:
            xf, zf = np.zeros((x.shape[0], 1)), np.zeros((z.shape[0], 1))
        _, _, fwd, bwd = feature_problem(xf, x[:, -1], zf, z[:, -1], a, b, device)
        return DeviceProblem(fwd, bwd, (xf * xf).sum(1), (zf * zf).sum(1))
    if isinstance(cost, SeparableLowRankCost):
        _, _, fwd, bwd = feature_problem(cost._u, None, cost._v, None, a, b, device)
        return DeviceProblem(fwd, bwd, cost._ra.copy(), cost._cb.copy())
    n, m = cost.shape
    if n * m > _DENSE_MAX_ENTRIES:
        raise TypeError(
            f"cost provider {type(cost).__name__} has no feature form and {n}x{m} entries is too "
            "large to stream densely; use SquaredEuclideanCost or SeparableLowRankCost"
        )
    if getattr(cost, "_dev", None) is not None:
        c = cost._dev.to(device=device, dtype=torch.float64).contiguous()
    else:
        dense = cost.full() if hasattr(cost, "full") else cost.rows(0, n)
        c = torch.as_tensor(np.ascontiguousarray(dense), dtype=torch.float64, device=device)
    la = torch.log2(engine.to_dev64(a, device))
    lb = torch.log2(engine.to_dev64(b, device))
    fwd = engine.DenseHalfUpdate(c, lb)
    bwd = engine.DenseHalfUpdate(c.t().contiguous(), la)
    return DeviceProblem(fwd, bwd, np.zeros(n), np.zeros(m))


def run_loop(problem: DeviceProblem, a, b, config: SinkhornConfig, f0, g0, device):
    """Run the device loop from reference-parametrised (f0, g0); returns the
    reference-parametrised potentials, stats and the marginal error."""
    a_w, b_w = engine.to_dev64(a, device), engine.to_dev64(b, device)
    f0 = np.asarray(f0, dtype=np.float64)
    g0 = np.asarray(g0, dtype=np.float64)
    _set_precision(problem, min(config.eps, config.anneal_from or config.eps), f0, g0)
    ft = engine.to_dev64(f0 - problem.row_sep, device)
    gt = engine.to_dev64(g0 - problem.col_sep, device)
    loop = engine.SinkhornLoop(problem.fwd, problem.bwd, a_w, b_w, device)
    cfg = config.loop_config()
    small = a_w.numel() * b_w.numel() <= _GRAPH_MAX_PAIRS
    stats = loop.run(ft, gt, cfg, use_graph=small and cfg.max_sweeps >= 4)
    sym_break = stats.broke and cfg.mode == "symmetrized"
    loop.tentatives(ft, gt, need_f=not stats.broke, need_g=not sym_break)
    err = loop.marginal_error(ft, gt, stats.lam)
    f = ft.cpu().numpy() + problem.row_sep
    g = gt.cpu().numpy() + problem.col_sep
    return f, g, stats, err, (ft, gt, loop)


def sinkhorn(a, b, cost, config: SinkhornConfig) -> SinkhornResult:
    """Entropic OT between weights a and b under ``cost`` (reference sinkhorn.py:191-258)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n, m = cost.shape
    if a.shape != (n,) or b.shape != (m,):
        raise ValueError("weight shapes do not match the cost provider")
    if config.warm_start is not None:
        f0 = np.array(config.warm_start[0], dtype=np.float64)
        g0 = np.array(config.warm_start[1], dtype=np.float64)
        if f0.shape != (n,) or g0.shape != (m,):
            raise ValueError("warm-start potential shapes do not match the problem")
    else:
        f0, g0 = np.zeros(n), np.zeros(m)
    device = engine.require_cuda()
    problem = device_problem(cost, a, b, device)
    f, g, stats, err, dev = run_loop(problem, a, b, config, f0, g0, device)
    coupling = ImplicitCoupling(f, g, cost, a, b, stats.eps_eff, device=dev)
    coupling._marginal_err = err
    return SinkhornResult(coupling=coupling, iterations=stats.iterations, marginal_err=err,
                          converged=stats.converged)


def transport_cost(coupling) -> float:
    """<C, pi> over the coupling's own cost provider (reference sinkhorn.py:261-266):
    the fused device passes of plan.py (no host blocks)."""
    from .plan import plan_sums

    if isinstance(coupling, ImplicitCoupling):
        return plan_sums(coupling).transport
    return float(sum((blk * coupling.cost.rows(i0, i1)).sum()
                     for i0, i1, blk in coupling.row_blocks()))


def eot_primal_value(coupling, cost=None, eps: float | None = None) -> float:
    """<C, pi> + eps KL(pi | a x b) (reference sinkhorn.py:269-284)."""
    if isinstance(coupling, ImplicitCoupling):
        eps = coupling.eps_eff if eps is None else eps
        return transport_cost(coupling) + eps * kl_divergence(coupling)
    if cost is None or eps is None:
        raise ValueError("dense couplings need an explicit cost provider and temperature")
    lin = sum(float((blk * cost.rows(i0, i1)).sum()) for i0, i1, blk in coupling.row_blocks())
    return lin + eps * kl_divergence(coupling)
