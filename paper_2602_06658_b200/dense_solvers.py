"""Dense-plan GW baselines (reference solvers.py:384-553, 625-641; SURVEY.md
§8(f) row 4): the kernel-trick EGW solver and the classical projected-descent
Entropic-GW, used as cross-solver equivalence oracles under the
``max_dense_entries`` guard.

Everything lives on the GPU in fp64: the centred kernels K_X, K_Y, the plan
pi (N x M), the sandwich K_X pi K_Y (two DGEMMs per outer step, cuBLAS on the
FP64 tensor pipe), the step costs, the plan rebuilt from the Sinkhorn
potentials and the KL / objective reductions; each inner Sinkhorn runs the
dense-cost half-update kernel (``cntgw_softmin_dense``) on a device-resident
``DenseCost``. Only the returned ``DenseCoupling`` is copied to the host.
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import torch

from . import engine
from .kernels import _kernel_dev
from .measures import DenseCoupling
from .sinkhorn import DenseCost, sinkhorn


class _DenseState:
    """Shared machinery for the kernel-trick and classical baselines."""

    family = "dense"

    def __init__(self, src_cost, tgt_cost, a, b, cfg):
        from .solvers import _StepStats  # noqa: F401  (type used by step)

        self.cfg = cfg
        self.a_np = np.asarray(a, dtype=np.float64)
        self.b_np = np.asarray(b, dtype=np.float64)
        n, m = self.a_np.size, self.b_np.size
        guard = cfg.max_dense_entries
        for label, entries in (("plan", n * m), ("source kernel", n * n), ("target kernel", m * m)):
            if entries > guard:
                raise ValueError(
                    f"{label} would hold {entries} entries, beyond the memory guard "
                    f"({guard}); use the feature-space solver or raise max_dense_entries")
        dev = engine.require_cuda()
        self.dev = dev
        self.cx = torch.as_tensor(np.asarray(src_cost, dtype=np.float64), device=dev)
        self.cy = torch.as_tensor(np.asarray(tgt_cost, dtype=np.float64), device=dev)
        if tuple(self.cx.shape) != (n, n) or tuple(self.cy.shape) != (m, m):
            raise ValueError("cost matrix shapes do not match the weights")
        self.a = torch.as_tensor(self.a_np, device=dev)
        self.b = torch.as_tensor(self.b_np, device=dev)
        self.kx = _kernel_dev(self.cx, self.a)
        self.ky = _kernel_dev(self.cy, self.b)
        self.dx = torch.diagonal(self.kx).clone()
        self.dy = torch.diagonal(self.ky).clone()
        tx = float(self.a @ self.dx)
        ty = float(self.b @ self.dy)
        self.constant = (float(self.a @ (self.cx**2) @ self.a) + float(self.b @ (self.cy**2) @ self.b)
                         - 4.0 * tx * ty)
        self.pi = self._initial_plan()
        self.sandwich = self.kx @ self.pi @ self.ky
        self.f = np.zeros(n)
        self.g = np.zeros(m)
        self.coupling = None
        self.record = []
        self.last_inner_err = 0.0

    def _initial_plan(self) -> torch.Tensor:
        cfg = self.cfg
        if cfg.init == "product":
            return torch.outer(self.a, self.b)
        if cfg.init == "coupling":
            raw = getattr(cfg.init_coupling, "matrix", cfg.init_coupling)
            pi = np.asarray(raw, dtype=np.float64)
            if pi.shape != (self.a_np.size, self.b_np.size):
                raise ValueError("init_coupling shape does not match the weights")
            return torch.as_tensor(np.array(pi), device=self.dev)
        raise ValueError(
            f"init={cfg.init!r} is not available for dense solvers; use 'product' or 'coupling'")

    def _step_cost(self) -> torch.Tensor:
        raise NotImplementedError

    def _objective(self, pi_new, sandwich_new, kl) -> float:
        raise NotImplementedError

    def _warm_start(self):
        return self.f, self.g

    def step(self, inner_budget=None, anneal_from=None):
        from .solvers import _StepStats

        cfg = self.cfg
        inner = cfg.inner.with_warm_start(*self._warm_start())
        if inner_budget is not None:
            inner = replace(inner, n_inner=inner_budget, threshold=None)
        if anneal_from is not None:
            inner = replace(inner, anneal_from=anneal_from)
        c = self._step_cost()
        res = sinkhorn(self.a_np, self.b_np, DenseCost(c), inner.with_temperature(cfg.eps))
        self.f, self.g = res.coupling.f, res.coupling.g
        # pi = exp(log a + f/eps + log b + g/eps - C/eps) (measures.py:185-195),
        # KL from the same log-ratio (f + g - C)/eps (measures.py:245-252)
        inv = 1.0 / res.coupling.eps_eff
        f = torch.as_tensor(self.f, device=self.dev)
        g = torch.as_tensor(self.g, device=self.dev)
        row = torch.log(self.a) + f * inv
        col = torch.log(self.b) + g * inv
        pi_new = torch.exp(row[:, None] + col[None, :] - c * inv)
        kl = float((pi_new * ((f[:, None] + g[None, :] - c) * inv)).sum())
        sandwich_new = self.kx @ pi_new @ self.ky
        # ||Gamma(pi') - Gamma(pi)||_HS via the kernel trick
        delta_sq = (float((pi_new * sandwich_new).sum()) - 2.0 * float((pi_new * self.sandwich).sum())
                    + float((self.pi * self.sandwich).sum()))
        objective = self._objective(pi_new, sandwich_new, kl)
        self.pi = pi_new
        self.sandwich = sandwich_new
        self.coupling = res.coupling
        self.last_inner_err = res.marginal_err
        if cfg.record_iterates:
            self.record.append(pi_new.cpu().numpy())
        return _StepStats(objective, math.sqrt(max(delta_sq, 0.0)), res.marginal_err, res.iterations)

    def result(self, trace, converged, schedule=None):
        from .solvers import EgwResult, SolverError

        try:
            final = DenseCoupling(self.pi.cpu().numpy(), self.a_np, self.b_np)
        except ValueError as exc:
            raise SolverError(
                f"final plan failed validation ({exc}); raise n_inner or use the "
                "adaptive wrapper") from exc
        return EgwResult(gamma=None, coupling=final, trace=trace,
                         value=trace.objectives[-1] if len(trace) else math.nan,
                         converged=converged,
                         iterates=self.record if self.cfg.record_iterates else None,
                         schedule=schedule)


class _KernelGwState(_DenseState):
    def _step_cost(self) -> torch.Tensor:
        return -4.0 * torch.outer(self.dx, self.dy) - 16.0 * self.sandwich

    def _objective(self, pi_new, sandwich_new, kl) -> float:
        gamma_sq = float((pi_new * sandwich_new).sum())
        sigma_ss = 0.25 * float(self.dx @ pi_new @ self.dy)
        return self.constant + 8.0 * (-gamma_sq + (self.cfg.eps / 8.0) * kl - 2.0 * sigma_ss)


class _EntropicGwState(_DenseState):
    def __init__(self, src_cost, tgt_cost, a, b, cfg):
        super().__init__(src_cost, tgt_cost, a, b, cfg)
        self.sx = (self.cx**2) @ self.a
        self.sy = (self.cy**2) @ self.b
        self.rx = self.cx @ self.a
        self.ry = self.cy @ self.b
        self.mx = float(self.a @ self.rx)
        self.my = float(self.b @ self.ry)
        self.cxy_sandwich = self.cx @ self.pi @ self.cy
        # separable offset between this step cost and the kernel-trick cost at
        # the same plan (solvers.py:506-514)
        self._u, self._v = self._separable_offset(self.pi)
        self.f = self._u.cpu().numpy()
        self.g = self._v.cpu().numpy()

    def _separable_offset(self, pi):
        u = 2.0 * self.sx - 4.0 * (self.cx @ (pi @ self.ry)) + 2.0 * self.my * self.rx
        v = 2.0 * self.sy - 4.0 * (self.cy @ (pi.t() @ self.rx)) + 2.0 * self.mx * self.ry
        return u, v

    def _warm_start(self):
        u, v = self._separable_offset(self.pi)
        warm = (self.f + (u - self._u).cpu().numpy(), self.g + (v - self._v).cpu().numpy())
        self._u, self._v = u, v
        return warm

    def _step_cost(self) -> torch.Tensor:
        return 2.0 * self.sx[:, None] + 2.0 * self.sy[None, :] - 4.0 * self.cxy_sandwich

    def _objective(self, pi_new, sandwich_new, kl) -> float:
        self.cxy_sandwich = self.cx @ pi_new @ self.cy
        mu = pi_new.sum(1)
        nu = pi_new.sum(0)
        quartic = (float(mu @ (self.cx**2) @ mu) + float(nu @ (self.cy**2) @ nu)
                   - 2.0 * float((pi_new * self.cxy_sandwich).sum()))
        return quartic + self.cfg.eps * kl


def solve_kernel_gw(src_cost, tgt_cost, a, b, cfg):
    """Kernel-trick EGW solve on dense plans, exact for any CNT cost (solvers.py:629-633)."""
    from .solvers import _run_outer

    return _run_outer(_KernelGwState(src_cost, tgt_cost, a, b, cfg), cfg)


def solve_entropic_gw(src_cost, tgt_cost, a, b, cfg):
    """Classical projected-descent baseline with the full loss gradient (solvers.py:636-638)."""
    from .solvers import _run_outer

    return _run_outer(_EntropicGwState(src_cost, tgt_cost, a, b, cfg), cfg)
