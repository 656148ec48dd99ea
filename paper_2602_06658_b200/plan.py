"""Device reductions over an implicit plan (the consumers of the plan factors).

The reference evaluates every consumer of an ``ImplicitCoupling`` by walking
row blocks of the reconstructed plan on the host: ``row_marginal`` /
``col_marginal`` (measures.py:197-207), ``marginal_error`` (:229-235),
``kl_divergence`` (:238-256), ``transport_cost`` / ``eot_primal_value``
(sinkhorn.py:261-284), ``gamma_step`` (solvers.py:190-196) and the
``_cnt_reductions`` behind ``egw_objective`` (solvers.py:227-282). Here they
all come from two fused K4 passes on the GPU (``cntgw_plan_reduce``: one over
pi, one over pi^T), with the cost rebuilt on the fly from the provider's
features — no N x M array, no host exponentials:

  pass over pi   : r_i = sum_j pi_ij, (pi A)_i for accumulation features A
                   (zf, or the caller's), (pi zs)_i, argmax_j pi_ij
  pass over pi^T : c_j = sum_i pi_ij, (pi^T xf)_j, (pi^T xs)_j, argmax_i

and, with the cost split as C_ij = row_sep_i + col_sep_j + C~_ij,
C~_ij = -2 <xf_i, zf_j> + (xs_i - zs_j)^2,

  sum pi C~      = -2 sum_i <xf_i, (pi zf)_i> + sum_i r_i xs_i^2
                   - 2 sum_i xs_i (pi zs)_i + sum_j c_j zs_j^2
  <C, pi>        = sum r row_sep + sum c col_sep + sum pi C~
  eps KL(pi|ab)  = sum_i r_i f~_i + sum_j c_j g~_j - sum pi C~

(f~ = f - row_sep, g~ = g - col_sep: log(pi_ij / a_i b_j) = (f_i + g_j -
C_ij)/eps, so the separable parts cancel and the identity is exact). Costs
without a feature form (``DenseCost``, duck-typed providers) take a blocked
fp64 pass on the GPU instead.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine
from ._native import F64, LIB, call

# rows per block of the generic (feature-less) pass: block x M fp64 entries
_GENERIC_BLOCK_ENTRIES = 1 << 25


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class FeatureForm:
    """C_ij = row_sep_i + col_sep_j - 2 <xf_i, zf_j> + (xs_i - zs_j)^2 on the device (fp64)."""

    def __init__(self, xf, xs, zf, zs, row_sep, col_sep):
        self.xf, self.xs, self.zf, self.zs = xf, xs, zf, zs
        self.row_sep, self.col_sep = row_sep, col_sep
        self.k = xf.shape[1]
        self.kd = engine.padded_kd(max(self.k, 1))

    def transpose(self) -> "FeatureForm":
        return FeatureForm(self.zf, self.zs, self.xf, self.xs, self.col_sep, self.row_sep)


def feature_form(cost, device) -> FeatureForm | None:
    """The feature form of this package's cost providers, else None."""
    from .sinkhorn import SeparableLowRankCost, SquaredEuclideanCost

    def dev(x):
        return engine.to_dev64(np.ascontiguousarray(x), device)

    if isinstance(cost, SquaredEuclideanCost):
        x, z = cost._x, cost._z
        if x.shape[1] == 1:
            xf, zf = np.zeros((x.shape[0], 1)), np.zeros((z.shape[0], 1))
        else:
            xf, zf = x[:, :-1], z[:, :-1]
        xf, zf = dev(xf), dev(zf)
        return FeatureForm(xf, dev(x[:, -1]), zf, dev(z[:, -1]), (xf * xf).sum(1), (zf * zf).sum(1))
    if isinstance(cost, SeparableLowRankCost):
        u, v = dev(cost._u), dev(cost._v)
        return FeatureForm(u, torch.zeros(u.shape[0], dtype=torch.float64, device=device), v,
                           torch.zeros(v.shape[0], dtype=torch.float64, device=device),
                           dev(cost._ra), dev(cost._cb))
    return None


def row_pass(form: FeatureForm, f_t, g_t, a, b, eps, acc, acc_s):
    """One K4 pass over pi_ij = a_i b_j exp((f~_i + g~_j - C~_ij)/eps):
    (r, pi acc (n x e), pi acc_s, argmax_j), all device fp64 / int64."""
    device = f_t.device
    n, m = form.xf.shape[0], form.zf.shape[0]
    kd = form.kd
    xf = engine.to_dev64(form.xf, device, kd)
    zf = engine.to_dev64(form.zf, device, kd)
    acc = acc.contiguous()
    e = acc.shape[1]
    st = engine.SweepState(device)
    st.init(eps)
    stride = LIB.cntgw_col_stride(F64, kd, 1)
    rec = torch.empty(int(LIB.cntgw_cols_padded(m)) * stride, dtype=torch.float64, device=device)
    log2a, log2b = torch.log2(a), torch.log2(b)
    s = _stream()
    call("cntgw_prep_cols", st.ptr, F64, kd, 1, zf.data_ptr(), kd, form.zs.data_ptr(), g_t.data_ptr(),
         log2b.data_ptr(), m, rec.data_ptr(), s)
    r = torch.empty(n, dtype=torch.float64, device=device)
    pi_acc = torch.empty(n * e, dtype=torch.float64, device=device)
    pi_s = torch.empty(n, dtype=torch.float64, device=device)
    am = torch.empty(n, dtype=torch.int64, device=device)
    ws = torch.empty(int(LIB.cntgw_plan_reduce_workspace(n, m, kd, e)), dtype=torch.uint8, device=device)
    call("cntgw_plan_reduce", st.ptr, kd, e, xf.data_ptr(), kd, form.xs.data_ptr(), f_t.data_ptr(),
         log2a.data_ptr(), rec.data_ptr(), acc.data_ptr(), e, acc_s.contiguous().data_ptr(), n, m,
         r.data_ptr(), pi_acc.data_ptr(), pi_s.data_ptr(), am.data_ptr(), ws.data_ptr(), ws.numel(), s)
    return r, pi_acc.view(n, e), pi_s, am


class PlanSums:
    """Every scalar and marginal the reference reads off an implicit plan,
    computed once per coupling on the GPU (fp64)."""

    def __init__(self, row, col, transport, kl, argmax_row, argmax_col):
        self.row, self.col = row, col  # device (n,), (m,)
        self.transport, self.kl = transport, kl
        self.argmax_row, self.argmax_col = argmax_row, argmax_col

    @property
    def marginal_error(self) -> float:
        return self._err

    @staticmethod
    def _finish(row, col, a, b, transport, kl, am_r, am_c):
        ps = PlanSums(row, col, transport, kl, am_r, am_c)
        ps._err = float((row - a).abs().sum() + (col - b).abs().sum())
        return ps


def _coupling_tensors(coupling, device):
    """(f, g, a, b) on the device, uploaded once per coupling (its arrays are
    read-only, measures.py)."""
    cached = getattr(coupling, "_dev_factors", None)
    if cached is not None and cached[0].device == device:
        return cached
    out = tuple(engine.to_dev64(v, device) for v in (coupling.f, coupling.g, coupling.source_weights,
                                                     coupling.target_weights))
    coupling._dev_factors = out
    return out


def plan_sums(coupling) -> PlanSums:
    """Cached device reductions of an ImplicitCoupling (see module docstring)."""
    cached = getattr(coupling, "_plan_sums", None)
    if cached is not None:
        return cached
    device = engine.require_cuda()
    form = feature_form(coupling.cost, device)
    f, g, a, b = _coupling_tensors(coupling, device)
    eps = coupling.eps_eff
    if form is None:
        out = _generic_sums(coupling, f, g, a, b, eps, device)
    else:
        f_t, g_t = f - form.row_sep, g - form.col_sep
        zf = engine.to_dev64(form.zf, device, form.kd)
        xf = engine.to_dev64(form.xf, device, form.kd)
        r, pi_zf, pi_zs, am_r = row_pass(form, f_t, g_t, a, b, eps, zf, form.zs)
        c, _, _, am_c = row_pass(form.transpose(), g_t, f_t, b, a, eps, xf, form.xs)
        k = form.k
        pc = (-2.0 * (xf[:, :k] * pi_zf[:, :k]).sum() + (r * form.xs * form.xs).sum()
              - 2.0 * (form.xs * pi_zs).sum() + (c * form.zs * form.zs).sum())
        transport = float((r * form.row_sep).sum() + (c * form.col_sep).sum() + pc)
        kl = float(((r * f_t).sum() + (c * g_t).sum() - pc) / eps)
        out = PlanSums._finish(r, c, a, b, transport, kl, am_r, am_c)
    coupling._plan_sums = out
    return out


def _cost_rows_dev(cost, i0, i1, device):
    rows_dev = getattr(cost, "_rows_dev", None)
    if rows_dev is not None:
        return rows_dev(i0, i1, device)
    return torch.as_tensor(np.ascontiguousarray(cost.rows(i0, i1), dtype=np.float64), device=device)


def log_plan_block(coupling, i0, i1, device=None) -> torch.Tensor:
    """log pi over rows [i0, i1) on the device (reference measures.py:185-195)."""
    device = device or engine.require_cuda()
    f, g, a, b = _coupling_tensors(coupling, device)
    inv = 1.0 / coupling.eps_eff
    c = _cost_rows_dev(coupling.cost, i0, i1, device)
    return (torch.log(a[i0:i1]) + f[i0:i1] * inv)[:, None] + (torch.log(b) + g * inv)[None, :] - c * inv


def block_rows(n, m) -> int:
    return max(1, min(n, _GENERIC_BLOCK_ENTRIES // max(m, 1)))


def _generic_sums(coupling, f, g, a, b, eps, device) -> PlanSums:
    """Blocked fp64 pass on the GPU for providers without a feature form."""
    n, m = coupling.shape
    inv = 1.0 / eps
    la, lb = torch.log(a) + f * inv, torch.log(b) + g * inv
    r = torch.empty(n, dtype=torch.float64, device=device)
    c = torch.zeros(m, dtype=torch.float64, device=device)
    am_r = torch.empty(n, dtype=torch.int64, device=device)
    col_best = torch.full((m,), -math.inf, dtype=torch.float64, device=device)
    am_c = torch.zeros(m, dtype=torch.int64, device=device)
    transport = torch.zeros((), dtype=torch.float64, device=device)
    klsum = torch.zeros((), dtype=torch.float64, device=device)
    step = block_rows(n, m)
    for i0 in range(0, n, step):
        i1 = min(i0 + step, n)
        cost = _cost_rows_dev(coupling.cost, i0, i1, device)
        logp = la[i0:i1, None] + lb[None, :] - cost * inv
        p = torch.exp(logp)
        r[i0:i1] = p.sum(1)
        c += p.sum(0)
        am_r[i0:i1] = torch.argmax(logp, dim=1)
        transport += (p * cost).sum()
        klsum += (p * ((f[i0:i1, None] + g[None, :] - cost) * inv)).sum()
        best, arg = logp.max(dim=0)  # first max within the block; strict > keeps earlier blocks
        upd = best > col_best
        col_best = torch.where(upd, best, col_best)
        am_c = torch.where(upd, arg + i0, am_c)
    return PlanSums._finish(r, c, a, b, float(transport), float(klsum), am_r, am_c)


def dense_sums(matrix: torch.Tensor, a: torch.Tensor, b: torch.Tensor):
    """(row, col, KL(pi | a x b)) of an explicit plan on the device, 0 log 0 = 0."""
    row, col = matrix.sum(1), matrix.sum(0)
    ref = a[:, None] * b[None, :]
    keep = matrix > 0.0
    kl = float(torch.where(keep, matrix * torch.log(torch.where(keep, matrix, 1.0) / ref), 0.0).sum())
    return row, col, kl
