"""Device engine: the Sinkhorn loop and its half-update operators on one GPU.

Everything here operates on CUDA tensors and launches the C-ABI kernels of
``libcntgw_b200.so`` on torch's current stream. The loop state (sweep counter,
eps_n, threshold decision, done flag) lives in device memory
(``cntgw_sweep_state``), so sweeps are enqueued back to back without host
round trips, and chunks of sweeps are replayed as CUDA graphs for small
problems; the host reads the state once per chunk to learn whether a
threshold run finished.

Cost model every feature provider reduces to (include/cntgw_b200.h):
    C_ij = row_sep_i + col_sep_j - 2 <xf_i, zf_j> + (xs_i - zs_j)^2
with fp64 interaction potentials f~ = f - row_sep, g~ = g - col_sep on device.

Precision: the exponent t_ij is assembled in fp32 (FFMA2) when its terms are
small enough that fp32 rounding stays below ~2e-4 log2 units, else in fp64
(DFMA; B200 runs fp64 at half the fp32 rate). ``choose_precision`` makes the
call from the problem's scales; CNTGW_PRECISION=f32|f64 forces it.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import F32, F32C, F64, F64S, LIB, TF32X3, SweepStateStruct, call

SUPPORTED_KD = (1, 2, 3, 4, 8, 16, 32, 64)
# fp32 exponent assembly is used while lam * (term magnitudes) stays below this
# (fp32 ulp there is 2^-12 log2 units ~ 1.7e-4 relative error per plan entry)
F32_EXPONENT_LIMIT = 4096.0


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "cntgw_b200 needs a CUDA device (B200/sm_100a); there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)


def padded_kd(k: int) -> int:
    for kd in SUPPORTED_KD:
        if k <= kd:
            return kd
    raise ValueError(f"feature width {k} exceeds the supported maximum {SUPPORTED_KD[-1]}")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t) -> int:
    return 0 if t is None else t.data_ptr()


def to_dev(x, device, dtype, kd=None) -> torch.Tensor:
    """Contiguous device copy in ``dtype``, zero-padded to kd columns if given."""
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x)
        if not x.flags.writeable:
            x = x.copy()
    t = torch.as_tensor(x).to(device=device, dtype=dtype)
    if kd is not None:
        if t.ndim == 1:
            t = t[:, None]
        if t.shape[1] < kd:
            t = torch.nn.functional.pad(t, (0, kd - t.shape[1]))
    return t.contiguous()


def to_dev64(x, device, kd=None) -> torch.Tensor:
    return to_dev(x, device, torch.float64, kd)


def to_dev32(x, device, kd=None) -> torch.Tensor:
    return to_dev(x, device, torch.float32, kd)


def exponent_scale(eps: float, feat_r, sq_r, feat_c, sq_c, pot_abs: float = 0.0) -> float:
    """Upper bound (log2 units) of the terms the half-update adds: lam (|pot| +
    2 |x||z| + (|s_r| + |s_c|)^2)."""
    lam = math.log2(math.e) / eps

    def rowmax(t):
        return float(t.norm(dim=1).max()) if t.numel() else 0.0

    def absmax(t):
        return float(t.abs().max()) if t is not None and t.numel() else 0.0

    dot = 2.0 * rowmax(feat_r) * rowmax(feat_c)
    sq = (absmax(sq_r) + absmax(sq_c)) ** 2
    return lam * (pot_abs + dot + sq)


# CNTGW_F32C (centred fp32 on locality-ordered tiles): a (row group, column
# tile) pair whose fp32 pair term can exceed this bound (log2 units; fp32 ulp
# there is 2^-8) runs in fp64 inside the kernel (CNTGW_CTR_TILE_LIMIT, read
# by the library); the path is chosen for a cold problem while at most
# CTR_MAX_DEFERRED of the pairs need that fallback (softmin_ctr.cuh).
CTR_TILE_LIMIT = float(os.environ.get("CNTGW_CTR_TILE_LIMIT", 65536.0))
CTR_MAX_DEFERRED = 0.05
# ... and only for half-updates of at least this many pairs: below it the
# fp64 kernels take a few milliseconds, the planning pass and the per-step
# path decision do not pay off (C3, 1e10 pairs: 1.72 s centred vs 1.08 s
# fp64), and fp64 keeps fp64-level agreement with the reference's discrete
# decisions (threshold stops, divergence guard)
CTR_MIN_PAIRS = float(os.environ.get("CNTGW_CTR_MIN_PAIRS", 2.0 ** 34))
CTR_ROW_GROUP, CTR_COL_TILE = 128, 256


def ctr_supported(kd: int, sq: bool) -> bool:
    return kd + int(bool(sq)) <= 8


def locality_order(coords: torch.Tensor) -> torch.Tensor:
    """Permutation visiting the points in Morton (Z-curve) order of their first
    min(d, 3) coordinates (cntgw_locality_codes + a stable device sort)."""
    x = coords.to(torch.float64)
    if x.ndim == 1:
        x = x[:, None]
    x = x.contiguous()
    n, d = x.shape
    codes = torch.empty(n, dtype=torch.int64, device=x.device)
    bbox = torch.empty(6, dtype=torch.float64, device=x.device)
    call("cntgw_locality_codes", x.data_ptr(), n, d, d, bbox.data_ptr(), codes.data_ptr(), _stream())
    return torch.sort(codes, stable=True).indices


def cluster_order(points: torch.Tensor, sq: torch.Tensor | None = None, k: int = 64, sweeps: int = 8,
                  seed: int = 0) -> torch.Tensor:
    """Permutation grouping high-dimensional points by a k-means clustering
    (CNTGW_F64S row groups / column stages): k seeded centres, `sweeps`
    Lloyd iterations (streamed assignment ``cntgw_km_assign``; centres as a
    one-hot fp64 GEMM, deterministic), then points sorted by (cluster, squared
    coordinate) — at Gamma = 0 the GW cost depends on the points only through
    (s_i - t_j)^2, and the order keeps that band contiguous — or by (cluster,
    Morton code of the first coordinates) without one."""
    x = points.to(torch.float64).contiguous()
    n, d = x.shape
    k = max(1, min(k, n))
    gen = torch.Generator(device="cpu").manual_seed(seed)
    pick = torch.randperm(n, generator=gen)[:k].to(x.device)
    centers = x[pick].contiguous()
    assign = torch.empty(n, dtype=torch.int64, device=x.device)
    own = torch.empty(n, dtype=torch.float64, device=x.device)
    for _ in range(sweeps):
        call("cntgw_km_assign", x.data_ptr(), n, d, centers.data_ptr(), k, assign.data_ptr(),
             own.data_ptr(), _stream())
        onehot = torch.nn.functional.one_hot(assign, k).to(torch.float64)
        counts = onehot.sum(0)
        sums = onehot.t() @ x
        keep = counts > 0
        centers = torch.where(keep[:, None], sums / counts.clamp_min(1.0)[:, None], centers).contiguous()
    call("cntgw_km_assign", x.data_ptr(), n, d, centers.data_ptr(), k, assign.data_ptr(),
         own.data_ptr(), _stream())
    fine = locality_order(x[:, : min(d, 3)]) if sq is None else torch.sort(sq, stable=True).indices
    rank = torch.empty_like(fine)
    rank[fine] = torch.arange(n, device=x.device)
    return torch.sort(assign * n + rank, stable=True).indices


def side_order(feat: torch.Tensor, sq: torch.Tensor | None) -> torch.Tensor:
    """Locality order of a point cloud: Morton codes when the points are
    low-dimensional (the centred path's tiles), a k-means cluster order above
    (the measured-plan path's row groups and column stages)."""
    real = int((feat.abs().amax(0) > 0).sum()) if feat.numel() else 0
    if real <= 3 or feat.shape[1] not in (4, 8, 16, 32, 64):
        return locality_order(feat if sq is None else torch.cat([feat, sq[:, None]], 1))
    return cluster_order(feat, sq)


def _tile_radii(pts: torch.Tensor, order: torch.Tensor, tile: int) -> torch.Tensor:
    """max |p - mean| of each consecutive `tile`-point group in `order`."""
    p = pts[order]
    n = p.shape[0]
    full = n // tile * tile
    out = []
    if full:
        g = p[:full].view(-1, tile, p.shape[1])
        out.append((g - g.mean(1, keepdim=True)).norm(dim=2).amax(1))
    if full < n:
        t = p[full:]
        out.append((t - t.mean(0, keepdim=True)).norm(dim=1).amax()[None])
    return torch.cat(out)


def _side_points(side) -> torch.Tensor:
    return side.feat64 if side.sq64 is None else torch.cat([side.feat64, side.sq64[:, None]], 1)


def centred_radii(eps: float, rows: "Side", cols: "Side"):
    """(group radii of the rows, tile radii of the columns in log2-scaled units):
    their product bounds the fp32 pair term of a (group, tile) pair."""
    lam = math.log2(math.e) / eps
    rr = _tile_radii(_side_points(rows), rows.locality(), CTR_ROW_GROUP)
    rc = _tile_radii(_side_points(cols), cols.locality(), CTR_COL_TILE) * (2.0 * lam)
    return rr, rc


def centred_scale(eps: float, rows: "Side", cols: "Side") -> float:
    """Worst (group, tile) bound of the fp32 pair term (diagnostic)."""
    rr, rc = centred_radii(eps, rows, cols)
    return float(rr.max() * rc.max())


def centred_choice_fraction(eps: float, rows: "Side", cols: "Side") -> float:
    """The deferred fraction choose_precision compares (both half-update
    directions), or 1.0 for problems below CTR_MIN_PAIRS."""
    if float(rows.n) * float(cols.n) < CTR_MIN_PAIRS:
        return 1.0
    return max(centred_deferred_fraction(eps, rows, cols), centred_deferred_fraction(eps, cols, rows))


def centred_deferred_fraction(eps: float, rows: "Side", cols: "Side") -> float:
    """Fraction of (row group, column tile) pairs the kernel will run in fp64."""
    rr, rc = centred_radii(eps, rows, cols)
    rc_sorted = torch.sort(rc).values
    need = CTR_TILE_LIMIT / rr.clamp_min(1e-300)  # a tile is deferred when rc > need
    over = rc_sorted.numel() - torch.searchsorted(rc_sorted, need, right=True)
    return float(over.sum()) / (rr.numel() * rc.numel())


def tc_supported(kd: int, sq: bool) -> bool:
    """Shapes the tcgen05 3xTF32 half-update serves (include/cntgw_b200.h)."""
    return kd in (8, 16) and not sq


# CNTGW_F64S (fp64 with a measured block-sparse plan) for cold problems, from
# this many pairs per half-update: below it a dense fp64 sweep is cheaper than
# the plan's ~15 small launches per half-update. Measured crossovers on the
# cold laws (tools/gpu/r2_s3_45.sh, time per outer step): kd = 3 between
# N = 8192 (dense 24 ms, F64S 35 ms) and 16384 (87 / 46 ms); kd = 32 between
# N = 2048 (28 / 48 ms) and 4096 (52 / 30 ms); at N = 65536 / 32768 the plan
# is 8x / 12x faster. CNTGW_F64S_MIN_PAIRS overrides.
def f64s_min_pairs(kd: int) -> float:
    env = os.environ.get("CNTGW_F64S_MIN_PAIRS")
    if env is not None:
        return float(env)
    return 2.0 ** 24 if kd >= 16 else 2.0 ** 27


def choose_precision(scale: float, kd: int = 0, sq: bool = True, ctr_deferred=None,
                     pairs: float = 0.0) -> int:
    """Cold problems: the centred fp32 path while few tile pairs need its fp64
    fallback (``ctr_deferred``, a callable evaluated only then), else fp64
    (with a measured block-sparse plan for large problems, CNTGW_F64S);
    otherwise the tensor cores where the shape allows."""
    forced = os.environ.get("CNTGW_PRECISION", "auto").lower()
    if forced in ("f32", "fp32"):
        return F32
    if forced in ("f64", "fp64"):
        return F64
    if forced in ("f64s",):
        return F64S
    if forced in ("tc", "tf32x3"):
        return TF32X3 if tc_supported(kd, sq) else F32
    if forced in ("f32c", "ctr"):
        return F32C if ctr_supported(kd, sq) else F64
    if scale >= F32_EXPONENT_LIMIT:
        # cold problems past the crossover: fp64 with the measured block-sparse plan
        if pairs >= f64s_min_pairs(kd) and os.environ.get("CNTGW_F64S", "1") != "0":
            return F64S
        if (ctr_deferred is not None and ctr_supported(kd, sq)
                and os.environ.get("CNTGW_CTR", "1") != "0" and ctr_deferred() <= CTR_MAX_DEFERRED):
            return F32C
        return F64
    return TF32X3 if tc_supported(kd, sq) else F32


class SweepState:
    """Device-resident ``cntgw_sweep_state``."""

    SIZE = ctypes.sizeof(SweepStateStruct)

    def __init__(self, device):
        self.buf = torch.zeros(self.SIZE, dtype=torch.uint8, device=device)
        self.ptr = self.buf.data_ptr()

    def init(self, eps, anneal_from=None, threshold=None, max_sweeps=1, mode="symmetrized"):
        call("cntgw_sweep_init", self.ptr, float(eps), float(anneal_from or 0.0),
             float(threshold or 0.0), int(max_sweeps), 1 if mode == "symmetrized" else 0, _stream())

    def begin(self):
        call("cntgw_sweep_begin", self.ptr, _stream())

    def read(self) -> SweepStateStruct:
        return SweepStateStruct.from_buffer_copy(self.buf.cpu().numpy().tobytes())

    def done_flag(self) -> bool:
        off = SweepStateStruct.done.offset
        return bool(self.buf[off:off + 4].cpu().view(torch.int32).item())


class Side:
    """One marginal as the kernels see it: dot features (n x kd), the optional
    squared-difference coordinate, weights. fp64 is the source of truth; the
    fp32 copies feed the fp32 kernels."""

    def __init__(self, feat64: torch.Tensor, sq64: torch.Tensor | None, w: torch.Tensor,
                 order: torch.Tensor | None = None):
        self.feat64 = feat64
        self.sq64 = sq64
        self.w = w
        self.log2w = torch.log2(w)
        self._f32 = None
        self.order = order  # locality order of the points (CNTGW_F32C), lazily from feat64
        self.f64s_order = None  # CNTGW_F64S's order when it differs (set per loop by the solver)

    def locality(self) -> torch.Tensor:
        if self.order is None:
            self.order = side_order(self.feat64, self.sq64)
        return self.order

    def plan_order(self) -> torch.Tensor:
        """The point order of the measured-plan path (CNTGW_F64S)."""
        return self.f64s_order if self.f64s_order is not None else self.locality()

    @staticmethod
    def make(feat, sq, w, device, kd):
        return Side(to_dev64(feat, device, kd), None if sq is None else to_dev64(sq, device),
                    to_dev64(w, device))

    @property
    def n(self) -> int:
        return self.feat64.shape[0]

    @property
    def kd(self) -> int:
        return self.feat64.shape[1]

    def refresh32(self):
        """Re-round the fp32 copies in place (their addresses may be baked into
        captured CUDA graphs, so they are never reallocated)."""
        if self._f32 is None:
            self._f32 = (self.feat64.float(), None if self.sq64 is None else self.sq64.float())
        else:
            self._f32[0].copy_(self.feat64)
            if self.sq64 is not None:
                self._f32[1].copy_(self.sq64)

    def feat(self, prec):
        """(features, sq) in the dtype the precision path reads (TF32X3 reads fp32)."""
        if prec == F64:
            return self.feat64, self.sq64
        if self._f32 is None:
            self.refresh32()
        return self._f32


class HalfUpdate:
    """out_rows = S(pot_cols): pack the column side's records, then stream them."""

    def __init__(self, rows: Side, cols: Side, sq: bool, prec: int = F32):
        self.rows, self.cols, self.sq = rows, cols, bool(sq)
        self.kd = rows.kd
        assert cols.kd == self.kd
        self._prec = F32
        dev = rows.feat64.device
        precs = (F32, F64, TF32X3) if tc_supported(self.kd, self.sq) else (F32, F64)
        rec_bytes = 0
        for p in precs:
            stride = LIB.cntgw_col_stride(p, self.kd, int(self.sq))
            _native.check(0 if stride > 0 else stride, "cntgw_col_stride")
            rec_bytes = max(rec_bytes, stride * (8 if p == F64 else 4))
        self.rec = torch.empty(LIB.cntgw_cols_padded(cols.n) * rec_bytes // 8, dtype=torch.float64,
                               device=dev)
        if ctr_supported(self.kd, self.sq):
            precs = precs + (F32C,)
            # row / column blocks of the centred path (fixed addresses for graph capture)
            self.ctr_rows = torch.empty(int(LIB.cntgw_ctr_rows_bytes(rows.n, self.kd, int(self.sq))),
                                        dtype=torch.uint8, device=dev)
            self.ctr_cols = torch.empty(int(LIB.cntgw_ctr_cols_bytes(cols.n, self.kd, int(self.sq))),
                                        dtype=torch.uint8, device=dev)
        wsb = max(LIB.cntgw_softmin_workspace(p, rows.n, cols.n, self.kd, int(self.sq)) for p in precs)
        self.ws = torch.empty(max(int(wsb), 16), dtype=torch.uint8, device=dev)
        self.f64s_rows = None
        # CNTGW_F64S: the rows block (order | features | s) and the columns' feature records are
        # fixed within a loop; a driver that owns the loop gathers the rows once (hoist_rows)
        # instead of once per half-update and lets pack() rewrite only the bias column
        self.rows_hoisted = False
        self.prec = prec  # (the setter sizes the F64S buffers: after the fields above)

    @property
    def prec(self) -> int:
        return self._prec

    @prec.setter
    def prec(self, p: int):
        if p in (F32C, F64S):  # orders and buffers are made eagerly, never inside a graph capture
            self.rows.locality()
            self.cols.locality()
        if p == F64S:
            r, c, dev = self.rows, self.cols, self.rows.feat64.device
            if self.f64s_rows is None:
                self.f64s_rows = torch.empty(int(LIB.cntgw_f64s_rows_bytes(r.n, self.kd)), dtype=torch.uint8,
                                             device=dev)
            need = int(LIB.cntgw_softmin_workspace(F64S, r.n, c.n, self.kd, int(self.sq)))
            if self.ws.numel() < need:  # the measured plan (tmin per row and stage)
                self.ws = torch.empty(need, dtype=torch.uint8, device=dev)
        self._prec = p

    def pack(self, state: SweepState, pot_cols: torch.Tensor | None, prec=None):
        prec = self.prec if prec is None else prec
        c = self.cols
        if prec == F32C:
            call("cntgw_prep_cols_ctr", state.ptr, self.kd, int(self.sq), c.feat64.data_ptr(), self.kd,
                 _p(c.sq64 if self.sq else None), _p(pot_cols), c.log2w.data_ptr(),
                 c.locality().data_ptr(), c.n, self.ctr_cols.data_ptr(), _stream())
            return
        if prec == F64S:
            # (hoisted: the owner of the loop guarantees fixed column features, so after the
            # loop's first sweep only the bias column is rewritten)
            call("cntgw_update_cols_f64s" if self.rows_hoisted else "cntgw_prep_cols_f64s",
                 state.ptr, self.kd, int(self.sq), c.feat64.data_ptr(), self.kd,
                 _p(c.sq64 if self.sq else None), _p(pot_cols), c.log2w.data_ptr(),
                 c.plan_order().data_ptr(), c.n, self.rec.data_ptr(), _stream())
            return
        feat, sq = c.feat(prec)
        call("cntgw_prep_cols", state.ptr, prec, self.kd, int(self.sq), feat.data_ptr(), self.kd,
             _p(sq), _p(pot_cols), c.log2w.data_ptr(), c.n, self.rec.data_ptr(), _stream())

    def stream(self, state: SweepState, out=None, skip=True, row_add=None, out_max=None,
               out_sum=None):
        r = self.rows
        if self.prec == F32C:
            sq = r.sq64 if self.sq else None
            call("cntgw_prep_rows_ctr", self.kd, int(self.sq), r.feat64.data_ptr(), self.kd, _p(sq),
                 r.locality().data_ptr(), r.n, self.ctr_rows.data_ptr(), _stream())
            feat, rec = self.ctr_rows, self.ctr_cols
        elif self.prec == F64S:
            sq = r.sq64 if self.sq else None
            if not self.rows_hoisted:
                self._prep_rows_f64s()
            feat, rec = self.f64s_rows, self.rec
        else:
            feat, sq = r.feat(self.prec)
            rec = self.rec
        call("cntgw_softmin", state.ptr, int(skip), self.prec, self.kd, int(self.sq),
             feat.data_ptr(), self.kd, _p(sq), _p(row_add), rec.data_ptr(), r.n, self.cols.n,
             _p(out), _p(out_max), _p(out_sum), self.ws.data_ptr(), self.ws.numel(), _stream())

    def _prep_rows_f64s(self):
        r = self.rows
        call("cntgw_prep_rows_f64s", self.kd, int(self.sq), r.feat64.data_ptr(), self.kd,
             _p(r.sq64 if self.sq else None), r.plan_order().data_ptr(), r.n, self.f64s_rows.data_ptr(),
             _stream())

    def hoist_rows(self):
        """Gather the F64S rows block now and skip the per-call gather until
        ``rows_hoisted`` is cleared (the owner clears it whenever the row
        features or their order change)."""
        if self.prec == F64S:
            self._prep_rows_f64s()
            self.rows_hoisted = True

    def __call__(self, state, pot_cols, out, skip=True, row_add=None):
        self.pack(state, pot_cols)
        self.stream(state, out, skip=skip, row_add=row_add)

    def partials(self, state, pot_cols, out_max, out_sum, skip=True):
        """Per-row partial LSE pairs (log2 units) over this operator's columns."""
        self.pack(state, pot_cols)
        self.stream(state, None, skip=skip, out_max=out_max, out_sum=out_sum)

    def finalize(self, state, mx, sm, out, skip=True, row_add=None):
        call("cntgw_lse_finalize", state.ptr, int(skip), self.prec, mx.data_ptr(), sm.data_ptr(),
             _p(row_add), out.numel(), out.data_ptr(), _stream())


class DenseHalfUpdate:
    """Half-update over an explicit fp64 cost matrix (DenseCost provider,
    reference sinkhorn.py:30-56 keeps it in float64)."""

    def __init__(self, cost: torch.Tensor, cols_log2w: torch.Tensor):
        self.cost = cost.contiguous()
        self.log2w = cols_log2w
        self.prec = F64

    def __call__(self, state, pot_cols, out, skip=True, row_add=None):
        n, m = self.cost.shape
        call("cntgw_softmin_dense", state.ptr, int(skip), self.cost.data_ptr(), m,
             pot_cols.data_ptr(), self.log2w.data_ptr(), _p(row_add), n, m, out.data_ptr(),
             _stream())


@dataclass
class LoopConfig:
    eps: float
    mode: str = "symmetrized"
    n_inner: int | None = None
    threshold: float | None = None
    max_inner: int = 10000
    anneal_from: float | None = None

    @property
    def max_sweeps(self) -> int:
        return self.max_inner if self.threshold is not None else self.n_inner


@dataclass
class LoopStats:
    iterations: int
    converged: bool
    eps_eff: float
    broke: bool
    lam: float


class SinkhornLoop:
    """Device Sinkhorn loop over two half-update operators (sinkhorn.py:191-258).

    ``fwd(state, g, out)`` computes the f-tentative from g, ``bwd(state, f, out)``
    the g-tentative from f; ``comm`` (optional) turns the g-update into the
    row-sharded form (partial LSE + all-reduce), see dist.py.
    """

    def __init__(self, fwd, bwd, a_w: torch.Tensor, b_w: torch.Tensor, device, comm=None):
        self.fwd, self.bwd, self.comm = fwd, bwd, comm
        self.a_w, self.b_w = a_w, b_w
        self.n, self.m = a_w.numel(), b_w.numel()
        self.state = SweepState(device)
        self.ft = torch.zeros(self.n, dtype=torch.float64, device=device)
        self.gt = torch.zeros(self.m, dtype=torch.float64, device=device)
        # row-gap partials sized for the largest shard (same length on every rank)
        self.gap_n = comm.gap_rows(self.n) if comm is not None else self.n
        self.pr = torch.zeros(LIB.cntgw_gap_blocks(self.gap_n), dtype=torch.float64, device=device)
        self.pc = torch.zeros(LIB.cntgw_gap_blocks(self.m), dtype=torch.float64, device=device)
        self._graphs = {}

    def set_precision(self, prec: int):
        for op in (self.fwd, self.bwd):
            if isinstance(op, HalfUpdate):
                op.prec = prec
                op.rows_hoisted = False

    def hoist_rows(self):
        """Once per loop (fixed features, order and path): see HalfUpdate.hoist_rows."""
        for op in (self.fwd, self.bwd):
            if isinstance(op, HalfUpdate):
                op.hoist_rows()

    def unhoist_rows(self):
        for op in (self.fwd, self.bwd):
            if isinstance(op, HalfUpdate):
                op.rows_hoisted = False

    # -- one sweep (every launch is a no-op once the state says done) --------
    def _g_update(self, f, out, skip=True):
        if self.comm is None:
            self.bwd(self.state, f, out, skip=skip)
        else:
            self.comm.g_update(self, f, out, skip=skip)

    def _gap(self, w, pot, tent, partials):
        call("cntgw_sweep_gap", self.state.ptr, w.data_ptr(), pot.data_ptr(), tent.data_ptr(),
             pot.numel(), partials.data_ptr(), _stream())

    def sweep(self, f, g, mode):
        st = self.state
        st.begin()
        if mode == "symmetrized":
            self.fwd(st, g, self.ft)
            self._g_update(f, self.gt)
            self._gap(self.a_w, f, self.ft, self.pr)
            self._gap(self.b_w, g, self.gt, self.pc)
            pr, nr = (self.pr, self.n) if self.comm is None else self.comm.reduce_gap_partials(self)
            call("cntgw_sweep_finish", st.ptr, pr.data_ptr(), nr, self.pc.data_ptr(), self.m, _stream())
            call("cntgw_sweep_apply", st.ptr, f.data_ptr(), self.ft.data_ptr(), self.n, 1, _stream())
            call("cntgw_sweep_apply", st.ptr, g.data_ptr(), self.gt.data_ptr(), self.m, 1, _stream())
        else:
            self.fwd(st, g, self.ft)
            self._gap(self.a_w, f, self.ft, self.pr)
            pr, nr = (self.pr, self.n) if self.comm is None else self.comm.reduce_gap_partials(self)
            call("cntgw_sweep_finish", st.ptr, pr.data_ptr(), nr, 0, 0, _stream())
            call("cntgw_sweep_apply", st.ptr, f.data_ptr(), self.ft.data_ptr(), self.n, 0, _stream())
            self._g_update(f, g)

    def run(self, f, g, cfg: LoopConfig, chunk: int | None = None, use_graph: bool = False) -> LoopStats:
        """Run the loop to completion; f, g (fp64 interaction potentials) update in place."""
        self.state.init(cfg.eps, cfg.anneal_from, cfg.threshold, cfg.max_sweeps, cfg.mode)
        total = cfg.max_sweeps
        if chunk is None:
            chunk = total if cfg.threshold is None else min(total, 16)
        launched = 0
        while launched < total:
            k = min(chunk, total - launched)
            if use_graph:
                self._replay(f, g, cfg.mode, k)
            else:
                for _ in range(k):
                    self.sweep(f, g, cfg.mode)
            launched += k
            if cfg.threshold is not None and launched < total and self.state.done_flag():
                break
        self.state.begin()  # marks a fully used budget as done
        s = self.state.read()
        broke = bool(s.converged) and cfg.threshold is not None
        return LoopStats(iterations=int(s.applied), converged=bool(s.converged),
                         eps_eff=float(s.eps_n), broke=broke, lam=float(s.lam_d))

    def _replay(self, f, g, mode, k):
        prec = tuple(getattr(op, "prec", None) for op in (self.fwd, self.bwd))
        # (a graph captured with hoisted rows holds no row gather and bias-only column packs:
        # it must not serve a caller that did not hoist)
        hoisted = tuple(getattr(op, "rows_hoisted", False) for op in (self.fwd, self.bwd))
        key = (f.data_ptr(), g.data_ptr(), mode, k, prec, hoisted)
        graph = self._graphs.get(key)
        if graph is None:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=side):
                for _ in range(k):
                    self.sweep(f, g, mode)
            torch.cuda.current_stream().wait_stream(side)
            self._graphs[key] = graph
        graph.replay()

    def tentatives_g(self, f, skip=True):
        """g-tentative of the current pair into self.gt (row-sharded: exchange)."""
        self._g_update(f, self.gt, skip=skip)

    def tentatives(self, f, g, need_f=True, need_g=True):
        """f/g tentatives of the current pair at the loop's final lambda (no skip)."""
        if need_f:
            self.fwd(self.state, g, self.ft, skip=False)
        if need_g:
            self._g_update(f, self.gt, skip=False)
        return self.ft, self.gt

    def marginal_error(self, f, g, lam):
        """Unweighted L1 error ||r - a||_1 + ||c - b||_1 from the tentatives (fp64)."""
        r = self.a_w * torch.exp2(lam * (f - self.ft))
        c = self.b_w * torch.exp2(lam * (g - self.gt))
        err_r = (r - self.a_w).abs().sum()
        if self.comm is not None:
            err_r = self.comm.all_sum(err_r)
        return float(err_r + (c - self.b_w).abs().sum())
