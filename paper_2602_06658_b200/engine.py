"""Device engine: the Sinkhorn loop and fused reductions on one GPU.

Everything here operates on CUDA tensors and launches the C-ABI kernels of
``libcntgw_b200.so`` on torch's current stream. The loop state (sweep counter,
eps_n, threshold decision, done flag) lives in device memory
(``cntgw_sweep_state``), so sweeps are enqueued back to back without host
round trips and chunks of sweeps can be replayed as CUDA graphs; the host
reads the state once per chunk to learn whether a threshold run finished.

Cost model every feature provider reduces to (see include/cntgw_b200.h):
    C_ij = row_sep_i + col_sep_j - 2 <xf_i, zf_j> + (xs_i - zs_j)^2
with interaction potentials f~ = f - row_sep and g~ = g - col_sep on device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import LIB, SweepStateStruct, call

SUPPORTED_KD = (1, 2, 3, 4, 8, 16, 32, 64)


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


def to_dev32(x, device, kd=None) -> torch.Tensor:
    """float32 contiguous device copy, zero-padded to kd columns if given."""
    t = torch.as_tensor(np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x)
    t = t.to(device=device, dtype=torch.float32)
    if kd is not None:
        if t.ndim == 1:
            t = t[:, None]
        if t.shape[1] < kd:
            t = torch.nn.functional.pad(t, (0, kd - t.shape[1]))
    return t.contiguous()


def to_dev64(x, device) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x)
    return t.to(device=device, dtype=torch.float64).contiguous()


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
        host = self.buf.cpu().numpy().tobytes()
        return SweepStateStruct.from_buffer_copy(host)

    def done_flag(self) -> bool:
        off = SweepStateStruct.done.offset
        return bool(self.buf[off:off + 4].cpu().view(torch.int32).item())


@dataclass
class Side:
    """One marginal as the kernels see it (dot features, sq coordinate, weights)."""

    feat: torch.Tensor  # n x kd float32 (zero-padded)
    sq: torch.Tensor | None  # n float32, the squared-difference coordinate
    w: torch.Tensor  # n float64
    log2w: torch.Tensor  # n float32

    @property
    def n(self) -> int:
        return self.feat.shape[0]

    @property
    def kd(self) -> int:
        return self.feat.shape[1]

    @staticmethod
    def make(feat, sq, w, device, kd):
        w64 = to_dev64(w, device)
        return Side(
            feat=to_dev32(feat, device, kd),
            sq=None if sq is None else to_dev32(sq, device),
            w=w64,
            log2w=torch.log2(w64).to(torch.float32),
        )


class HalfUpdate:
    """out_rows = S(pot_cols): pack the column side's records, then stream them."""

    def __init__(self, rows: Side, cols: Side, sq: bool):
        self.rows, self.cols, self.sq = rows, cols, bool(sq)
        self.kd = rows.kd
        assert cols.kd == self.kd
        dev = rows.feat.device
        stride = LIB.cntgw_col_stride(self.kd, int(self.sq))
        _native.check(0 if stride > 0 else stride, "cntgw_col_stride")
        self.stride = stride
        self.rec = torch.empty(LIB.cntgw_cols_padded(cols.n) * stride, dtype=torch.float32, device=dev)
        wsb = LIB.cntgw_softmin_workspace(rows.n, cols.n, self.kd, int(self.sq))
        self.ws = torch.empty(max(int(wsb), 16), dtype=torch.uint8, device=dev)

    def pack(self, state: SweepState, pot_cols: torch.Tensor | None):
        c = self.cols
        call("cntgw_prep_cols", state.ptr, self.kd, int(self.sq), c.feat.data_ptr(), self.kd,
             _p(c.sq), _p(pot_cols), c.log2w.data_ptr(), c.n, self.rec.data_ptr(), _stream())

    def stream(self, state: SweepState, out=None, skip=True, row_add=None, out_max=None,
               out_sum=None):
        r = self.rows
        call("cntgw_softmin", state.ptr, int(skip), self.kd, int(self.sq), r.feat.data_ptr(),
             self.kd, _p(r.sq), _p(row_add), self.rec.data_ptr(), r.n, self.cols.n, _p(out),
             _p(out_max), _p(out_sum), self.ws.data_ptr(), self.ws.numel(), _stream())

    def __call__(self, state, pot_cols, out, skip=True, row_add=None):
        self.pack(state, pot_cols)
        self.stream(state, out, skip=skip, row_add=row_add)


class DenseHalfUpdate:
    """Half-update over an explicit cost matrix (DenseCost provider)."""

    def __init__(self, cost: torch.Tensor, cols_log2w: torch.Tensor):
        self.cost = cost.contiguous()
        self.log2w = cols_log2w

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
        self.ft = torch.zeros(self.n, dtype=torch.float32, device=device)
        self.gt = torch.zeros(self.m, dtype=torch.float32, device=device)
        self.pr = torch.zeros(LIB.cntgw_gap_blocks(self.n), dtype=torch.float64, device=device)
        self.pc = torch.zeros(LIB.cntgw_gap_blocks(self.m), dtype=torch.float64, device=device)
        self._graphs = {}

    # -- one sweep (all launches skip once the state says done) --------------
    def _g_update(self, f, out):
        if self.comm is None:
            self.bwd(self.state, f, out)
        else:
            self.comm.g_update(self, f, out)

    def _gap(self, side, w, pot, tent, partials):
        call("cntgw_sweep_gap", self.state.ptr, side, w.data_ptr(), pot.data_ptr(),
             tent.data_ptr(), pot.numel(), partials.data_ptr(), _stream())

    def sweep(self, f, g, mode):
        st = self.state
        st.begin()
        if mode == "symmetrized":
            self.fwd(st, g, self.ft)
            self._g_update(f, self.gt)
            self._gap(0, self.a_w, f, self.ft, self.pr)
            self._gap(1, self.b_w, g, self.gt, self.pc)
            if self.comm is not None:
                self.comm.reduce_gap_partials(self)
            call("cntgw_sweep_finish", st.ptr, self.pr.data_ptr(), self.n, self.pc.data_ptr(),
                 self.m, _stream())
            call("cntgw_sweep_apply", st.ptr, f.data_ptr(), self.ft.data_ptr(), self.n, 1, _stream())
            call("cntgw_sweep_apply", st.ptr, g.data_ptr(), self.gt.data_ptr(), self.m, 1, _stream())
        else:
            self.fwd(st, g, self.ft)
            self._gap(0, self.a_w, f, self.ft, self.pr)
            if self.comm is not None:
                self.comm.reduce_gap_partials(self)
            call("cntgw_sweep_finish", st.ptr, self.pr.data_ptr(), self.n, 0, 0, _stream())
            call("cntgw_sweep_apply", st.ptr, f.data_ptr(), self.ft.data_ptr(), self.n, 0, _stream())
            self._g_update(f, g)

    def run(self, f, g, cfg: LoopConfig, chunk: int | None = None, use_graph: bool = False) -> LoopStats:
        """Run the loop to completion; f, g (interaction potentials) are updated in place."""
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
        # one more begin() marks a fully used budget as done
        self.state.begin()
        s = self.state.read()
        broke = bool(s.converged) and cfg.threshold is not None
        return LoopStats(iterations=int(s.applied), converged=bool(s.converged),
                         eps_eff=float(s.eps_n), broke=broke, lam=float(s.lam))

    def _replay(self, f, g, mode, k):
        key = (f.data_ptr(), g.data_ptr(), mode, k)
        graph = self._graphs.get(key)
        if graph is None:
            # warm-up launch outside capture sets kernel attributes once
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=side):
                for _ in range(k):
                    self.sweep(f, g, mode)
            torch.cuda.current_stream().wait_stream(side)
            self._graphs[key] = graph
            # the capture did not execute anything: fall through to replay
        graph.replay()

    def tentatives(self, f, g, need_f=True, need_g=True):
        """f/g tentatives of the current pair at the loop's final lambda (no skip)."""
        if need_f:
            self.fwd(self.state, g, self.ft, skip=False)
        if need_g:
            if self.comm is None:
                self.bwd(self.state, f, self.gt, skip=False)
            else:
                self.comm.g_update(self, f, self.gt, skip=False)
        return self.ft, self.gt

    def marginal_error(self, f, g, lam):
        """Unweighted L1 error ||r - a||_1 + ||c - b||_1 from the tentatives (fp64)."""
        lam = float(lam)
        r = self.a_w * torch.exp2(lam * (f.double() - self.ft.double()))
        c = self.b_w * torch.exp2(lam * (g.double() - self.gt.double()))
        err_r = (r - self.a_w).abs().sum()
        if self.comm is not None:
            err_r = self.comm.all_sum(err_r)
        return float(err_r + (c - self.b_w).abs().sum())
