"""Row-sharded multi-GPU execution.

One process per GPU. The N source rows are partitioned contiguously across
ranks; target features, the target potential g and Gamma are replicated. Per
Sinkhorn sweep:

  * f-update: local (own rows against all M columns), no communication;
  * g-update: every rank streams its local rows into per-column partial LSE
    pairs (m_j, s_j) (``cntgw_softmin`` with out_max/out_sum), then the
    exchange step M_j = max_ranks m_j, s_j <- s_j 2^(m_j - M_j),
    S_j = sum_ranks s_j, and ``cntgw_lse_finalize`` — every rank ends with
    the identical full g, so no broadcast is needed;
  * threshold check: the row-gap partials are summed over ranks; the column
    gap is computed redundantly on every rank.

The outer step sums Gamma_{t+1}, the KL/objective terms and the row error
over ranks with one all-reduce of a (16 + D*E)-double buffer.

Two transports carry the exchanges:

  * ``NativeComm`` (NCCL over NVLink/NVSwitch on the GPU box): the library's
    own NCCL communicator (``cntgw_comm_*``, csrc/comm.cu), every collective
    enqueued on the compute stream by the C ABI, so the sharded solve is
    captured as ONE CUDA graph like the single-GPU one (solvers._DeviceSolve);
  * torch.distributed (gloo: the CPU tests and host-mediated functional runs
    of several ranks on one GPU), driven from the host loop.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class DistInfo:
    rank: int = 0
    world: int = 1
    local_rank: int = 0

    @property
    def enabled(self) -> bool:
        return self.world > 1


def init_from_env(backend: str | None = None) -> DistInfo:
    """Initialise torch.distributed from torchrun's environment (no-op at world 1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return DistInfo(rank=rank, world=world, local_rank=local)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous near-equal split of n rows: rank r owns [lo, hi)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def combine_partial_lse(mx: torch.Tensor, sm: torch.Tensor, group=None) -> None:
    """In-place cross-rank merge of per-column partial LSE pairs (log2 units)
    over torch.distributed: after the call every rank holds (M_j, S_j) with
    2^M_j S_j = sum_ranks 2^m_j s_j. Ranks with an empty (-inf, 0) partial
    contribute nothing. On CUDA tensors the rescale is the library's
    ``cntgw_lse_rescale`` kernel; CPU tensors (the gloo tests' stand-in
    operators) take the same arithmetic in torch."""
    local = mx.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    if mx.is_cuda:
        from ._native import call

        call("cntgw_lse_rescale", local.data_ptr(), mx.data_ptr(), sm.data_ptr(), sm.numel(), _stream())
    else:
        keep = (sm > 0) & (local > -torch.inf)
        sm.copy_(torch.where(keep, sm * torch.exp2(local - mx), torch.zeros_like(sm)))
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)


def native_comm_wanted() -> bool:
    """The library's own NCCL communicator is used under an NCCL process group
    (CNTGW_NATIVE_COMM=0 keeps torch.distributed's collectives)."""
    if os.environ.get("CNTGW_NATIVE_COMM", "1") == "0" or not torch.cuda.is_available():
        return False
    return dist.is_available() and dist.is_initialized() and dist.get_backend() == "nccl"


class NativeComm:
    """NCCL communicator of libcntgw_b200.so (csrc/comm.cu): collectives on the
    caller's stream, capturable inside the solve's CUDA graph. ``world == 1``
    builds a single-rank communicator without torch.distributed (used to run
    the sharded code path on one GPU)."""

    def __init__(self, info: DistInfo):
        from ._native import LIB, call

        if not LIB.cntgw_comm_available():
            raise RuntimeError("libnccl.so.2 could not be resolved for the native communicator")
        self.info = info
        nbytes = int(LIB.cntgw_comm_id_bytes())
        uid = ctypes.create_string_buffer(nbytes)
        if info.rank == 0:
            call("cntgw_comm_unique_id", uid)
        if info.world > 1:
            box = [uid.raw if info.rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            uid = ctypes.create_string_buffer(box[0], nbytes)
        handle = ctypes.c_void_p()
        call("cntgw_comm_init", ctypes.byref(handle), info.world, info.rank, uid)
        self.handle = handle.value
        self._call = call

    def allreduce(self, send: torch.Tensor, recv: torch.Tensor | None = None, op: str = "sum"):
        recv = send if recv is None else recv
        self._call("cntgw_comm_allreduce", self.handle, send.data_ptr(), recv.data_ptr(), send.numel(),
                   1 if op == "max" else 0, _stream())

    def combine_lse(self, m_local: torch.Tensor, m_glob: torch.Tensor, sm: torch.Tensor):
        self._call("cntgw_comm_combine_lse", self.handle, m_local.data_ptr(), m_glob.data_ptr(),
                   sm.data_ptr(), sm.numel(), _stream())

    def close(self):
        if getattr(self, "handle", None):
            self._call("cntgw_comm_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RowShardComm:
    """Collective hooks the device loop calls when rows are sharded.

    ``native`` (a NativeComm) makes every hook a stream-ordered C-ABI call
    (graph-capturable); without it the hooks use torch.distributed from the
    host. ``n_rows_max`` is the largest shard, so that the gap partials have
    the same length on every rank."""

    def __init__(self, info: DistInfo, group=None, native: NativeComm | None = None,
                 n_rows_max: int | None = None):
        self.info = info
        self.group = group
        self.native = native
        self.n_rows_max = n_rows_max
        self._bufs = {}

    @property
    def capturable(self) -> bool:
        return self.native is not None

    def _buf(self, name, n, device):
        t = self._bufs.get(name)
        if t is None or t.numel() != n or t.device != device:
            t = torch.zeros(n, dtype=torch.float64, device=device)
            self._bufs[name] = t
        return t

    def prepare(self, m: int, n_partials: int, device) -> None:
        """Allocate the exchange buffers up front (never inside a graph capture)."""
        for name, n in (("mx", m), ("sm", m), ("mglob", m), ("prglob", n_partials)):
            self._buf(name, n, device)

    def gap_rows(self, n_local: int) -> int:
        return max(n_local, self.n_rows_max or 0)

    def g_update(self, loop, f, out, skip=True):
        """g-tentative over all ranks' rows: partial LSE, exchange, finalize."""
        bwd = loop.bwd
        mx = self._buf("mx", out.numel(), out.device)
        sm = self._buf("sm", out.numel(), out.device)
        bwd.partials(loop.state, f, mx, sm, skip=skip)
        if self.native is not None:
            mg = self._buf("mglob", out.numel(), out.device)
            self.native.combine_lse(mx, mg, sm)
            bwd.finalize(loop.state, mg, sm, out, skip=skip)
        else:
            combine_partial_lse(mx, sm, self.group)
            bwd.finalize(loop.state, mx, sm, out, skip=skip)

    def reduce_gap_partials(self, loop):
        """Row-gap partials summed over ranks; returns (partials, rows) for
        cntgw_sweep_finish."""
        if self.native is not None:
            glob = self._buf("prglob", loop.pr.numel(), loop.pr.device)
            self.native.allreduce(loop.pr, glob)  # out of place: no feedback into pr
            return glob, loop.gap_n
        total = loop.pr.sum().reshape(1)
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=self.group)
        loop.pr.zero_()
        loop.pr[:1].copy_(total)
        return loop.pr, loop.gap_n

    def allreduce_(self, t: torch.Tensor) -> None:
        """In-place SUM over ranks (stream-ordered with the native comm)."""
        if self.native is not None:
            self.native.allreduce(t)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def allmax_(self, t: torch.Tensor) -> None:
        if self.native is not None:
            self.native.allreduce(t, op="max")
        else:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)

    def all_sum(self, t: torch.Tensor) -> torch.Tensor:
        t = t.clone().reshape(-1)
        self.allreduce_(t)
        return t if t.numel() > 1 else t[0]
