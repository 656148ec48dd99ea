"""Row-sharded multi-GPU execution.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the GPU
box; gloo in the CPU tests). The N source rows are partitioned contiguously
across ranks; target features, the target potential g and Gamma are
replicated. Per Sinkhorn sweep:

  * f-update: local (own rows against all M columns), no communication;
  * g-update: every rank streams its local rows into per-column partial LSE
    pairs (m_j, s_j) (``cntgw_softmin`` with out_max/out_sum), then
    all-reduce MAX of m, local rescale s_j <- s_j 2^(m_j - M_j), all-reduce
    SUM of s, and ``cntgw_lse_finalize`` — every rank ends with the identical
    full g, so no broadcast is needed;
  * threshold check: the row gap is an all-reduce SUM of one scalar; the
    column gap is computed redundantly on every rank.

The outer step reduces Gamma_{t+1}, the KL/objective terms and the row error
with one all-reduce SUM of a (16 + D*E)-double buffer.
"""

from __future__ import annotations

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


def combine_partial_lse(mx: torch.Tensor, sm: torch.Tensor, group=None) -> None:
    """In-place cross-rank merge of per-column partial LSE pairs (log2 units):
    after the call every rank holds (M_j, S_j) with
    2^M_j S_j = sum_ranks 2^m_j s_j. Ranks with an empty (-inf, 0) partial
    contribute nothing."""
    local = mx.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    scale = torch.exp2(local - mx)
    scale = torch.where(sm > 0, scale, torch.zeros_like(scale))
    sm.mul_(scale)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)


class RowShardComm:
    """Collective hooks the device loop calls when rows are sharded."""

    def __init__(self, info: DistInfo, group=None):
        self.info = info
        self.group = group
        self._bufs = {}

    def _buf(self, name, n, device):
        t = self._bufs.get(name)
        if t is None or t.numel() != n or t.device != device:
            t = torch.empty(n, dtype=torch.float64, device=device)
            self._bufs[name] = t
        return t

    def g_update(self, loop, f, out, skip=True):
        """g-tentative over all ranks' rows (partial LSE + two all-reduces)."""
        bwd = loop.bwd
        mx = self._buf("mx", out.numel(), out.device)
        sm = self._buf("sm", out.numel(), out.device)
        bwd.partials(loop.state, f, mx, sm, skip=skip)
        combine_partial_lse(mx, sm, self.group)
        bwd.finalize(loop.state, mx, sm, out, skip=skip)

    def reduce_gap_partials(self, loop):
        """Row gap = sum over ranks; the total goes into slot 0 of the partials."""
        total = loop.pr.sum().reshape(1)
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=self.group)
        loop.pr.zero_()
        loop.pr[:1].copy_(total)

    def all_sum(self, t: torch.Tensor) -> torch.Tensor:
        t = t.clone().reshape(-1)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t if t.numel() > 1 else t[0]
