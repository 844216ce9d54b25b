"""Multi-GPU host logic (one process per GPU, torch.distributed for the plumbing).

The PSCWin layer shards across images with no data-path collective ("weak" scaling): each rank
processes its own images; the only collectives are the timing reduction (max over ranks) and barriers.
These helpers are backend-agnostic (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import os
from typing import Tuple


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_range(n_items: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) share of n_items for `rank` (sizes differ by at most one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def image_seed(global_index: int) -> int:
    """Input seed of the image with global index i (identical whichever rank processes it)."""
    return global_index


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (the step time); identity without an initialised process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------------------------- window-row bands
def band_rows(H: int, window: int, world: int):
    """Split the H token rows of one image into `world` contiguous bands of whole window rows. A ragged remainder
    (H % window rows) joins the last full window row, so every band holds at least `window` rows: a band must hold
    the halo rows its neighbours need (up to window - 1 from each edge; pscwin_band_io_offsets rejects a band
    shorter than that). Returns [(row_begin, row_end)] in rank order."""
    units = max(H // window, 1)        # window rows; the last one absorbs the ragged tail
    if world <= 0 or world > units:
        raise ValueError(f"cannot split {H} rows ({units} whole window rows) over {world} ranks")
    out = []
    for r in range(world):
        lo, hi = shard_range(units, world, r)
        out.append((lo * window, H if hi == units else hi * window))
    return out


class TorchDistExchange:
    """The three inter-rank transfers of the band path (include/pscwin.h "row bands") over torch.distributed:
    NCCL on the GPU box (device tensors, NVLink), gloo in the CPU tests. Tensors are byte views of the ranks'
    workspaces; sizes agree pairwise by construction (pscwin_band_io_offsets)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _p2p(self, ops):
        ops = [op for op in ops if op is not None]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def ring(self, send, recv):
        """conv history: rank g's send -> rank (g+1) mod world's recv."""
        if self.world == 1:
            recv.copy_(send)
            return
        nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        self._p2p([self.dist.P2POp(self.dist.isend, send, nxt, self.group),
                   self.dist.P2POp(self.dist.irecv, recv, prv, self.group)])

    def allgather(self, send, recv):
        """scan records: recv = concat over ranks (rank order) of send."""
        if self.world == 1:
            recv.copy_(send)
            return
        self.dist.all_gather(list(recv.view(self.world, -1).unbind(0)), send, group=self.group)

    def halo(self, send_prev, send_next, recv_prev, recv_next):
        """QKV halo: send_prev -> rank-1's recv_next, send_next -> rank+1's recv_prev (empty at the edges)."""
        d, ops = self.dist, []
        if send_prev.numel():
            ops.append(d.P2POp(d.isend, send_prev, self.rank - 1, self.group))
        if send_next.numel():
            ops.append(d.P2POp(d.isend, send_next, self.rank + 1, self.group))
        if recv_prev.numel():
            ops.append(d.P2POp(d.irecv, recv_prev, self.rank - 1, self.group))
        if recv_next.numel():
            ops.append(d.P2POp(d.irecv, recv_next, self.rank + 1, self.group))
        self._p2p(ops)
