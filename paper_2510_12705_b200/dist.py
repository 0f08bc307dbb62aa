"""Multi-GPU batch driver pieces: one process per GPU, batches of
independent matrices partitioned across ranks, results gathered with one
collective.  A single matrix never spans GPUs (its sweeps are ordered; a
cross-GPU hop would sit on the critical path every cycle).

The only data-path collective is the final all-gather of (d, e) -- NCCL over
NVLink on the GPU box, gloo in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition(batch: int, world: int, rank: int):
    """Contiguous near-even split of `batch` matrices: rank gets
    [start, start + count); the first batch % world ranks get one extra."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad partition arguments")
    base, extra = divmod(batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def gather_results(d: torch.Tensor, e: torch.Tensor, world: int, counts=None):
    """All-gather every rank's (d, e) slices.  d: (B_r, n), e: (B_r, n-1).
    Ranks may hold different counts (uneven split): tensors are padded to
    the max count so one fixed-shape all_gather_into_tensor suffices.
    Returns (D, E) of shape (sum B_r, n) / (sum B_r, n-1) on every rank."""
    if world == 1:
        return d, e
    n = d.shape[1]
    ne = e.shape[1]
    if counts is None:
        c = torch.tensor([d.shape[0]], dtype=torch.int64, device=d.device)
        allc = [torch.zeros_like(c) for _ in range(world)]
        dist.all_gather(allc, c)
        counts = [int(x.item()) for x in allc]
    mx = max(counts)
    buf = torch.zeros(mx, n + ne, dtype=d.dtype, device=d.device)
    buf[: d.shape[0], :n] = d
    buf[: e.shape[0], n:] = e
    out = torch.empty(world * mx, n + ne, dtype=d.dtype, device=d.device)
    dist.all_gather_into_tensor(out, buf)
    parts = [out[r * mx: r * mx + counts[r]] for r in range(world)]
    cat = torch.cat(parts, 0)
    return cat[:, :n], cat[:, n:]
