"""Cyclic partition of a sweep over ranks (step a8).

The flat index range [begin, end) is cut into calls of `chunk` consecutive
configurations dealt round-robin: rank r sweeps calls r, r + N, r + 2N, ...
on its own (no communicator), and one allgather of every call's survivor count
gives each call its global offset (offset of call q = survivors of calls
0..q-1), so the joined result is still in index order.  Host plumbing only:
the sweeps themselves run in libme.so; the allgather is torch.distributed
(NCCL on the GPU, gloo in the CPU tests)."""
from __future__ import annotations

from typing import List, Sequence, Tuple


def cyclic_calls(begin: int, end: int, chunk: int, rank: int, world: int) -> List[Tuple[int, int]]:
    """The calls of `rank`: [(b, e)] for calls q = rank, rank + world, ..."""
    if chunk <= 0 or world <= 0 or not 0 <= rank < world or end < begin:
        raise ValueError("bad cyclic partition arguments")
    return [(b, min(end, b + chunk)) for b in range(begin, end, chunk)][rank::world]


def n_calls(begin: int, end: int, chunk: int) -> int:
    return -(-(end - begin) // chunk) if end > begin else 0


def cyclic_join(local_counts: Sequence[int], calls_total: int, world: int, device=None, group=None):
    """Allgather the per-call survivor counts of every rank (in this rank's
    call order) and return (offsets, counts, total): offsets[q] and counts[q]
    for every call q of the whole range, as int64 tensors on `device`."""
    import torch
    import torch.distributed as dist

    per_rank = -(-calls_total // world) if calls_total else 0
    cnt = torch.zeros(max(per_rank, 1), dtype=torch.int64, device=device)
    if len(local_counts):
        cnt[:len(local_counts)] = torch.as_tensor(list(local_counts), dtype=torch.int64)
    parts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(parts, cnt, group=group)
    # call q lives on rank q % world in slot q // world
    by_call = torch.stack(parts).t().reshape(-1)[:calls_total]
    return torch.cumsum(by_call, 0) - by_call, by_call, int(by_call.sum())
