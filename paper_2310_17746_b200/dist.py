"""torch.distributed mirror of the library's multi-device combine, for
callers that shard [L, R) across their own processes instead of handing
devices to one ws_ctx (the library's own path: Sieve(devices=..., world=...),
which runs ONE ncclAllGather inside libwheelsieve_cuda.so).

Same contract as the library: contiguous ws_partition super-ranges, and one
all_gather of the 32-byte record {count, sum, xor, largest} per rank folded
by ws_combine_checks (NCCL has no XOR reduction).  Works with the nccl
backend (GPU tensors) and gloo (CPU tensors, used by the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from .wheelsieve import Checks, combine_checks as _fold, partition

MASK = (1 << 64) - 1


def _dev():
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _to_i64(x: int) -> int:
    x &= MASK
    return x - (1 << 64) if x >= 1 << 63 else x


def combine_checks(local: Checks, group=None) -> Checks:
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rec = torch.tensor([_to_i64(local.count), _to_i64(local.sum), _to_i64(local.xor),
                        _to_i64(local.largest)], dtype=torch.int64, device=_dev())
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec, group=group)
    allr = torch.stack(out).cpu().numpy().view(np.uint64)
    return _fold([Checks(*(int(v) for v in row)) for row in allr])


def max_over_ranks(v: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(v: int, group=None) -> int:
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.int64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def sharded_count(L: int, R: int, rank: int, world: int,
                  local_fn: Optional[Callable[[int, int], Checks]] = None,
                  segment_slots: int = 1 << 18, group=None) -> Checks:
    """Count (with checksums) [L, R) split into contiguous per-rank
    super-ranges (ws_partition); local_fn(lo, hi) sieves the rank's share
    (default: a GPU Sieve on the current device).  No data-path exchange:
    one all_gather of the 32-byte result records at the end."""
    lo, hi = partition(L, R, rank, world, segment_slots)
    if local_fn is None:
        from .wheelsieve import Sieve
        import torch
        with Sieve(device=torch.cuda.current_device(), segment_slots=segment_slots) as sv:
            local = sv.count_range(lo, hi, checks=True)
    else:
        local = local_fn(lo, hi)
    return combine_checks(local, group)
