"""Sample-index sharding across ranks.

The residual kernels partition the sample indices [0, n) of every (technique, side) block-cyclically:
blocks of SHARD_BLOCK = 2^16 consecutive indices, block b owned by rank b mod world.  The kernel computes the
mapping itself (rr_residual.cu: i = ((blk * shard_count + shard_index) << 16) | off); this module is its
host-side statement, used by tools and by the multi-process tests, and the one NCCL/gloo collective of
the path (the reduction of the per-rank residual images).
"""
from __future__ import annotations

from typing import List, Tuple

SHARD_BLOCK = 1 << 16


def shard_ranges(n: int, shard_index: int, shard_count: int, block: int = SHARD_BLOCK) -> List[Tuple[int, int]]:
    """Half-open index ranges [i0, i1) of [0, n) owned by `shard_index` of `shard_count`."""
    if shard_count < 1 or not 0 <= shard_index < shard_count:
        raise ValueError("bad shard")
    out = []
    b = shard_index
    while b * block < n:
        out.append((b * block, min(n, (b + 1) * block)))
        b += shard_count
    return out


def reduce_image(img, dst: int = 0):
    """Sum the per-rank residual images on `dst` (the path's only collective: NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.reduce(img, dst=dst, op=dist.ReduceOp.SUM)
    return img
