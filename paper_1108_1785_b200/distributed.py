"""Multi-GPU plumbing for the hot path.

Records shard by contiguous index ranges, exactly the reference's worker
slicing (rate_engine.cpp:341-344: boundaries ``n*i/workers``); each rank
accumulates its shard into its own device partials (K2), the partials are
combined with one grouped all-reduce over NCCL (NVLink), and every rank then
runs K3 on the combined partials. The combine is exact by construction: the
per-site state is a commutative monoid (integer sums as 32-bit limbs in
64-bit lanes, f64 min/max, u32 bucket counts).

Partials layout (gnetmon.h, gnm_partials):
  sums     int64 [n_sites*4 + 4]   SUM  (octets, ubps limb0/1/2 per site; tallies)
  min_bps  float64 [n_sites]       MIN  (+inf when empty)
  max_bps  float64 [n_sites]       MAX  (0 when empty)
  hist     int32 [n_sites*10008]   SUM  (sector-blocked bucket-major, see gnetmon.h)
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank's shard: the reference's boundaries n*i/workers."""
    return n * rank // world, n * (rank + 1) // world


def allreduce_partials(t: dict, group=None) -> None:
    """In-place all-reduce of one rank's partials (torch tensors, any device
    the process group's backend supports: CUDA for NCCL, CPU for gloo)."""
    dist.all_reduce(t["sums"], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(t["hist"], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(t["min_bps"], op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(t["max_bps"], op=dist.ReduceOp.MAX, group=group)


def limbs_to_int(sums: torch.Tensor, n_sites: int) -> list[tuple[int, int]]:
    """(octets, exact micro-bps) per site from the reduced limb sums."""
    s = sums.cpu().tolist()
    return [(s[4 * i], s[4 * i + 1] + (s[4 * i + 2] << 32) + (s[4 * i + 3] << 64))
            for i in range(n_sites)]
