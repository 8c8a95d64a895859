"""Multi-GPU plumbing for the hot path.

Records shard by contiguous index ranges, exactly the reference's worker
slicing (rate_engine.cpp:341-344: boundaries ``n*i/workers``); each rank
accumulates its shard into its own device partials (K2). The combine is two
small all-reduces over NCCL (NVLink), the two rounds of the exact median:

  round 1  sums / min / max / coarse  -> every rank holds the global
           per-site sums and the global super-bucket counts;
  (each rank: ``Engine.prepare_median`` finds every site's median
           super-bucket from the global coarse counts and counts its OWN
           flows inside it, from its own per-flow log)
  round 2  fine                       -> the global counts of those 64
           buckets; every rank can then finalize (K3b).

Payload at 10k sites: ~0.4 MB of sums + 6.3 MB coarse + 2.6 MB fine, instead
of 400 MB of dense histograms. The combine is exact by construction: the
per-site state is a commutative monoid (integer sums as 32-bit limbs in
64-bit lanes, f64 min/max, u32 counts), and the median
super-bucket every rank derives from the same reduced coarse counts is the
same.

Partials layout (gnetmon.h, gnm_partials):
  sums     int64 [n_sites*4 + 4]   SUM  (octets, ubps limb0/1/2 per site; tallies)
  min_bps  float64 [n_sites]       MIN  (+inf when empty)
  max_bps  float64 [n_sites]       MAX  (0 when empty)
  coarse   int32 [157*n_sites]     SUM  (flows per (super-bucket, site), sb-major)
  fine     int32 [n_sites*64]      SUM  (after prepare_median)
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank's shard: the reference's boundaries n*i/workers."""
    return n * rank // world, n * (rank + 1) // world


def allreduce_partials(t: dict, group=None) -> None:
    """Round 1: in-place all-reduce of one rank's sums, min/max and coarse
    counts (torch tensors on any device the group's backend supports: CUDA
    for NCCL, CPU for gloo)."""
    dist.all_reduce(t["sums"], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(t["coarse"], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(t["min_bps"], op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(t["max_bps"], op=dist.ReduceOp.MAX, group=group)


def allreduce_fine(t: dict, group=None) -> None:
    """Round 2: all-reduce of the median super-buckets' fine counts."""
    dist.all_reduce(t["fine"], op=dist.ReduceOp.SUM, group=group)


def combine(engine, catalog, group=None, stream=None) -> None:
    """The whole combine for one rank's engine: round 1, prepare, round 2
    (and, in per-host mode, the same for the (site, host) rows).
    ``stream``: the torch stream wrapping the engine's stream (collectives
    are ordered after K2 on it)."""
    t = engine.device_tensors(catalog)
    stream = _engine_stream(engine, t, stream)
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        allreduce_partials(t, group)
    engine.prepare_median(catalog)
    with ctx:
        allreduce_fine(t, group)
    if getattr(engine, "_hosts", False):
        combine_hosts(engine, catalog, group, stream)


def key_union(local: torch.Tensor, group=None) -> torch.Tensor:
    """Sorted union of every rank's sorted int64 keys (variable lengths)."""
    world = dist.get_world_size(group)
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = max(int(x.item()) for x in sizes)
    pad = torch.full((max(m, 1),), -1, dtype=torch.int64, device=local.device)
    pad[:local.numel()] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    allk = torch.cat([p[:int(k.item())] for p, k in zip(parts, sizes)])
    return torch.unique(allk, sorted=True)


def combine_hosts(engine, catalog, group=None, stream=None) -> None:
    """Per-host rows across ranks (gnetmon.h gnm_hosts_*): the union of the
    ranks' (site, host) keys, then the two rounds of the exact median on
    the union's rows. Keys are site << 32 | host (< 2^63: int64 order is
    the key order)."""
    local = engine.hosts_local_keys(catalog)
    union = key_union(local, group)
    t = engine.hosts_set_keys(union)
    stream = _engine_stream(engine, t, stream)
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        dist.all_reduce(t["sums"], op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t["coarse"], op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t["min_bps"], op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(t["max_bps"], op=dist.ReduceOp.MAX, group=group)
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    engine.hosts_prepare_median()
    with ctx:
        dist.all_reduce(t["fine"], op=dist.ReduceOp.SUM, group=group)
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()


def _engine_stream(engine, t: dict, stream):
    """The stream the collectives run on: the caller's, else -- for CUDA
    partials -- the engine's own stream, so the all-reduces are ordered after
    K2 and before K3a/K2b/K3b (the engine launches on a non-blocking stream
    that torch's current stream does not order against)."""
    if stream is not None or not t["sums"].is_cuda or not hasattr(engine, "stream_handle"):
        return stream
    return torch.cuda.ExternalStream(engine.stream_handle(), device=t["sums"].device)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def limbs_to_int(sums: torch.Tensor, n_sites: int) -> list[tuple[int, int]]:
    """(octets, exact micro-bps) per site from the reduced limb sums."""
    s = sums.cpu().tolist()
    return [(s[4 * i], s[4 * i + 1] + (s[4 * i + 2] << 32) + (s[4 * i + 3] << 64))
            for i in range(n_sites)]
