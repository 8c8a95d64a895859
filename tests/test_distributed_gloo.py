"""The N>1 path on CPU: two gloo ranks shard the records by index
(rate_engine.cpp:341-344 boundaries), build per-rank partials in the device
layout (gnetmon.h gnm_partials), and run the two-round exact-median combine
with the same functions bench.py uses on NCCL: all-reduce of sums / min /
max / coarse counts, each rank's median super-bucket and its own fine counts
inside it (here from the rank's oracle histograms; on the GPU K3a + K2b from
the rank's log), all-reduce of the fine counts. The combined result equals
the single-process oracle bit-exactly (SPEC.md:310 partition independence)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import parity
from paper_1108_1785_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


COARSE, FINE = 157, 64


def partials_from_oracle(acc, n_sites):
    """Oracle accumulators -> the device partial layout (limbs in int64 lanes,
    coarse counts sb-major)."""
    sums = np.zeros(n_sites * 4 + 4, np.int64)
    lo = acc["ubps_lo"].astype(np.uint64)
    sums[0:4 * n_sites:4] = acc["octets"].astype(np.int64)
    sums[1:4 * n_sites:4] = (lo & np.uint64(0xFFFFFFFF)).astype(np.int64)
    sums[2:4 * n_sites:4] = (lo >> np.uint64(32)).astype(np.int64)
    sums[3:4 * n_sites:4] = acc["ubps_hi"].astype(np.int64)
    sums[4 * n_sites:] = acc["tallies"].astype(np.int64)
    hist = acc["hist"].astype(np.int64)
    padded = np.zeros((n_sites, COARSE * FINE), np.int64)
    padded[:, :hist.shape[1]] = hist
    coarse = padded.reshape(n_sites, COARSE, FINE).sum(axis=2).T.reshape(-1)
    return {"sums": torch.from_numpy(sums), "min_bps": torch.from_numpy(acc["min"].copy()),
            "max_bps": torch.from_numpy(acc["max"].copy()),
            "coarse": torch.from_numpy(coarse.astype(np.int32)),
            "fine": torch.zeros(n_sites * FINE, dtype=torch.int32)}, padded


def median_superbucket(coarse, n_sites):
    """K3a's rule: the first super-bucket whose cumulative count reaches
    ceil(count/2), and the median's rank inside it."""
    c = coarse.reshape(COARSE, n_sites).T.astype(np.int64)
    cnt = c.sum(axis=1)
    target = (cnt + 1) // 2
    cum = np.cumsum(c, axis=1)
    msb = np.argmax(cum >= target[:, None], axis=1)
    before = np.where(msb > 0, cum[np.arange(n_sites), msb - 1], 0)
    return cnt, msb, target - before


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle import Oracle
    orc = Oracle()
    sites, cols = parity.engine_stress_set(30_000, seed=77)
    from paper_1108_1785_b200 import SiteCatalog
    cat = SiteCatalog()
    for i, c in enumerate(sites):
        cat.register_site(f"s{i}", c)
    p, s = cat.entries_arrays()
    oc = orc.catalog(p, s)
    b, e = D.shard_range(len(cols[0]), rank, world)
    acc = orc.aggregate(tuple(c[b:e] for c in cols), oc, len(sites))
    n = len(sites)
    t, dense = partials_from_oracle(acc, n)
    D.allreduce_partials(t)                       # round 1
    cnt, msb, rank_in = median_superbucket(t["coarse"].numpy(), n)
    own = dense.reshape(n, COARSE, FINE)[np.arange(n), msb]  # this rank's flows in it
    t["fine"].copy_(torch.from_numpy(own.reshape(-1).astype(np.int32)))
    D.allreduce_fine(t)                           # round 2
    if rank == 0:
        fine = t["fine"].numpy().astype(np.int64).reshape(n, FINE)
        j = np.argmax(np.cumsum(fine, axis=1) >= rank_in[:, None], axis=1)
        k = msb * FINE + j
        mn, mx = t["min_bps"].numpy(), t["max_bps"].numpy()
        med = np.where(k == 10000, 1e8, k * 10000.0 + 5000.0)
        med = np.minimum(np.maximum(med, mn), mx)
        per = D.limbs_to_int(t["sums"], n)
        want = orc.finalize(orc.aggregate(cols, oc, n))
        present = cnt > 0
        ok = (np.array_equal(cnt.astype(np.uint64), np.asarray(want["count"]))
              and np.array_equal(np.array([x[0] for x in per], np.uint64), want["octets"])
              and np.array_equal(np.array([x[1] & (2**64 - 1) for x in per], np.uint64), want["ubps_lo"])
              and np.array_equal(np.array([x[1] >> 64 for x in per], np.uint64), want["ubps_hi"])
              and np.array_equal(mn[present].view(np.uint64), np.asarray(want["min"])[present].view(np.uint64))
              and np.array_equal(mx[present].view(np.uint64), np.asarray(want["max"])[present].view(np.uint64))
              and np.array_equal(med[present].view(np.uint64), np.asarray(want["median"])[present].view(np.uint64))
              and np.array_equal(t["sums"].numpy()[4 * n:].astype(np.uint64), want["tallies"]))
        q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_combine_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


def test_shard_ranges_tile_the_batch():
    for n in (0, 1, 7, 1000, 10**9 + 3):
        for world in (1, 2, 3, 8):
            ranges = [D.shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
