"""The N>1 path on CPU: two gloo ranks shard the records by index
(rate_engine.cpp:341-344 boundaries), build per-rank partials in the device
layout (gnetmon.h gnm_partials), all-reduce them with the same function
bench.py uses on NCCL, and the combined result equals the single-process
oracle bit-exactly (SPEC.md:310 partition independence)."""
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


def partials_from_oracle(acc, n_sites):
    """Oracle accumulators -> the device partial layout (limbs in int64 lanes)."""
    sums = np.zeros(n_sites * 4 + 4, np.int64)
    lo = acc["ubps_lo"].astype(np.uint64)
    sums[0:4 * n_sites:4] = acc["octets"].astype(np.int64)
    sums[1:4 * n_sites:4] = (lo & np.uint64(0xFFFFFFFF)).astype(np.int64)
    sums[2:4 * n_sites:4] = (lo >> np.uint64(32)).astype(np.int64)
    sums[3:4 * n_sites:4] = acc["ubps_hi"].astype(np.int64)
    sums[4 * n_sites:] = acc["tallies"].astype(np.int64)
    return {"sums": torch.from_numpy(sums), "min_bps": torch.from_numpy(acc["min"].copy()),
            "max_bps": torch.from_numpy(acc["max"].copy()),
            "hist": torch.from_numpy(acc["hist"].reshape(-1).astype(np.int32))}


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
    t = partials_from_oracle(acc, len(sites))
    D.allreduce_partials(t)
    if rank == 0:
        n = len(sites)
        hist = t["hist"].numpy().astype(np.uint32).reshape(n, 10001)
        per = D.limbs_to_int(t["sums"], n)
        comb = {"count": hist.sum(axis=1).astype(np.uint64), "octets": np.array([x[0] for x in per], np.uint64),
                "ubps_lo": np.array([x[1] & (2**64 - 1) for x in per], np.uint64),
                "ubps_hi": np.array([x[1] >> 64 for x in per], np.uint64),
                "min": t["min_bps"].numpy(), "max": t["max_bps"].numpy(), "hist": hist,
                "tallies": t["sums"].numpy()[4 * n:].astype(np.uint64)}
        got = orc.finalize(comb)
        want = orc.finalize(orc.aggregate(cols, oc, n))
        ok = all(np.array_equal(np.asarray(got[k]).view(np.uint64) if np.asarray(got[k]).dtype == np.float64
                                else got[k], np.asarray(want[k]).view(np.uint64)
                                if np.asarray(want[k]).dtype == np.float64 else want[k])
                 for k in ("count", "octets", "ubps_lo", "ubps_hi", "min", "max", "avg", "median",
                           "tallies"))
        q.put(ok and np.array_equal(got["hist"], want["hist"]))
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
