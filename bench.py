#!/usr/bin/env python3
"""Benchmark of the flow-analysis hot path (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gnetmon|reference]

A step = one full pass of the hot path over one batch: classify -> attribute
-> rate -> per-site aggregate (K2) -> [NCCL all-reduce of per-site partials
when N > 1] -> per-site median/avg/flag (K3) -> site table to the host.

Workload (BASELINE.json configs[2], the config the north-star roofline target
is quoted on): D3 = 100M synthetic NetFlow records per GPU, 10k /24 sites,
Zipf(s=1) site popularity, generated once per rank by the counter-based
generator (rank r takes global indices [r*n, (r+1)*n), so N GPUs process
N*100M records of the D4 shape: weak scaling). 3.2 GB of SoA input per GPU
is > 25x the 126 MB L2, so no L2 flush is needed between steps.

`value`  : records/s, inputs resident in HBM, device-timed (CUDA events on the
           engine stream, max over ranks).
`e2e`    : records/s through the same public call with the batch in PINNED
           HOST memory: the double-buffered H2D loader runs inside every step.
`roofline`: K2's algorithmic 32 B/record over its CUDA-event time vs the
           measured HBM copy bandwidth (MEASURED_PEAKS.json).
`cpu_baseline`: the unmodified reference (oracle/_ref) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALG_BYTES_PER_RECORD = 32  # src, dst, d_pkts, d_octets (u32) + start_ms, end_ms (u64)
NOMINAL_HBM_GBS = 8000.0   # the north star's "~8 TB/s" (SURVEY.md §8d asks for both fractions)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
METRIC = "flow records/sec analysed"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 100; D5: 600 batches; reference arm: 20 samples)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="gnetmon", choices=["gnetmon", "reference"])
    ap.add_argument("--workload", default="D3")
    ap.add_argument("--records", type=int, default=None, help="records per GPU (default: workload)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-sample", type=int, default=2_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hot-mode", default="auto", choices=["auto", "off", "force"])
    ap.add_argument("--input", default="soa", choices=["soa", "aos"],
                    help="record layout handed to the API: SoA columns (default, the north star's "
                         "loader layout) or the reference's 64-byte FlowRecord rows (gnm_analyze_aos)")
    ap.add_argument("--no-pageable", action="store_true", help="skip the pageable-host e2e leg")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary AoS / per-host device legs")
    ap.add_argument("--no-adapter", action="store_true",
                    help="skip the C++ drop-in leg (integration/_build/adapter_bench)")
    ap.add_argument("--hosts", action="store_true",
                    help="per-host mode: every step also builds SiteResult::hosts")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("GNM_BENCH_ONE_DEVICE"):  # test hook: every rank on cuda:0 (gloo; see tests)
        local = 0
    return world, rank, local


# ---- clocks --------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- helpers --------------------------------------------------------------------

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"  # B200_PROFILING.md fallback


def load_traffic(workload: str):
    p = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload)
        if e:
            return e
    return None


def pinned_columns(n: int):
    """Six pinned host columns (torch pinned buffers) + numpy views."""
    import torch
    ts = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(4)]
    ts += [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(2)]
    views = [t.numpy().view(np.uint32) for t in ts[:4]] + [t.numpy().view(np.uint64) for t in ts[4:]]
    return ts, views


def reference_sample(w, n_sample: int):
    # `workloads` and `oracle` only: the reference arm never maps libgnetmon.so
    import workloads
    from oracle import Reference
    R = Reference()
    cols = workloads.generate(w, n_sample)
    cat = R.catalog([[c] for c in w.sites.cidrs])
    rec = R.records(cols)
    return R, cat, rec


def reference_workers(n_sample: int, nproc: int) -> list[int]:
    """Worker counts whose per-(site, host) 40 KB histograms fit in half of
    the available RAM (the reference allocates one per host per worker)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    out = []
    for w in [1, 2, 4, 8, 16, 32, 64, nproc]:
        if w > nproc or w in out:
            continue
        hosts_per_worker = min(80_000, n_sample // w)
        if w * hosts_per_worker * 40_004 * 1.3 < 0.5 * avail:
            out.append(w)
    return out or [1]


def reference_plan(w, n: int, runs: int, budget_s: float, probe_records: int = 10_000_000):
    """The reference's CPU timing setup on this box: the workload's first
    records (up to all n), the fastest worker count probed at a
    representative size (its per-call histogram allocation -- 40 KB per
    (site, host) per worker -- dominates small samples, so the probe must not
    be tiny), and the largest sample whose `runs` timed calls fit
    `budget_s`. Returns (R, cat, rec, m, best_workers, probe_ms_by_workers)."""
    nproc = os.cpu_count() or 1
    m_probe = min(n, probe_records)
    R, cat, rec = reference_sample(w, m_probe)
    workers = reference_workers(m_probe, nproc)
    R.time_range(rec, cat, 0, m_probe, 1)  # warm-up: page faults, allocator
    probe = {wk: R.time_range(rec, cat, 0, m_probe, wk) for wk in workers}
    best = min(probe, key=probe.get)
    per_record_ms = probe[best] / m_probe
    m = int(budget_s * 1e3 / max(1, runs) / per_record_ms)
    m = max(m_probe, min(n, m))
    if m != m_probe:
        del rec
        R, cat, rec = reference_sample(w, m)
        if best not in reference_workers(m, nproc):
            best = max(reference_workers(m, nproc))
    return R, cat, rec, m, best, probe


def workload_config(w, n: int, n_sites: int, world: int, args) -> dict:
    """The `config` object both arms print (the GPU arm's workload; the
    reference arm times bounded samples of it, stated in cpu_baseline)."""
    return {"workload": f"{w.name}: {n} records/GPU, {n_sites} /24 sites, Zipf s={w.zipf_s}, "
                        f"8 hosts/site, 40% forward",
            "records_per_gpu": n, "sites": n_sites, "input": args.input,
            "hosts": ("per-host rows built every step" if args.hosts
                      else "site level only (gnm_ctx_set_hosts off)"),
            "parallelism": f"index shards x{world}",
            "l2": "inputs 3.2 GB/GPU > 126 MB L2; no flush needed" if n >= 10_000_000
                  else "inputs may fit L2"}


def self_launch(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: relaunch this script as N
    ranks on this node (one per GPU, rendezvous on 127.0.0.1), exactly as the
    driver's torchrun form does; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ---- the reference arm -------------------------------------------------------

def run_reference_arm(args):
    """The reference's own CPU path (unmodified flowmon::aggregate from
    oracle/_ref) on this box's host cores, on the GPU arm's workload, metric
    and config: every step is a bounded sample (the workload's first M
    records, M sized from a warmed probe so the whole run stays within a few
    minutes), at the fastest worker count. Rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import workloads
    w = workloads.workload(args.workload)
    n = args.records or w.n
    nproc = os.cpu_count() or 1
    steps = args.steps if args.steps is not None else 10
    # Each step is the workload's first m records (all n when ~300 s of CPU
    # time allows), at the fastest worker count probed on 10M records.
    budget_s = float(os.environ.get("GNM_REF_BUDGET_S", "300"))
    R, cat, rec, m, best, probe = reference_plan(w, n, steps + args.warmup, budget_s,
                                                 probe_records=min(args.cpu_sample * 5, n))
    for _ in range(args.warmup):
        R.time_range(rec, cat, 0, m, best)
    ts = [R.time_range(rec, cat, 0, m, best) for _ in range(steps)]
    total_ms = sum(ts)
    value = m * len(ts) / (total_ms / 1e3)
    n_probe = min(args.cpu_sample * 5, n)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "records/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": total_ms / len(ts), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/u64 int + f64", "data": "synthetic",
        "config": workload_config(w, n, len(w.sites.base), world, args),
        "cpu_baseline": {"value": value, "unit": "records/s", "cores": best, "kind": "reference",
                         "sample": (f"each step: all {n} records of the workload" if m == n else
                                    f"each step: the first {m} of the workload's {n} records per GPU")
                                   + f" (hosts computed, as the reference always does); unmodified "
                                   f"flowmon::aggregate(FilterParams{{}}, workers={best}, Hash) from "
                                   f"oracle/_ref (-O3 -DNDEBUG); worker probe on {n_probe} records, ms by "
                                   f"workers {json.dumps({str(k): round(v, 1) for k, v in probe.items()})}; "
                                   f"nproc={nproc}, cpu={cpu_model()}"},
        "e2e": {"value": value, "unit": "records/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parallelism_note": f"cpu threads={best}",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- the GPU arm ----------------------------------------------------------------

# ---- D5: streaming 1-minute batches ---------------------------------------------

def stream_line(args, m=None, steps=None):
    """BASELINE.json configs[4]: continuous 1-minute batches through the
    window-fused public call (snapshot + aggregate, monitor.cpp:109-120),
    each from pinned host memory (chunked double-buffered H2D inside the
    call), result table back to the host. Reports records/s and the
    per-batch end-to-end latency distribution over --steps batches (default
    600). Batch j's records end inside its minute except ~5% late arrivals
    from the previous one, which the window drops. A ring of 16 distinct
    minutes is pre-generated and replayed."""
    import dataclasses
    import torch
    from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    base = synth.workload("D5")
    m = m or args.records or base.n
    cat = SiteCatalog()
    base.sites.register(cat)
    ring = []
    t0 = base.window_start_ms
    for j in range(16):
        w = dataclasses.replace(base, window_start_ms=t0 + j * 60_000 - 3_000, window_ms=63_000)
        ts, views = pinned_columns(m)
        synth.generate(w, m, index_offset=j * m, out=views)
        ring.append((FlowBatch(*views), t0 + j * 60_000, [t.to(f"cuda:{local}") for t in ts]))
    torch.cuda.synchronize()
    eng = Engine(local)
    steps = steps or args.steps or 600
    for j in range(max(args.warmup, 3)):
        b, lo, _ = ring[j % 16]
        eng.aggregate_window(b, cat, lo, lo + 60_000)
    lat = []
    analysed = 0
    clocks = ClockSampler(local)
    if not os.environ.get("GNM_BENCH_NO_CLOCKS"):  # diagnosis only: the line then has no clocks
        clocks.start()
    t_all = time.perf_counter()
    for i in range(steps):
        b, lo, _ = ring[i % 16]
        t = time.perf_counter()
        r = eng.aggregate_window(b, cat, lo, lo + 60_000)
        lat.append((time.perf_counter() - t) * 1e3)
        analysed += r.tallies.total()
    wall = time.perf_counter() - t_all
    clk = clocks.stop()
    # The same batches already resident in HBM (no H2D), device-timed.
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local}")
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for i in range(steps):
        _, lo, dev = ring[i % 16]
        eng.aggregate_window(FlowBatch(*dev), cat, lo, lo + 60_000)
    ev1.record(stream)
    torch.cuda.synchronize()
    dev_ms = ev0.elapsed_time(ev1)
    eng.close()
    q = np.percentile(np.array(lat), [50, 99])
    line = {
        "metric": METRIC, "value": m * steps / (dev_ms / 1e3), "unit": "records/s", "n_gpus": 1,
        "steps": steps, "warmup": args.warmup, "ms_per_step": dev_ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64 int + f64", "data": "synthetic",
        "config": {"workload": f"D5: {steps} one-minute batches of {m} records ({len(base.sites.base)} "
                               f"sites, ~5% late arrivals dropped by the window), snapshot+aggregate fused",
                   "records_per_batch": m, "parallelism": "1 GPU, batches back to back"},
        "e2e": {"value": m * steps / wall, "unit": "records/s", "h2d_bytes_per_step": m * ALG_BYTES_PER_RECORD,
                "d2h_bytes_per_step": (cat.site_count() + 1) * 72,
                "latency_ms": {"p50": float(q[0]), "p99": float(q[1]), "max": float(max(lat))},
                "records_in_window_per_batch": analysed / steps},
        "clocks": clk,
    }
    return line


def run_stream(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    print(json.dumps(stream_line(args)), flush=True)
    return 0


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.steps is None and args.impl != "reference" and args.workload != "D5":
        args.steps = 100
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "D5":
        return run_stream(args)

    import torch
    import torch.distributed as dist
    from paper_1108_1785_b200 import Engine, FlowBatch, FlowRecords, SiteCatalog, synth
    from paper_1108_1785_b200 import distributed as D

    world, rank, local = dist_env()
    # GNM_BENCH_FORCE_DIST: test hook, the N>1 code path (process group, the
    # combine every step, max over ranks) at world size 1 -- NCCL on the one
    # GPU a test box has.
    distributed = world > 1 or bool(os.environ.get("GNM_BENCH_FORCE_DIST"))
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} device(s) visible")
    if distributed:
        # NCCL over NVLink; GNM_BENCH_BACKEND=gloo is a test hook for several
        # ranks on the one GPU a test box has (NCCL refuses shared devices).
        backend = os.environ.get("GNM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    w = synth.workload(args.workload)
    n = args.records or w.n
    cat = SiteCatalog()
    w.sites.register(cat)

    # Inputs: this rank's index shard, in pinned host memory (the e2e arm's
    # source) and resident in HBM (the `value` arm's source).
    host_t, host = pinned_columns(n)
    synth.generate(w, n, index_offset=rank * n, out=host)
    dev_t = [t.to(f"cuda:{local}", non_blocking=False) for t in host_t]
    torch.cuda.synchronize()
    dev_batch = FlowBatch(*dev_t)
    host_batch = FlowBatch(*host)
    if args.input == "aos":
        # The reference's own span<const FlowRecord> layout: 64 B rows, pinned.
        rows_t = torch.empty(n * 64, dtype=torch.uint8).pin_memory()
        rows = rows_t.numpy()
        synth._lib().gnm_synth_to_aos(n, *[c.ctypes.data for c in host], rows.ctypes.data)
        del dev_t, dev_batch
        dev_rows = rows_t.to(f"cuda:{local}")
        torch.cuda.synchronize()
        dev_batch = FlowRecords(dev_rows)
        host_batch = FlowRecords(rows)

    eng = Engine(local)
    eng.set_hot_mode(args.hot_mode)
    if os.environ.get("GNM_BENCH_NO_GRAPHS"):  # diagnosis: launch kernel by kernel
        eng.set_graphs(False)
    if args.hosts:
        eng.set_hosts(True)  # N > 1: distributed.combine also merges the host rows
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local}")
    # N > 1 over NCCL: the library's own communicator (gnm_ctx_comm_init; the
    # unique id travels over the torch process group), so every step is one
    # gnm_analyze call -- K2 on this rank's shard, round 1 (one grouped NCCL
    # call: sums / coarse SUM, min MIN, max MAX), K3a+K2b, round 2 (fine SUM),
    # K3b -- all on the engine stream and replayed as one CUDA graph. The
    # gloo test hook (several ranks on one GPU) combines through
    # torch.distributed instead (paper_1108_1785_b200.distributed).
    in_library = distributed and os.environ.get("GNM_BENCH_BACKEND", "nccl") == "nccl"
    if in_library:
        uid = [Engine.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.comm_init(world, rank, uid[0])

    def step(batch):
        if not distributed or in_library:
            return eng.aggregate(batch, cat)
        eng.accumulate(batch, cat)
        D.combine(eng, cat, stream=stream)
        return eng.finalize(cat)

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(batch, steps, breakdown=True):
        """`steps` back-to-back steps between two events on the engine
        stream (barrier + synchronize on both sides, max over ranks). The
        loop runs as a user's would (repeated device-batch calls replay the
        context's CUDA graph). The per-kernel breakdown comes from a
        separate, untimed pass with the context's own CUDA events around
        K1, K2 and the finalize kernels (events disable graph replay)."""
        for _ in range(args.warmup):
            step(batch)
        barrier()
        launches0 = eng.timing()["kernel_launches"]
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            res = step(batch)
        ev1.record(stream)
        barrier()
        launches = eng.timing()["kernel_launches"] - launches0
        ms = ev0.elapsed_time(ev1)
        if distributed:
            tt = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        per = {}
        if breakdown:
            nb = min(steps, 20)
            eng.enable_timing(True)
            for _ in range(nb):
                step(batch)
            barrier()
            t = eng.timing()
            eng.enable_timing(False)
            per = {"k1_plan": t["total_plan_ms"] / nb, "k2": t["total_accumulate_ms"] / nb,
                   "k3_finalize": t["total_finalize_ms"] / nb}
        return ms, launches, res, per

    clocks = ClockSampler(local)
    if not os.environ.get("GNM_BENCH_NO_CLOCKS"):  # diagnosis only: the line then has no clocks
        clocks.start()
    ms, launches, res, per = timed(dev_batch, args.steps)
    clk = clocks.stop()
    e2e_steps = args.e2e_steps or max(3, args.steps // 2)
    hb0 = eng.timing()["h2d_bytes"]
    e2e_ms, _, res_e2e, _ = timed(host_batch, e2e_steps, breakdown=False)
    # bytes the loader actually moved per step (non-windowed SoA: u32
    # durations in place of the two u64 timestamps)
    h2d_step = (eng.timing()["h2d_bytes"] - hb0) // (args.warmup + e2e_steps)
    # The same call from PAGEABLE host memory (a std::vector<FlowRecord> or a
    # plain numpy array, as the C++ adapter passes it): the loader stages
    # through pinned slots with multi-threaded copies.
    pg_ms = None
    if not args.no_pageable:
        if args.input == "aos":
            pg_batch = FlowRecords(np.array(rows, copy=True))
        else:
            pg_batch = FlowBatch(*[np.array(v, copy=True) for v in host])
        pg_steps = 3
        pg_ms, _, res_pg, _ = timed(pg_batch, pg_steps, breakdown=False)
        assert np.array_equal(res.table, res_pg.table), "device and pageable-host runs differ"
        del pg_batch

    total = n * world
    value = total * args.steps / (ms / 1e3)
    e2e_value = total * e2e_steps / (e2e_ms / 1e3)
    # The e2e roofline: this box's raw pinned host->device copy rate, the
    # same bytes the e2e step moves (one 128 MiB chunk at a time).
    h2d_bytes = h2d_step
    srcs = [host_t[i] for i in range(6)] if args.input == "soa" else [rows_t]
    scratch = torch.empty(128 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    flat = [t.view(torch.uint8) for t in srcs]
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    c0.record()
    for f in flat:
        for o in range(0, f.numel(), scratch.numel()):
            m = min(scratch.numel(), f.numel() - o)
            scratch[:m].copy_(f[o:o + m], non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_peak = sum(f.numel() for f in flat) / (c0.elapsed_time(c1) / 1e3) / 1e9
    del scratch
    k2_avg, plan_avg, k3_avg = per["k2"], per["k1_plan"], per["k3_finalize"]
    peak, peak_kind = load_peaks()
    achieved = n * ALG_BYTES_PER_RECORD / (k2_avg / 1e3) / 1e9
    traffic = load_traffic(args.workload) if args.input == "soa" else None
    n_sites = cat.site_count()
    d2h = (n_sites + 1) * 72
    if args.hosts:
        d2h += len(res.host_table) * 64
        assert np.array_equal(res.host_table, res_e2e.host_table), "device and host runs differ (hosts)"

    # Correctness guard on the measured runs: every record was classified.
    assert res.tallies.total() == total and res_e2e.tallies.total() == total, "tally mismatch"
    assert np.array_equal(res.table, res_e2e.table), "device and host runs differ"

    line = {
        "metric": METRIC, "value": value, "unit": "records/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32/u64 int + f64", "data": "synthetic",
        "config": workload_config(w, n, n_sites, world, args),
        "e2e": {"value": e2e_value, "unit": "records/s",
                "h2d_bytes_per_step": h2d_step,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps,
                "source": (f"pinned host {args.input.upper()}, chunked double-buffered H2D"
                           + ("; the loader sends u32 durations computed on host threads in place of "
                              "start/end (20 B/record)" if args.input == "soa" else "")),
                "h2d_gbs": h2d_bytes * e2e_steps / (e2e_ms / 1e3) / 1e9, "h2d_raw_copy_gbs": h2d_peak,
                "frac_of_raw_copy": (h2d_bytes * e2e_steps / (e2e_ms / 1e3) / 1e9) / h2d_peak,
                "pageable": None if pg_ms is None else {
                    "value": total * 3 / (pg_ms / 1e3), "unit": "records/s", "ms_per_step": pg_ms / 3,
                    "source": f"pageable host {args.input.upper()} (numpy, not pinned): multi-threaded "
                              f"staging copies into the loader's pinned slots"}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "kernel": "k2_soa (classify+attribute+rate+aggregate)",
                     "kernel_ms": k2_avg, "alg_bytes_per_record": ALG_BYTES_PER_RECORD,
                     "physical_bytes_per_record": ALG_BYTES_PER_RECORD if args.input == "soa" else 64,
                     "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS},
        "combine": (None if not distributed else
                    "in-library NCCL two-round combine (gnm_ctx_comm_init), in the CUDA graph" if in_library
                    else "torch.distributed (gloo test hook) two-round combine"),
        "gpu_launches": launches,
        "clocks": clk,
        "kernel_share": k2_avg / (ms / args.steps),
        "breakdown_ms": {"k1_plan": plan_avg, "k2": k2_avg, "k3_finalize": k3_avg,
                         "step": ms / args.steps, "source": "per-kernel CUDA events, separate untimed pass"},
    }
    if rank == 0 and world == 1 and not args.no_extras and args.input == "soa" and not args.hosts:
        # Secondary device-resident measurements of the same records, so the
        # driver's own line carries them: the reference's 64-byte FlowRecord
        # rows (k2_aos; roofline on their 64 B/record physical bytes) and
        # per-host mode (SiteResult::hosts every step). Same timing rules.
        sec = {}
        try:
            # per-host mode on its own context, as a user enabling it would run
            main_eng, main_stream = eng, stream
            eng = Engine(local)
            stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local}")
            try:
                eng.set_hosts(True)
                h_ms, _, h_res, h_per = timed(dev_batch, 30)
            finally:
                eng.close()
                eng, stream = main_eng, main_stream
            assert np.array_equal(h_res.table, res.table), "hosts-mode site rows differ"
            sec["hosts_device"] = {
                "value": total * 30 / (h_ms / 1e3), "unit": "records/s", "ms_per_step": h_ms / 30,
                "host_rows": len(h_res.host_table), "k2_ms": h_per["k2"],
                "source": "per-host rows (SiteResult::hosts) built every step, SoA in HBM, own context, 30 steps"}
            stage = np.empty(n * 64, np.uint8)  # pageable: no pinned memory left behind
            synth._lib().gnm_synth_to_aos(n, *[c.ctypes.data for c in host], stage.ctypes.data)
            rows_t = torch.from_numpy(stage).to(f"cuda:{local}")
            del stage
            torch.cuda.synchronize()
            a_ms, _, a_res, a_per = timed(FlowRecords(rows_t), 20)
            assert np.array_equal(a_res.table, res.table), "AoS and SoA results differ"
            sec["aos_device"] = {
                "value": total * 20 / (a_ms / 1e3), "unit": "records/s", "ms_per_step": a_ms / 20,
                "k2_ms": a_per["k2"], "k2_kernel": "k2_aos",
                "k2_frac_of_hbm_physical": n * 64 / (a_per["k2"] / 1e3) / 1e9 / peak,
                "source": "64-byte FlowRecord rows resident in HBM (gnm_analyze_aos), 20 steps"}
            del rows_t
            torch.cuda.empty_cache()
            # D5 (BASELINE configs[4]): 600 one-minute 833k-record batches,
            # snapshot window fused, from pinned host memory (own engine)
            d5 = stream_line(args, m=833_000, steps=600)
            sec["d5_streaming"] = {"value": d5["value"], "unit": "records/s",
                                   "ms_per_batch_device": d5["ms_per_step"], "e2e": d5["e2e"],
                                   "source": d5["config"]["workload"]}
        except Exception as e:  # a secondary leg never voids the headline
            sec["error"] = repr(e)[:300]
        line["secondary"] = sec
    if rank == 0 and world == 1 and not args.no_adapter and args.workload in ("D1", "D3"):
        # The reference's own call, flowmon::aggregate from a pageable
        # std::vector<FlowRecord>, served by the C++ adapter: the full
        # AnalysisResult (hosts and histograms included) end to end.
        exe = os.path.join(ROOT, "integration", "_build", "adapter_bench")
        if os.path.exists(exe):
            eng.close()
            host_t = host = host_batch = dev_batch = dev_t = srcs = flat = None  # noqa: F841 (release pinned inputs)
            import gc
            gc.collect()
            torch.cuda.empty_cache()
            if hasattr(torch._C, "_host_emptyCache"):  # give the pinned host cache back first
                torch._C._host_emptyCache()
            out = subprocess.run([exe, "--workload", args.workload, "--records", str(n), "--steps", "5",
                                  "--warmup", "2"], capture_output=True, text=True, timeout=900)
            lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if out.returncode == 0 and lines:
                a = json.loads(lines[-1])
                line["e2e"]["adapter"] = {"value": a["records_per_s"], "unit": "records/s",
                                          "ms_per_step": a["ms_per_step"], "source": a["source"],
                                          "host_rows": a["host_rows"]}
            else:
                line["e2e"]["adapter"] = {"value": None, "error": (out.stderr or out.stdout)[-300:]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            eng.close()
            R, cat_r, rec, m, best, probe = reference_plan(w, n, 3, 30.0, probe_records=min(args.cpu_sample * 5 // 2, n))
            ts = [R.time_range(rec, cat_r, 0, m, best) for _ in range(3)]
            line["cpu_baseline"] = {
                "value": m / (statistics.median(ts) / 1e3), "unit": "records/s", "cores": best,
                "kind": "reference",
                "sample": f"first {m} records of {w.name}, unmodified flowmon::aggregate (oracle/_ref, -O3), "
                          f"median of 3 at workers={best}; probe ms by workers on {min(args.cpu_sample * 5 // 2, n)} records "
                          f"{json.dumps({str(k): round(v, 1) for k, v in probe.items()})}; "
                          f"nproc={os.cpu_count()}, cpu={cpu_model()}; the --impl reference arm times larger samples"}
        except ImportError as e:
            line["cpu_baseline"] = {"value": None, "unit": "records/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
