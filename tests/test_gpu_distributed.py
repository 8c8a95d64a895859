"""The N>1 path on a real device: two ranks (gloo, both on cuda:0 -- gpurun
gives one GPU; NCCL refuses two ranks on one device) each accumulate their
index shard into their own engine's device partials (K2), run the exact
two-round combine bench.py runs over NCCL (paper_1108_1785_b200.distributed
.combine on the zero-copy partial views: all-reduce of sums / min / max /
coarse, K3a + K2b on the rank's own log, all-reduce of fine), and finalize.
Every rank's site table must equal the single-engine result bit-exactly."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, outdir, n, workload, backend="gloo"):
    import torch
    import torch.distributed as dist
    from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
    from paper_1108_1785_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    w = synth.workload(workload)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    a, b = D.shard_range(n, rank, world)
    eng = Engine(0)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
    for _ in range(2):  # twice: the partials and the log must reset between steps
        eng.accumulate(FlowBatch(*[c[a:b] for c in cols]).to_device(), cat)
        torch.cuda.synchronize()
        D.combine(eng, cat, stream=stream)
        res = eng.finalize(cat)
    np.save(os.path.join(outdir, f"table{rank}.npy"), res.table)
    np.save(os.path.join(outdir, f"tallies{rank}.npy"),
            np.array([res.tallies.forward, res.tallies.pure_ack, res.tallies.administrative,
                      res.tallies.unmatched], np.uint64))
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("workload,n", [("D2", 600_001), ("D3", 2_000_003)])
def test_two_rank_combine_on_device_matches_single(engine, workload, n):
    import torch.multiprocessing as mp
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth

    w = synth.workload(workload)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    want = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(2, _free_port(), d, n, workload), nprocs=2, join=True)
        for r in range(2):
            got = np.load(os.path.join(d, f"table{r}.npy"))
            np.testing.assert_array_equal(got, want.table, err_msg=f"rank {r}")
            t = np.load(os.path.join(d, f"tallies{r}.npy"))
            np.testing.assert_array_equal(t, np.array([want.tallies.forward, want.tallies.pure_ack,
                                                       want.tallies.administrative, want.tallies.unmatched],
                                                      np.uint64))


@pytest.mark.parametrize("extra", [[], ["--hosts"]])
def test_bench_multi_rank_line(extra):
    """bench.py's N>1 path (index shards, the combine every step, barrier +
    max-over-ranks timing) under torchrun with two ranks; gloo and one
    device here (test hooks), NCCL on a multi-GPU box."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GNM_BENCH_BACKEND="gloo", GNM_BENCH_ONE_DEVICE="1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
         "--records", "3000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"] + extra,
        cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "index shards x2"


@pytest.mark.parametrize("extra", [[], ["--hosts"]])
def test_bench_nccl_path_single_rank(extra):
    """bench.py's N>1 code path over NCCL (the backend the 8-GPU run uses),
    forced at world size 1 by the GNM_BENCH_FORCE_DIST test hook."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GNM_BENCH_FORCE_DIST="1")
    env.pop("GNM_BENCH_BACKEND", None)
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1",
         "--records", "3000000", "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"] + extra,
        cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["value"] > 0 and lines[0]["e2e"]["value"] > 0


def _rank_hosts(rank, world, port, outdir, n, workload):
    import torch
    import torch.distributed as dist
    from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
    from paper_1108_1785_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = synth.workload(workload)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    a, b = D.shard_range(n, rank, world)
    eng = Engine(0)
    eng.set_hosts(True)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
    for _ in range(2):
        eng.accumulate(FlowBatch(*[c[a:b] for c in cols]).to_device(), cat)
        torch.cuda.synchronize()
        D.combine(eng, cat, stream=stream)  # site rows and, in per-host mode, host rows
        res = eng.finalize(cat)
    np.save(os.path.join(outdir, f"table{rank}.npy"), res.table)
    np.save(os.path.join(outdir, f"hosts{rank}.npy"), res.host_table)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_combine_single_rank(engine):
    """The combine over NCCL itself (the backend bench.py uses at N>1): one
    rank, so the all-reduces are identities, but every collective runs on
    the engine's stream with the partials' real dtypes (int64 SUM, f64
    MIN/MAX, int32 SUM) and the table must equal the plain call's."""
    import torch.multiprocessing as mp
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth

    n, workload = 1_000_003, "D3"
    w = synth.workload(workload)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    want = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(1, _free_port(), d, n, workload, "nccl"), nprocs=1, join=True)
        np.testing.assert_array_equal(np.load(os.path.join(d, "table0.npy")), want.table)


@pytest.mark.parametrize("workload,n", [("D1", 300_001), ("D3", 1_500_007)])
def test_two_rank_host_rows_match_single(engine, workload, n):
    """Per-host rows across ranks (gnm_hosts_*): the union of the ranks'
    (site, host) keys and the two-round median on it give every rank the
    single engine's rows bit-exactly."""
    import torch.multiprocessing as mp
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth

    w = synth.workload(workload)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    engine.set_hosts(True)
    try:
        want = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    finally:
        engine.set_hosts(False)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_hosts, args=(2, _free_port(), d, n, workload), nprocs=2, join=True)
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"table{r}.npy")), want.table)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"hosts{r}.npy")), want.host_table,
                                          err_msg=f"rank {r}")
