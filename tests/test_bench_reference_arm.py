"""bench.py --impl reference (the unmodified reference's aggregate timed on
the host cores) under torchrun with two ranks: rank 0 alone prints the line,
with the contract's keys; the other rank exits 0 without work."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_reference_arm_under_torchrun(ref):
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
         "--gpus", "2", "--steps", "2", "--warmup", "1", "--cpu-sample", "100000"],
        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    for k in ("metric", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"


def test_bench_self_launches_gpus_n(ref):
    """`python bench.py --gpus 2` without torchrun relaunches itself as two
    ranks (the driver's plain BENCH form must not silently measure one)."""
    out = subprocess.run(
        [sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
         "--records", "200000", "--cpu-sample", "100000"],
        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_reference_arm_maps_no_product_library(ref):
    """The reference arm generates its inputs with `workloads` and times
    oracle/_ref: libgnetmon.so is never mapped into that process, and its
    config is the GPU arm's config (the sample is stated in cpu_baseline)."""
    prog = (
        "import os, sys, runpy, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0',\n"
        "            '--records', '300000', '--cpu-sample', '100000']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = sorted({l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')})\n"
        "print('MAPS ' + json.dumps([m for m in maps if m.startswith(os.getcwd())]))\n")
    out = subprocess.run([sys.executable, "-c", prog], cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, GNM_REF_BUDGET_S="2"))
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(next(x for x in out.stdout.splitlines() if x.startswith("{")))
    maps = json.loads(next(x for x in out.stdout.splitlines() if x.startswith("MAPS "))[5:])
    assert not any("libgnetmon" in m for m in maps), maps
    assert any(m.endswith("oracle/_ref/libflowmon_ref.so") for m in maps), maps
    assert line["config"]["records_per_gpu"] == 300000
    assert "each step" in line["cpu_baseline"]["sample"]
