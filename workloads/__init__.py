"""Synthetic workloads of SURVEY.md §8(d) (D1-D5 shapes), via libgnm_synth.so.

Bench/test input only. Counter-based, so ``index_offset`` yields any index
shard of a workload bit-identically (multi-GPU sharding, chunked oracles).
Standalone: importing it loads only workloads/lib/libgnm_synth.so, never the
product library, so bench.py's reference arm can generate the same records
without mapping libgnetmon.so.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

SYNTH_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libgnm_synth.so")


class _Spec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n", C.c_uint64), ("index_offset", C.c_uint64),
                ("n_sites", C.c_uint32), ("site_base", C.c_void_p), ("site_size", C.c_void_p),
                ("zipf_s", C.c_double), ("hosts_per_site", C.c_uint32),
                ("frac_ack", C.c_double), ("frac_admin", C.c_double), ("frac_fwd", C.c_double),
                ("mu", C.c_double), ("sigma", C.c_double),
                ("window_start_ms", C.c_uint64), ("window_ms", C.c_uint64)]


_synth = None


def _lib():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} missing: run make / __graft_entry__.build()")
        _synth = C.CDLL(SYNTH_PATH)
        _synth.gnm_synth_generate.restype = C.c_int
        _synth.gnm_synth_generate.argtypes = [C.POINTER(_Spec)] + [C.c_void_p] * 6
        _synth.gnm_synth_to_aos.restype = None
        _synth.gnm_synth_to_aos.argtypes = [C.c_uint64] + [C.c_void_p] * 7
    return _synth


@dataclass
class SiteLayout:
    """Sites as (CIDR text, first address, address count), registration order."""
    cidrs: list
    base: np.ndarray
    size: np.ndarray

    def register(self, catalog, prefix: str = "site") -> None:
        for i, c in enumerate(self.cidrs):
            catalog.register_site(f"{prefix}{i}", [c])


def sites_slash24(n: int) -> SiteLayout:
    """n /24 sites packed from 10.0.0.0: 10.{i/256}.{i%256}.0/24 (D1, D3)."""
    cidrs, base = [], []
    for i in range(n):
        b = (10 << 24) + (i << 8)
        base.append(b)
        cidrs.append(f"{b >> 24}.{b >> 16 & 255}.{b >> 8 & 255}.0/24")
    return SiteLayout(cidrs, np.array(base, np.uint32), np.full(n, 256, np.uint32))


def sites_mixed(n: int, seed: int = 2) -> SiteLayout:
    """D2: prefix lengths {24,23,22,20,16} with p={.60,.15,.15,.07,.03},
    packed disjointly (aligned) upward from 10.0.0.0."""
    rng = np.random.default_rng(seed)
    lens = rng.choice([24, 23, 22, 20, 16], size=n, p=[0.60, 0.15, 0.15, 0.07, 0.03])
    cidrs, base, size = [], [], []
    cur = 10 << 24
    for L in lens.tolist():
        span = 1 << (32 - L)
        cur = (cur + span - 1) // span * span
        cidrs.append(f"{cur >> 24}.{cur >> 16 & 255}.{cur >> 8 & 255}.{cur & 255}/{L}")
        base.append(cur)
        size.append(span)
        cur += span
    return SiteLayout(cidrs, np.array(base, np.uint32), np.array(size, np.uint32))


@dataclass
class Workload:
    name: str
    n: int
    sites: SiteLayout
    seed: int
    zipf_s: float = 0.0
    hosts_per_site: int = 8
    frac_ack: float = 0.30
    frac_admin: float = 0.20
    frac_fwd: float = 0.40
    mu: float = 14.5
    sigma: float = 1.5
    window_start_ms: int = 1_600_000_000_000
    window_ms: int = 60_000


def workload(name: str, n: int | None = None) -> Workload:
    """D1 100k/256 sites; D2 1M/1k mixed prefixes; D3 100M/10k Zipf(1);
    D4 1B with D3's distribution (sharded by index); D5 streaming batches."""
    if name == "D1":
        return Workload("D1", n or 100_000, sites_slash24(256), seed=1)
    if name == "D2":
        return Workload("D2", n or 1_000_000, sites_mixed(1000), seed=2, window_ms=3_600_000)
    if name == "D3":
        return Workload("D3", n or 100_000_000, sites_slash24(10_000), seed=3, zipf_s=1.0,
                        window_ms=3_600_000)
    if name == "D4":
        return Workload("D4", n or 1_000_000_000, sites_slash24(10_000), seed=4, zipf_s=1.0,
                        window_ms=3_600_000)
    if name == "D5":
        return Workload("D5", n or 833_000, sites_slash24(256), seed=5)
    raise ValueError(name)


def generate(w: Workload, n: int | None = None, index_offset: int = 0, out=None):
    """Columns (src, dst, pkts, octets, start, end) as numpy arrays (or into
    ``out``: six writable host arrays, e.g. pinned torch tensors' numpy views)."""
    n = w.n if n is None else n
    if out is None:
        out = (np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint32),
               np.empty(n, np.uint32), np.empty(n, np.uint64), np.empty(n, np.uint64))
    spec = _Spec(w.seed, n, index_offset, len(w.sites.base), w.sites.base.ctypes.data,
                 w.sites.size.ctypes.data, w.zipf_s, w.hosts_per_site, w.frac_ack, w.frac_admin,
                 w.frac_fwd, w.mu, w.sigma, w.window_start_ms, w.window_ms)
    rc = _lib().gnm_synth_generate(C.byref(spec), *[a.ctypes.data for a in out])
    if rc:
        raise RuntimeError(f"gnm_synth_generate failed ({rc})")
    return out


def to_aos(cols) -> np.ndarray:
    """SoA columns -> 64-byte FlowRecord AoS bytes (uint8 array, n*64)."""
    n = len(cols[0])
    out = np.empty(n * 64, np.uint8)
    _lib().gnm_synth_to_aos(n, *[np.ascontiguousarray(c).ctypes.data for c in cols], out.ctypes.data)
    return out
