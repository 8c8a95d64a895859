"""Python mirror of the reference's analytics API over the C-ABI.

Names, argument meaning and error behaviour follow flowmon's C++ interface
(paths relative to /root/reference/proj/core):

=============================  =============================================
this module                    reference
=============================  =============================================
``FilterParams``               rate_engine.hpp:22-29
``FlowClass``/``LookupMode``   rate_engine.hpp:31-33
``Cidr``/``parse_ipv4``        site_catalog.hpp:29-44
``SiteCatalog``                site_catalog.hpp:50-97 (CatalogError on
                               overlap / invalid CIDR, catalog unchanged)
``RateStats``/``SiteResult``   rate_engine.hpp:76-99
``ClassTallies``               rate_engine.hpp:101-110
``AnalysisResult``             rate_engine.hpp:112-119 (site level)
``aggregate``                  rate_engine.hpp:143-146 -> K2 + K3 on the GPU
``aggregate_partitioned``      rate_engine.hpp:149-154
``WarningState``/``evaluate_warnings``  monitor.hpp:20-52
=============================  =============================================

The records are a ``FlowBatch`` of SoA columns (the hot fields of
``FlowRecord``, netflow.hpp:59-67) in host (numpy / CPU torch) or device
(CUDA torch) memory, or ``FlowRecords`` holding the reference's 64-byte AoS
layout. Every analysis runs on the GPU through libgnetmon.so; there is no
CPU fallback (a missing device raises ``GnmError``).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (BUCKET_COUNT, FLOW_RECORD_DTYPE, SITE_STATS_DTYPE, gnm_batch_aos,
                   gnm_batch_soa, gnm_cidr, gnm_filter_params, gnm_partials, gnm_result,
                   gnm_netflow_stats, gnm_timing, gnm_warning, lib)

kBucketCount = BUCKET_COUNT
kBucketWidthBps = 10_000.0
kRateCapBps = 100_000_000.0
kDefaultWarnThresholdBps = 1_000_000.0

SiteId = int


class GnmError(RuntimeError):
    """A failing C-ABI call (status code + thread-local message)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"gnetmon status {status}: {message}")
        self.status = status


class CatalogError(ValueError):
    """site_catalog.hpp:16-27; ``kind`` is "Overlap" or "InvalidCidr"."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


class ArchiveError(RuntimeError):
    """flow_store.hpp:22-33; ``kind`` is "BadMagic", "BadVersion" or
    "TruncatedArchive" (IoFailure has no in-memory counterpart)."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


class RateError(ArithmeticError):
    """rate_engine.hpp:35-45; ``kind`` is "ZeroDuration" or "EmptyHistogram"."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


def _check(status: int) -> None:
    if status == _lib.OK:
        return
    msg = _lib.last_error()
    if status == _lib.ERR_OVERLAP:
        raise CatalogError("Overlap", msg)
    if status == _lib.ERR_INVALID_CIDR:
        raise CatalogError("InvalidCidr", msg)
    if status in (_lib.ERR_BAD_MAGIC, _lib.ERR_BAD_VERSION, _lib.ERR_TRUNCATED):
        raise ArchiveError({_lib.ERR_BAD_MAGIC: "BadMagic", _lib.ERR_BAD_VERSION: "BadVersion",
                            _lib.ERR_TRUNCATED: "TruncatedArchive"}[status], msg)
    raise GnmError(status, msg)


class FlowClass(enum.IntEnum):
    Forward = 0
    PureAck = 1
    Administrative = 2
    Unmatched = 3


class LookupMode(enum.IntEnum):
    Hash = 0
    Sequential = 1


@dataclass
class FilterParams:
    ack_avg_size_max: int = 96
    min_packets: int = 20
    min_duration_ms: int = 100
    workers: int = 1

    def _c(self) -> gnm_filter_params:
        return gnm_filter_params(self.ack_avg_size_max, self.min_packets, self.min_duration_ms,
                                 self.workers)


# ---- CIDRs and the registry ---------------------------------------------------

def parse_ipv4(text: str) -> int:
    out = C.c_uint32()
    _check(lib.gnm_ipv4_parse(text.encode(), C.byref(out)))
    return out.value


def format_ipv4(ip: int) -> str:
    return f"{ip >> 24}.{ip >> 16 & 255}.{ip >> 8 & 255}.{ip & 255}"


@dataclass(frozen=True)
class Cidr:
    addr: int = 0
    prefix_len: int = 0

    @staticmethod
    def parse(text: str) -> "Cidr":
        out = gnm_cidr()
        _check(lib.gnm_cidr_parse(text.encode(), C.byref(out)))
        return Cidr(out.addr, out.prefix_len)

    def network(self) -> int:
        mask = 0 if self.prefix_len == 0 else (0xFFFFFFFF << (32 - self.prefix_len)) & 0xFFFFFFFF
        return self.addr & mask

    def first_prefix24(self) -> int:
        return self.network() & 0xFFFFFF00

    def last_prefix24(self) -> int:
        if self.prefix_len >= 24:
            return self.first_prefix24()
        return self.first_prefix24() + ((1 << (24 - self.prefix_len)) - 1) * 256

    def to_string(self) -> str:
        return f"{format_ipv4(self.network())}/{self.prefix_len}"


class SiteCatalog:
    """Registry of named sites (site_catalog.hpp:50-97), backed by the C-ABI."""

    def __init__(self):
        h = C.c_void_p()
        _check(lib.gnm_registry_create(C.byref(h)))
        self._h = h
        self._cidrs: list[list[Cidr]] = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.gnm_registry_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def register_site(self, name: str, cidrs: Iterable) -> SiteId:
        parsed = [c if isinstance(c, Cidr) else
                  (Cidr.parse(c) if isinstance(c, str) else Cidr(int(c[0]), int(c[1])))
                  for c in cidrs]
        arr = (gnm_cidr * max(len(parsed), 1))(*[gnm_cidr(c.addr, c.prefix_len) for c in parsed])
        out = C.c_uint32()
        _check(lib.gnm_registry_register_site(self._h, name.encode(), arr, len(parsed),
                                              C.byref(out)))
        self._cidrs.append(parsed)
        return out.value

    def lookup(self, ip: int) -> Optional[SiteId]:
        s = lib.gnm_registry_lookup(self._h, ip & 0xFFFFFFFF)
        return None if s == _lib.NO_SITE else s

    def sequential_lookup(self, ip: int) -> Optional[SiteId]:
        s = lib.gnm_registry_sequential_lookup(self._h, ip & 0xFFFFFFFF)
        return None if s == _lib.NO_SITE else s

    def site(self, site_id: SiteId) -> str:
        name = lib.gnm_registry_site_name(self._h, site_id)
        if name is None:
            raise IndexError(f"no site {site_id}")
        return name.decode()

    def site_cidrs(self, site_id: SiteId) -> list[Cidr]:
        return list(self._cidrs[site_id])

    def site_count(self) -> int:
        return lib.gnm_registry_site_count(self._h)

    def entry_count(self) -> int:
        return lib.gnm_registry_entry_count(self._h)

    def empty(self) -> bool:
        return self.entry_count() == 0

    def entries_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        n = self.entry_count()
        p = np.zeros(n, np.uint32)
        s = np.zeros(n, np.uint32)
        lib.gnm_registry_entries(self._h, p.ctypes.data, s.ctypes.data, n)
        return p, s

    def entries(self) -> list[tuple[int, int]]:
        p, s = self.entries_arrays()
        return list(zip(p.tolist(), s.tolist()))

    def version(self) -> int:
        return lib.gnm_registry_version(self._h)

    # SiteCatalog::load / save text format (site_catalog.cpp:150-203).
    @staticmethod
    def load(text: str) -> "SiteCatalog":
        cat = SiteCatalog()
        for line in text.splitlines():
            line = line.split("#", 1)[0]
            fields = line.split()
            if len(fields) < 2:
                continue
            cat.register_site(fields[0], [c for c in fields[1].split(",") if c])
        return cat

    def save(self) -> str:
        return "".join(f"{self.site(i)} {','.join(c.to_string() for c in self._cidrs[i])}\n"
                       for i in range(self.site_count()))


# ---- record batches ------------------------------------------------------------

def _pinned_rows(n: int) -> np.ndarray:
    """n HOST_STATS_DTYPE rows in page-locked memory from torch's caching
    host allocator (reused once an earlier result is dropped): the D2H of the
    per-host rows then runs at the pinned rate instead of ~22 GB/s pageable
    (80k rows: ~0.1 ms instead of ~0.23). Plain numpy when torch is absent."""
    nbytes = n * _lib.HOST_STATS_DTYPE.itemsize
    try:
        import torch
        if nbytes >= (1 << 20) and torch.cuda.is_available():
            buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            return buf.numpy().view(_lib.HOST_STATS_DTYPE)  # the array keeps `buf` alive
    except ImportError:
        pass
    return np.empty(n, _lib.HOST_STATS_DTYPE)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _col_ptr(x, itemsize: int, name: str):
    """(pointer, length, on_device) of one column; numpy or torch."""
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError(f"column {name} must be contiguous")
        if x.element_size() != itemsize:
            raise ValueError(f"column {name} must have {itemsize}-byte elements")
        return x.data_ptr(), x.numel(), bool(x.is_cuda)
    a = np.asarray(x)
    want = np.uint32 if itemsize == 4 else np.uint64
    if a.dtype != want or not a.flags.c_contiguous:
        raise ValueError(f"column {name} must be a C-contiguous {np.dtype(want).name} array")
    return a.ctypes.data, a.size, False


class FlowBatch:
    """SoA columns of flow records: u32 src/dst/pkts/octets, u64 start/end ms."""

    COLUMNS = ("src_addr", "dst_addr", "d_pkts", "d_octets", "start_ms", "end_ms")
    WIDTHS = (4, 4, 4, 4, 8, 8)

    def __init__(self, src_addr, dst_addr, d_pkts, d_octets, start_ms, end_ms):
        self.cols = [src_addr, dst_addr, d_pkts, d_octets, start_ms, end_ms]
        ptrs, lens, dev = [], [], []
        for c, name, w in zip(self.cols, self.COLUMNS, self.WIDTHS):
            p, n, d = _col_ptr(c, w, name)
            ptrs.append(p)
            lens.append(n)
            dev.append(d)
        if len(set(lens)) != 1:
            raise ValueError("columns differ in length")
        if len(set(dev)) != 1:
            raise ValueError("columns must all be on the host or all on the device")
        self.n = lens[0]
        self.on_device = dev[0]
        self._ptrs = ptrs

    def __len__(self) -> int:
        return self.n

    def __getattr__(self, name):
        if name in FlowBatch.COLUMNS:
            return self.cols[FlowBatch.COLUMNS.index(name)]
        raise AttributeError(name)

    def _c(self) -> gnm_batch_soa:
        return gnm_batch_soa(*self._ptrs, self.n, _lib.MEM_DEVICE if self.on_device else _lib.MEM_HOST)

    def slice(self, begin: int, end: int) -> "FlowBatch":
        return FlowBatch(*[c[begin:end] for c in self.cols])

    @staticmethod
    def from_records(records: np.ndarray) -> "FlowBatch":
        r = np.asarray(records)
        return FlowBatch(*[np.ascontiguousarray(r[c]) for c in FlowBatch.COLUMNS])

    def to_records(self) -> np.ndarray:
        cols = [c.cpu().numpy() if _is_torch(c) else np.asarray(c) for c in self.cols]
        out = np.zeros(self.n, FLOW_RECORD_DTYPE)
        for name, c in zip(self.COLUMNS, cols):
            out[name] = c.view(np.uint32 if c.itemsize == 4 else np.uint64)
        out["first"] = (out["start_ms"] & 0xFFFFFFFF).astype(np.uint32)
        out["last"] = (out["end_ms"] & 0xFFFFFFFF).astype(np.uint32)
        return out

    def to_device(self, device="cuda") -> "FlowBatch":
        import torch
        cols = []
        for c in self.cols:
            if _is_torch(c):
                cols.append(c.to(device))
            else:
                a = np.asarray(c)
                cols.append(torch.from_numpy(a.view(np.int32 if a.itemsize == 4 else np.int64)).to(device))
        return FlowBatch(*cols)


class FlowRecords:
    """64-byte flowmon::FlowRecord AoS (netflow.hpp:59-67), host or device."""

    def __init__(self, records):
        if _is_torch(records):
            if not records.is_contiguous():
                raise ValueError("records must be contiguous")
            nbytes = records.numel() * records.element_size()
            self.ptr, self.on_device = records.data_ptr(), bool(records.is_cuda)
        else:
            a = np.asarray(records)
            if not a.flags.c_contiguous:
                raise ValueError("records must be C-contiguous")
            nbytes, self.ptr, self.on_device = a.nbytes, a.ctypes.data, False
        if nbytes % _lib.FLOW_RECORD_BYTES:
            raise ValueError("record buffer is not a multiple of 64 bytes")
        self.n = nbytes // _lib.FLOW_RECORD_BYTES
        self.records = records

    def __len__(self) -> int:
        return self.n

    def _c(self) -> gnm_batch_aos:
        return gnm_batch_aos(self.ptr, self.n, _lib.MEM_DEVICE if self.on_device else _lib.MEM_HOST)


# ---- results ------------------------------------------------------------------

@dataclass
class RateStats:
    max_bps: float = 0.0
    min_bps: float = 0.0
    avg_bps: float = 0.0
    median_bps: float = 0.0
    flow_count: int = 0


@dataclass
class HostResult:
    """rate_engine.hpp:84-91: one host's RateStats (and histogram when requested)."""
    stats: RateStats
    rate_ubps_sum: int = 0
    histogram: Optional[np.ndarray] = None


@dataclass
class SiteResult:
    stats: RateStats
    octets: int = 0                 # north-star byte sum (oracle extension)
    rate_ubps_sum: int = 0          # exact u128 sum of per-flow micro-bps
    below_threshold: bool = False   # K3 flag: median < threshold
    histogram: Optional[np.ndarray] = None  # 10001 u32 when requested
    hosts: dict = field(default_factory=dict)  # host IP -> HostResult (Engine.set_hosts)


@dataclass
class ClassTallies:
    forward: int = 0
    pure_ack: int = 0
    administrative: int = 0
    unmatched: int = 0

    def total(self) -> int:
        return self.forward + self.pure_ack + self.administrative + self.unmatched


class AnalysisResult:
    """rate_engine.hpp:112-119 at site level. ``sites`` (SiteId -> SiteResult,
    only sites with Forward flows, as the reference's map) is built lazily
    from ``table``, the raw gnm_site_stats rows of every registered site."""

    def __init__(self, window_start_ms: int = 0, window_end_ms: int = 0, sites: Optional[dict] = None,
                 tallies: Optional[ClassTallies] = None, table: Optional[np.ndarray] = None,
                 histograms: Optional[np.ndarray] = None,
                 threshold_bps: float = kDefaultWarnThresholdBps):
        self.window_start_ms = window_start_ms
        self.window_end_ms = window_end_ms
        self.tallies = tallies or ClassTallies()
        self.table = table
        self.histograms = histograms
        self.threshold_bps = threshold_bps
        self._sites = sites
        self.host_table = None       # HOST_STATS_DTYPE rows in (site, host) order (hosts mode)
        self.host_histograms = None  # [rows, 10001] u32 when requested

    @property
    def sites(self) -> dict:
        if self._sites is None:
            self._sites = {}
            t = self.table
            if t is not None:
                for s in np.nonzero(t["flow_count"])[0].tolist():
                    row = t[s].tolist()  # one conversion per row
                    (cnt, octs, lo, hi, mn, mx, avg, med, below, _) = row
                    self._sites[s] = SiteResult(
                        stats=RateStats(max_bps=mx, min_bps=mn, avg_bps=avg, median_bps=med,
                                        flow_count=cnt),
                        octets=octs, rate_ubps_sum=hi << 64 | lo, below_threshold=bool(below),
                        histogram=None if self.histograms is None else self.histograms[s])
            if self.host_table is not None:
                for i, row in enumerate(self.host_table.tolist()):
                    (site, host, cnt, lo, hi, mn, mx, avg, med) = row
                    self._sites[site].hosts[host] = HostResult(
                        stats=RateStats(max_bps=mx, min_bps=mn, avg_bps=avg, median_bps=med,
                                        flow_count=cnt),
                        rate_ubps_sum=hi << 64 | lo,
                        histogram=None if self.host_histograms is None else self.host_histograms[i])
        return self._sites

    @staticmethod
    def from_site_stats(n_sites: int, stats: dict, window_end_ms: int = 0) -> "AnalysisResult":
        """A result holding the given per-site RateStats (tests of the
        warning rule build results directly, monitor_test.cpp:23-47)."""
        t = np.zeros(n_sites, SITE_STATS_DTYPE)
        for s, st in stats.items():
            t[s]["flow_count"] = st.flow_count
            t[s]["median_bps"] = st.median_bps
            t[s]["min_bps"] = st.min_bps
            t[s]["max_bps"] = st.max_bps
            t[s]["avg_bps"] = st.avg_bps
        return AnalysisResult(window_end_ms=window_end_ms, table=t)

    def _c(self) -> gnm_result:
        t = self.table if self.table is not None else np.zeros(0, SITE_STATS_DTYPE)
        r = gnm_result()
        r.window_start_ms = self.window_start_ms
        r.window_end_ms = self.window_end_ms
        r.threshold_bps = self.threshold_bps
        r.sites_capacity = len(t)
        r.sites = t.ctypes.data if len(t) else None
        r.n_sites = len(t)
        return r


def _build_result(r: gnm_result, table: np.ndarray, hist: Optional[np.ndarray]) -> AnalysisResult:
    return AnalysisResult(window_start_ms=r.window_start_ms, window_end_ms=r.window_end_ms,
                          tallies=ClassTallies(r.tallies.forward, r.tallies.pure_ack,
                                               r.tallies.administrative, r.tallies.unmatched),
                          table=table, histograms=hist, threshold_bps=r.threshold_bps)


# ---- the device engine -----------------------------------------------------------

class Engine:
    """One gnm_ctx: a GPU, its streams, device partials and loader buffers."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.gnm_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._hosts = False

    @classmethod
    def _borrow(cls, handle, device: int) -> "Engine":
        """A non-owning Engine over a context owned elsewhere (a Group's rank)."""
        e = cls.__new__(cls)
        e._h = C.c_void_p(handle)
        e.device = device
        e._hosts = False
        e._owned = False
        return e

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "_owned", True):
                lib.gnm_ctx_destroy(self._h)
            self._h = None

    # ---- multi-GPU inside the library (gnetmon.h gnm_ctx_comm_*) -------------
    @staticmethod
    def comm_unique_id() -> bytes:
        """ncclGetUniqueId, for rank 0 to distribute (gnm_comm_unique_id)."""
        buf = (C.c_ubyte * _lib.COMM_ID_BYTES)()
        _check(lib.gnm_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, nranks: int, rank: int, unique_id: bytes) -> None:
        """Attach an NCCL communicator: from now on every finalize / aggregate
        combines the ranks' partials itself (two rounds, on this context's
        stream) and returns the global result. Blocks until all ranks join."""
        buf = (C.c_ubyte * _lib.COMM_ID_BYTES).from_buffer_copy(unique_id)
        _check(lib.gnm_ctx_comm_init(self._h, nranks, rank, buf))

    def comm_destroy(self) -> None:
        _check(lib.gnm_ctx_comm_destroy(self._h))

    def comm_size(self) -> int:
        return lib.gnm_ctx_comm_size(self._h)

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_stream(self, stream) -> None:
        """Run on an external CUDA stream (torch.cuda.Stream, raw handle or None)."""
        ptr = getattr(stream, "cuda_stream", stream)
        _check(lib.gnm_ctx_set_stream(self._h, C.c_void_p(ptr) if ptr else None))

    def stream_handle(self) -> int:
        """The cudaStream_t the engine launches on (for torch.cuda.ExternalStream)."""
        return lib.gnm_ctx_stream(self._h) or 0

    def set_chunk_records(self, n: int) -> None:
        _check(lib.gnm_ctx_set_chunk_records(self._h, n))

    def set_hot_mode(self, mode: str) -> None:
        """"auto" (default), "off" or "force" block-private hot-site accumulation."""
        m = {"off": _lib.HOT_OFF, "auto": _lib.HOT_AUTO, "force": _lib.HOT_FORCE}[mode]
        _check(lib.gnm_ctx_set_hot_mode(self._h, m))

    def set_graphs(self, on: bool = True) -> None:
        """Replay one CUDA graph for repeated device-batch analyses (default on)."""
        _check(lib.gnm_ctx_set_graphs(self._h, 1 if on else 0))

    def set_hosts(self, on: bool = True) -> None:
        """Per-host mode (SiteResult::hosts, rate_engine.cpp:272-289): every
        later result carries ``host_table`` and ``sites[s].hosts``. Only
        between accumulations."""
        _check(lib.gnm_ctx_set_hosts(self._h, 1 if on else 0))
        self._hosts = bool(on)

    def _attach_hosts(self, res: AnalysisResult, histograms: bool) -> AnalysisResult:
        if not getattr(self, "_hosts", False):
            return res
        n = lib.gnm_host_count(self._h)
        rows = _pinned_rows(max(n, 1))
        hist = np.empty((max(n, 1), BUCKET_COUNT), np.uint32) if histograms else None
        _check(lib.gnm_host_results(self._h, rows.ctypes.data, len(rows),
                                    hist.ctypes.data if hist is not None else None))
        res.host_table = rows[:n]
        res.host_histograms = None if hist is None else hist[:n]
        return res

    def host_histogram_entries(self):
        """The last hosts-mode result's per-host histograms, sparse: (row,
        bucket, count) arrays in (row, bucket) order, row indexing
        ``host_table`` (HostResult::histogram without the 40 KB per host)."""
        n = C.c_uint64()
        _check(lib.gnm_host_histogram_entries(self._h, None, None, None, 0, C.byref(n)))
        rows, bks, cnt = (np.empty(max(n.value, 1), np.uint32) for _ in range(3))
        _check(lib.gnm_host_histogram_entries(self._h, rows.ctypes.data, bks.ctypes.data, cnt.ctypes.data,
                                              len(rows), C.byref(n)))
        k = n.value
        return rows[:k], bks[:k], cnt[:k]

    def enable_timing(self, on: bool = True) -> None:
        _check(lib.gnm_ctx_enable_timing(self._h, 1 if on else 0))

    def timing(self) -> dict:
        t = gnm_timing()
        _check(lib.gnm_ctx_timing(self._h, C.byref(t)))
        return {"accumulate_ms": t.accumulate_ms, "finalize_ms": t.finalize_ms,
                "h2d_ms": t.h2d_ms, "k2_launches": t.k2_launches,
                "kernel_launches": t.kernel_launches, "records": t.records,
                "plan_ms": t.plan_ms, "total_plan_ms": t.total_plan_ms,
                "total_accumulate_ms": t.total_accumulate_ms,
                "total_finalize_ms": t.total_finalize_ms, "total_finalizes": t.total_finalizes,
                "total_k2_launches": t.total_k2_launches, "h2d_bytes": t.h2d_bytes}

    @staticmethod
    def _params(params: Optional[FilterParams]) -> gnm_filter_params:
        return (params or FilterParams())._c()

    def accumulate(self, batch, catalog: SiteCatalog, params: Optional[FilterParams] = None,
                   window: Optional[tuple] = None) -> None:
        """Add a batch to the accumulation. ``window=(start_ms, end_ms)``
        fuses FlowStore::snapshot (flow_store.cpp:62-80): only records with
        end_ms in [start_ms, end_ms) are analyzed."""
        p = self._params(params)
        b = batch._c()
        aos = isinstance(batch, FlowRecords)
        if window is not None:
            ws, we = int(window[0]), int(window[1])
            fn = lib.gnm_accumulate_window_aos if aos else lib.gnm_accumulate_window
            _check(fn(self._h, catalog.handle, C.byref(p), C.byref(b), ws, we))
        elif aos:
            _check(lib.gnm_accumulate_aos(self._h, catalog.handle, C.byref(p), C.byref(b)))
        else:
            _check(lib.gnm_accumulate(self._h, catalog.handle, C.byref(p), C.byref(b)))

    def _result(self, catalog: SiteCatalog, window_start_ms: int, window_end_ms: int,
                threshold_bps: float, histograms: bool):
        n = catalog.site_count()
        # gnm_finalize writes every row: no zero-fill on the step's critical path.
        table = np.empty(max(n, 1), SITE_STATS_DTYPE)
        hist = np.zeros((max(n, 1), BUCKET_COUNT), np.uint32) if histograms else None
        r = gnm_result()
        r.window_start_ms = window_start_ms
        r.window_end_ms = window_end_ms
        r.threshold_bps = threshold_bps
        r.sites_capacity = len(table)
        r.sites = table.ctypes.data
        r.histograms = hist.ctypes.data if hist is not None else None
        return r, table, hist, n

    def finalize(self, catalog: SiteCatalog, window_start_ms: int = 0, window_end_ms: int = 0,
                 threshold_bps: float = kDefaultWarnThresholdBps,
                 histograms: bool = False) -> AnalysisResult:
        r, table, hist, n = self._result(catalog, window_start_ms, window_end_ms, threshold_bps,
                                         histograms)
        _check(lib.gnm_finalize(self._h, catalog.handle, C.byref(r)))
        return self._attach_hosts(_build_result(r, table[:n], None if hist is None else hist[:n]), histograms)

    def reset(self) -> None:
        _check(lib.gnm_reset(self._h))

    def aggregate(self, view, catalog: SiteCatalog, params: Optional[FilterParams] = None,
                  workers: int = 1, mode: LookupMode = LookupMode.Hash, window_start_ms: int = 0,
                  window_end_ms: int = 0, threshold_bps: float = kDefaultWarnThresholdBps,
                  histograms: bool = False) -> AnalysisResult:
        """rate_engine.hpp:143-146. ``workers``/``mode`` are accepted and ignored:
        results are identical for any worker count and lookup mode by contract
        (engine_test.cpp:344-360). One gnm_analyze call."""
        p = self._params(params)
        b = view._c()
        r, table, hist, n = self._result(catalog, window_start_ms, window_end_ms, threshold_bps,
                                         histograms)
        if isinstance(view, FlowRecords):
            _check(lib.gnm_analyze_aos(self._h, catalog.handle, C.byref(p), C.byref(b), C.byref(r)))
        else:
            _check(lib.gnm_analyze(self._h, catalog.handle, C.byref(p), C.byref(b), C.byref(r)))
        return self._attach_hosts(_build_result(r, table[:n], None if hist is None else hist[:n]), histograms)

    def aggregate_window(self, view, catalog: SiteCatalog, window_start_ms: int, window_end_ms: int,
                         params: Optional[FilterParams] = None,
                         threshold_bps: float = kDefaultWarnThresholdBps,
                         histograms: bool = False) -> AnalysisResult:
        """FlowStore::snapshot(start, end) + aggregate(..., start, end) fused
        (monitor.cpp:109-120, run_cycle): records outside [start, end) by
        end_ms are neither analyzed nor tallied."""
        if isinstance(view, FlowRecords):
            self.accumulate(view, catalog, params, window=(window_start_ms, window_end_ms))
            return self.finalize(catalog, window_start_ms, window_end_ms, threshold_bps, histograms)
        p = self._params(params)
        b = view._c()
        r, table, hist, n = self._result(catalog, window_start_ms, window_end_ms, threshold_bps,
                                         histograms)
        _check(lib.gnm_analyze_window(self._h, catalog.handle, C.byref(p), C.byref(b), C.byref(r)))
        return self._attach_hosts(_build_result(r, table[:n], None if hist is None else hist[:n]), histograms)

    def decode_netflow(self, datagrams, offsets, out_device: bool = False):
        """Batched Collector::ingest_datagram without the store
        (collector.cpp:101-129): NetFlow v5 datagrams -> FlowRecord rows on
        the GPU (gnm_decode_netflow). ``datagrams``: one byte buffer (numpy
        uint8 or a CUDA uint8 tensor), ``offsets``: n+1 u64 boundaries.
        Returns (records, status, stats): records as a FLOW_RECORD_DTYPE
        array (or a CUDA uint8 tensor of rows when ``out_device``), status
        per datagram (0 ok, 1 bad version, 2 truncated, 3 bad count) and the
        collector's counters."""
        n = len(offsets) - 1
        if _is_torch(datagrams):
            import torch
            offs = offsets if _is_torch(offsets) else torch.as_tensor(np.asarray(offsets, np.uint64).view(np.int64),
                                                                       device=datagrams.device)
            d_ptr, nbytes, off_ptr, mem = datagrams.data_ptr(), datagrams.numel(), offs.data_ptr(), _lib.MEM_DEVICE
        else:
            buf = np.ascontiguousarray(datagrams, np.uint8)
            offs = np.ascontiguousarray(offsets, np.uint64)
            d_ptr = buf.ctypes.data if buf.size else None
            nbytes, off_ptr, mem = buf.size, offs.ctypes.data, _lib.MEM_HOST
        cap = 30 * n
        status = np.zeros(max(n, 1), np.uint8)
        st = gnm_netflow_stats()
        if out_device:
            import torch
            out = torch.empty(max(cap, 1) * 64, dtype=torch.uint8, device=f"cuda:{self.device}")
            out_ptr, out_mem = out.data_ptr(), _lib.MEM_DEVICE
        else:
            out = np.zeros(max(cap, 1), FLOW_RECORD_DTYPE)
            out_ptr, out_mem = out.ctypes.data, _lib.MEM_HOST
        _check(lib.gnm_decode_netflow(self._h, d_ptr, nbytes, off_ptr, n, mem, out_ptr, cap, out_mem,
                                      status.ctypes.data, C.byref(st)))
        k = st.records_accepted
        recs = out[:k * 64] if out_device else out[:k]
        stats = {"datagrams": st.datagrams, "decode_errors": st.decode_errors,
                 "records_rejected": st.records_rejected, "records_accepted": k}
        return recs, status[:n], stats

    @staticmethod
    def _archive_arg(archive):
        if _is_torch(archive):
            return archive.data_ptr(), archive.numel(), (_lib.MEM_DEVICE if archive.is_cuda else _lib.MEM_HOST), archive
        a = np.frombuffer(archive, np.uint8) if isinstance(archive, (bytes, bytearray)) else \
            np.ascontiguousarray(archive, np.uint8)
        return (a.ctypes.data if a.size else None), a.size, _lib.MEM_HOST, a

    def decode_archive(self, archive) -> np.ndarray:
        """FlowStore::load (flow_store.cpp:167-207) of an in-memory FLOWARC1
        archive (bytes, numpy uint8 or a uint8 tensor) on the GPU:
        FLOW_RECORD_DTYPE rows. Raises ArchiveError as the reference does."""
        ptr, n, mem, keep = self._archive_arg(archive)
        cap = max((n - 20) // 64, 0) if n >= 20 else 0
        out = np.zeros(max(cap, 1), FLOW_RECORD_DTYPE)
        k = C.c_uint64()
        _check(lib.gnm_decode_archive(self._h, ptr, n, mem, out.ctypes.data, cap, _lib.MEM_HOST, C.byref(k)))
        return out[:k.value]

    def aggregate_archive(self, archive, catalog: SiteCatalog, params: Optional[FilterParams] = None,
                          window_start_ms: int = 0, window_end_ms: int = 0,
                          threshold_bps: float = kDefaultWarnThresholdBps,
                          histograms: bool = False) -> AnalysisResult:
        """aggregate(FlowStore::load(archive), ...) (flowmon.cpp analyze):
        K2 reads the archive's big-endian entries in place."""
        ptr, n, mem, keep = self._archive_arg(archive)
        p = self._params(params)
        r, table, hist, ns = self._result(catalog, window_start_ms, window_end_ms, threshold_bps,
                                          histograms)
        _check(lib.gnm_analyze_archive(self._h, catalog.handle, C.byref(p), ptr, n, mem, C.byref(r)))
        return self._attach_hosts(_build_result(r, table[:ns], None if hist is None else hist[:ns]), histograms)

    def partials(self, catalog: SiteCatalog) -> dict:
        """Device pointers of the accumulation (gnm_get_partials) for a
        cross-GPU all-reduce; wrap with ``device_tensors``."""
        p = gnm_partials()
        _check(lib.gnm_get_partials(self._h, catalog.handle, C.byref(p)))
        return {"sums": (p.sums, p.sums_count), "min_bps": (p.min_bps, p.n_sites),
                "max_bps": (p.max_bps, p.n_sites), "coarse": (p.coarse, p.coarse_count),
                "fine": (p.fine, p.fine_count), "n_sites": p.n_sites}

    def prepare_median(self, catalog: SiteCatalog) -> None:
        """Round 2 of the exact median (gnm_prepare_median): after the
        sums/min/max/coarse all-reduce, find every site's median
        super-bucket and count this context's flows inside it into ``fine``
        (then all-reduce ``fine`` and finalize)."""
        _check(lib.gnm_prepare_median(self._h, catalog.handle))

    def device_tensors(self, catalog: SiteCatalog) -> dict:
        """torch views of the device partials (zero-copy, __cuda_array_interface__)."""
        import torch
        p = self.partials(catalog)

        class _View:
            def __init__(self, ptr, n, typestr):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                                 "data": (ptr, False), "version": 3}

        dev = torch.device("cuda", self.device)
        return {
            "sums": torch.as_tensor(_View(p["sums"][0], p["sums"][1], "<i8"), device=dev),
            "min_bps": torch.as_tensor(_View(p["min_bps"][0], p["min_bps"][1], "<f8"), device=dev),
            "max_bps": torch.as_tensor(_View(p["max_bps"][0], p["max_bps"][1], "<f8"), device=dev),
            "coarse": torch.as_tensor(_View(p["coarse"][0], p["coarse"][1], "<i4"), device=dev),
            "fine": torch.as_tensor(_View(p["fine"][0], p["fine"][1], "<i4"), device=dev),
        }

    # -- per-host rows across GPUs (gnetmon.h gnm_hosts_*) --------------------------
    def _view(self, ptr, n, typestr):
        import torch

        class _V:
            def __init__(self):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3}
        return torch.as_tensor(_V(), device=torch.device("cuda", self.device))

    def hosts_local_keys(self, catalog: SiteCatalog):
        """This context's distinct (site << 32 | host) keys, sorted: a zero-copy
        int64 CUDA tensor (valid until finalize)."""
        import torch
        ptr, n = C.c_void_p(), C.c_uint64()
        _check(lib.gnm_hosts_local_keys(self._h, catalog.handle, C.byref(ptr), C.byref(n)))
        if n.value == 0:
            return torch.empty(0, dtype=torch.int64, device=torch.device("cuda", self.device))
        return self._view(ptr.value, n.value, "<i8")

    def hosts_set_keys(self, keys) -> dict:
        """Round 1 of the per-host combine: partials of the sorted key union
        (an int64 CUDA tensor on this device) as zero-copy tensors."""
        keys = keys.contiguous()
        p = _lib.gnm_host_partials()
        _check(lib.gnm_hosts_set_keys(self._h, keys.data_ptr() if keys.numel() else None, keys.numel(),
                                      C.byref(p)))
        n = max(p.n, 1)
        return {"sums": self._view(p.sums, 3 * n, "<i8"), "min_bps": self._view(p.min, n, "<f8"),
                "max_bps": self._view(p.max, n, "<f8"), "coarse": self._view(p.coarse, 157 * n, "<i4"),
                "fine": self._view(p.fine, 64 * n, "<i4"), "n": p.n}

    def hosts_prepare_median(self) -> None:
        _check(lib.gnm_hosts_prepare_median(self._h))

    def classify(self, batch: FlowBatch, catalog: SiteCatalog,
                 params: Optional[FilterParams] = None, out=None):
        """Per-record class << 30 | site (gnm_classify)."""
        p = self._params(params)
        b = batch._c()
        if out is None:
            out = np.zeros(batch.n, np.uint32)
        if _is_torch(out):
            ptr, mem = out.data_ptr(), (_lib.MEM_DEVICE if out.is_cuda else _lib.MEM_HOST)
        else:
            ptr, mem = out.ctypes.data, _lib.MEM_HOST
        _check(lib.gnm_classify(self._h, catalog.handle, C.byref(p), C.byref(b), ptr, mem))
        return out


_tls = threading.local()


def default_engine(device: Optional[int] = None) -> Engine:
    if device is None:
        device = 0
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    if device not in engines:
        engines[device] = Engine(device)
    return engines[device]


def aggregate(view, catalog: SiteCatalog, params: Optional[FilterParams] = None,
              workers: int = 1, mode: LookupMode = LookupMode.Hash, window_start_ms: int = 0,
              window_end_ms: int = 0, **kw) -> AnalysisResult:
    """flowmon::aggregate (rate_engine.hpp:143-146) on the GPU."""
    return default_engine().aggregate(view, catalog, params, workers, mode, window_start_ms,
                                      window_end_ms, **kw)


def aggregate_partitioned(view: FlowBatch, catalog: SiteCatalog, params: Optional[FilterParams],
                          boundaries: Sequence[int], mode: LookupMode = LookupMode.Hash,
                          window_start_ms: int = 0, window_end_ms: int = 0,
                          **kw) -> AnalysisResult:
    """flowmon::aggregate_partitioned (rate_engine.hpp:149-154): each slice
    is accumulated by its own K2 launch into the same partials."""
    eng = default_engine()
    prev = 0
    for b in list(boundaries) + [len(view)]:
        eng.accumulate(view.slice(prev, b), catalog, params)
        prev = b
    return eng.finalize(catalog, window_start_ms, window_end_ms, **kw)


# ---- warnings ------------------------------------------------------------------

class WarningState:
    """monitor.hpp:20-37 (per-site streak counters)."""

    def __init__(self):
        h = C.c_void_p()
        _check(lib.gnm_warning_state_create(C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.gnm_warning_state_destroy(self._h)
            self._h = None

    def streak(self, site: SiteId) -> int:
        return lib.gnm_warning_state_streak(self._h, site)


@dataclass
class SiteWarning:
    site: SiteId = 0
    site_name: str = ""
    median_bps: float = 0.0
    consecutive_bad_hours: int = 0


def evaluate_warnings(result: AnalysisResult, catalog: SiteCatalog, state: WarningState,
                      threshold_bps: float = kDefaultWarnThresholdBps) -> list[SiteWarning]:
    """monitor.cpp:13-34: median < threshold extends a site's streak, a good
    hour resets it, zero-flow sites are frozen, streak >= 2 warns."""
    r = result._c()
    cap = max(r.n_sites, 1)
    out = (gnm_warning * cap)()
    n = C.c_size_t()
    _check(lib.gnm_evaluate_warnings(C.byref(r), state._h, threshold_bps, out, cap, C.byref(n)))
    return [SiteWarning(out[i].site, catalog.site(out[i].site), out[i].median_bps,
                        out[i].consecutive_bad_hours) for i in range(n.value)]


class Group:
    """One process driving several GPUs (gnetmon.h gnm_group_*): a context per
    device and an NCCL clique; ``aggregate`` shards the batch by the
    reference's worker boundaries n*i/N (rate_engine.cpp:341-344), every rank
    accumulates its shard on its own host thread and the partials combine in
    two rounds inside the library. ``kind="loopback"`` exchanges through host
    memory instead (a test hook: several ranks on one GPU)."""

    def __init__(self, devices, kind: str = "nccl"):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        k = {"nccl": _lib.GROUP_NCCL, "loopback": _lib.GROUP_LOOPBACK}[kind]
        _check(lib.gnm_group_create(devs, len(devices), k, C.byref(h)))
        self._h = h
        self.devices = list(devices)
        self.engines = [Engine._borrow(lib.gnm_group_ctx(h, i), d) for i, d in enumerate(devices)]
        self._hosts = False

    def close(self):
        if getattr(self, "_h", None):
            lib.gnm_group_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __len__(self):
        return lib.gnm_group_size(self._h)

    def set_hosts(self, on: bool = True) -> None:
        for e in self.engines:
            e.set_hosts(on)
        self._hosts = bool(on)

    def aggregate(self, view, catalog: SiteCatalog, params: Optional[FilterParams] = None,
                  window_start_ms: int = 0, window_end_ms: int = 0,
                  threshold_bps: float = kDefaultWarnThresholdBps, histograms: bool = False) -> AnalysisResult:
        p = Engine._params(params)
        b = view._c()
        r, table, hist, n = self.engines[0]._result(catalog, window_start_ms, window_end_ms, threshold_bps,
                                                    histograms)
        fn = lib.gnm_group_analyze_aos if isinstance(view, FlowRecords) else lib.gnm_group_analyze
        _check(fn(self._h, catalog.handle, C.byref(p), C.byref(b), C.byref(r)))
        res = _build_result(r, table[:n], None if hist is None else hist[:n])
        if self._hosts:
            k = lib.gnm_group_host_count(self._h)
            rows = _pinned_rows(max(k, 1))
            _check(lib.gnm_group_host_results(self._h, rows.ctypes.data, len(rows)))
            res.host_table = rows[:k]
            res.host_histograms = None
        return res

    def host_histogram_entries(self):
        """The group's per-host histograms (summed over the ranks), sparse:
        (row, bucket, count) in (row, bucket) order."""
        n = C.c_uint64()
        _check(lib.gnm_group_host_histogram_entries(self._h, None, None, None, 0, C.byref(n)))
        rows, bks, cnt = (np.empty(max(n.value, 1), np.uint32) for _ in range(3))
        _check(lib.gnm_group_host_histogram_entries(self._h, rows.ctypes.data, bks.ctypes.data, cnt.ctypes.data,
                                                    len(rows), C.byref(n)))
        k = n.value
        return rows[:k], bks[:k], cnt[:k]
