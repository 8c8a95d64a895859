"""ctypes wrappers of the C restatement and the compiled reference.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(_HERE, "lib", "liborc.so")
REF_PATH = os.path.join(_HERE, "_ref", "libflowmon_ref.so")
BUCKETS = 10001
NO_SITE = 0xFFFFFFFF
DEFAULT_PARAMS = (96, 20, 100)


class _Params(C.Structure):
    _fields_ = [("ack_avg_size_max", C.c_uint32), ("min_packets", C.c_uint32),
                ("min_duration_ms", C.c_uint32), ("workers", C.c_uint32)]


def _p(a) -> int:
    return np.ascontiguousarray(a).ctypes.data


def _cols(cols):
    src, dst, pkts, octs, start, end = cols
    return (np.ascontiguousarray(src, np.uint32), np.ascontiguousarray(dst, np.uint32),
            np.ascontiguousarray(pkts, np.uint32), np.ascontiguousarray(octs, np.uint32),
            np.ascontiguousarray(start, np.uint64), np.ascontiguousarray(end, np.uint64))


class Oracle:
    """The plain-C restatement (gnm_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORC_PATH):
            raise ImportError(f"{ORC_PATH} missing: run `make -C oracle`")
        L = C.CDLL(ORC_PATH)
        V = C.c_void_p
        L.orc_catalog_create.restype = V
        L.orc_catalog_create.argtypes = [V, V, C.c_size_t]
        L.orc_catalog_destroy.argtypes = [V]
        L.orc_lookup.restype = C.c_uint32
        L.orc_lookup.argtypes = [V, C.c_uint32]
        L.orc_sequential_lookup.restype = C.c_uint32
        L.orc_sequential_lookup.argtypes = [V, C.c_uint32]
        L.orc_cidr_first_prefix24.restype = C.c_uint32
        L.orc_cidr_first_prefix24.argtypes = [C.c_uint32, C.c_int]
        L.orc_cidr_last_prefix24.restype = C.c_uint32
        L.orc_cidr_last_prefix24.argtypes = [C.c_uint32, C.c_int]
        L.orc_flow_rate.restype = C.c_double
        L.orc_flow_rate.argtypes = [C.c_uint32, C.c_uint64]
        L.orc_rate_ubps_parts.argtypes = [C.c_uint32, C.c_uint64, V, V]
        L.orc_bucket_index.restype = C.c_uint32
        L.orc_bucket_index.argtypes = [C.c_double]
        L.orc_classify.argtypes = [V] * 6 + [C.c_size_t, C.POINTER(_Params), V, V]
        L.orc_aggregate.argtypes = ([V] * 6 + [C.c_size_t, C.POINTER(_Params), V, C.c_int,
                                                C.c_uint32] + [V] * 8)
        L.orc_median_bps.restype = C.c_double
        L.orc_median_bps.argtypes = [V, C.c_uint64]
        L.orc_site_stats.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                     V, V, V]
        L.orc_evaluate_warnings.restype = C.c_size_t
        L.orc_evaluate_warnings.argtypes = [C.c_uint32, V, V, V, C.c_double, V]
        L.orc_flow_keys.argtypes = [V] * 6 + [C.c_size_t, C.POINTER(_Params), V] + [V] * 7
        L.orc_u128_to_double.restype = C.c_double
        L.orc_u128_to_double.argtypes = [C.c_uint64, C.c_uint64]
        self.L = L

    # -- catalog --------------------------------------------------------------
    def catalog(self, prefix24, site) -> "OrcCatalog":
        p = np.ascontiguousarray(prefix24, np.uint32)
        s = np.ascontiguousarray(site, np.uint32)
        return OrcCatalog(self.L, self.L.orc_catalog_create(_p(p), _p(s), len(p)))

    def lookup(self, cat: "OrcCatalog", ip: int) -> Optional[int]:
        s = self.L.orc_lookup(cat.h, ip)
        return None if s == NO_SITE else s

    def sequential_lookup(self, cat: "OrcCatalog", ip: int) -> Optional[int]:
        s = self.L.orc_sequential_lookup(cat.h, ip)
        return None if s == NO_SITE else s

    # -- scalar functions -----------------------------------------------------
    def flow_rate(self, octets: int, duration: int) -> float:
        return self.L.orc_flow_rate(octets, duration)

    def rate_ubps(self, octets: int, duration: int) -> int:
        lo, hi = C.c_uint64(), C.c_uint64()
        self.L.orc_rate_ubps_parts(octets, duration, C.byref(lo), C.byref(hi))
        return hi.value << 64 | lo.value

    def bucket_index(self, rate: float) -> int:
        return self.L.orc_bucket_index(rate)

    def median_bps(self, row: np.ndarray, count: int) -> float:
        r = np.ascontiguousarray(row, np.uint32)
        return self.L.orc_median_bps(_p(r), count)

    # -- batch functions ------------------------------------------------------
    def classify(self, cols, cat: "OrcCatalog", params=DEFAULT_PARAMS) -> np.ndarray:
        c = _cols(cols)
        out = np.zeros(len(c[0]), np.uint32)
        p = _Params(*params, 1)
        self.L.orc_classify(*[_p(x) for x in c], len(c[0]), C.byref(p), cat.h, _p(out))
        return out

    def aggregate(self, cols, cat: "OrcCatalog", n_sites: int, params=DEFAULT_PARAMS,
                  sequential: bool = False, acc: Optional[dict] = None) -> dict:
        """reduce_slice + finalize's site merge; ``acc`` continues a chunked run."""
        c = _cols(cols)
        if acc is None:
            acc = {"count": np.zeros(n_sites, np.uint64), "octets": np.zeros(n_sites, np.uint64),
                   "ubps_lo": np.zeros(n_sites, np.uint64), "ubps_hi": np.zeros(n_sites, np.uint64),
                   "min": np.full(n_sites, np.inf), "max": np.zeros(n_sites),
                   "hist": np.zeros((n_sites, BUCKETS), np.uint32),
                   "tallies": np.zeros(4, np.uint64)}
        p = _Params(*params, 1)
        self.L.orc_aggregate(*[_p(x) for x in c], len(c[0]), C.byref(p), cat.h,
                             1 if sequential else 0, n_sites,
                             *[acc[k].ctypes.data for k in ("count", "octets", "ubps_lo", "ubps_hi",
                                                           "min", "max", "hist", "tallies")])
        return acc

    def finalize(self, acc: dict) -> dict:
        """stats_from per site: adds avg / median (count 0 -> 0)."""
        n = len(acc["count"])
        avg = np.zeros(n)
        med = np.zeros(n)
        a, m = C.c_double(), C.c_double()
        for s in range(n):
            self.L.orc_site_stats(int(acc["count"][s]), int(acc["ubps_lo"][s]), int(acc["ubps_hi"][s]),
                                  float(acc["min"][s]), float(acc["max"][s]), acc["hist"][s].ctypes.data,
                                  C.byref(a), C.byref(m))
            avg[s], med[s] = a.value, m.value
        out = dict(acc)
        out["avg"] = avg
        out["median"] = med
        return out

    def analyze(self, cols, cat: "OrcCatalog", n_sites: int, params=DEFAULT_PARAMS) -> dict:
        return self.finalize(self.aggregate(cols, cat, n_sites, params))

    def flow_keys(self, cols, cat: "OrcCatalog", params=DEFAULT_PARAMS) -> dict:
        c = _cols(cols)
        n = len(c[0])
        out = {"cls": np.zeros(n, np.uint8), "site": np.zeros(n, np.uint32), "host": np.zeros(n, np.uint32),
               "bucket": np.zeros(n, np.uint32), "rate": np.zeros(n), "ubps_lo": np.zeros(n, np.uint64),
               "ubps_hi": np.zeros(n, np.uint64)}
        p = _Params(*params, 1)
        self.L.orc_flow_keys(*[_p(x) for x in c], n, C.byref(p), cat.h,
                             *[out[k].ctypes.data for k in ("cls", "site", "host", "bucket", "rate",
                                                           "ubps_lo", "ubps_hi")])
        return out

    def host_stats(self, cols, cat: "OrcCatalog", params=DEFAULT_PARAMS, hist: bool = False) -> dict:
        """SiteResult::hosts of finalize (rate_engine.cpp:272-289): one row per
        (site, host) in (site, host) order -- the std::map iteration order --
        with stats_from (:242-253) of the host's flows. ``hist``: sparse
        histograms (row, bucket, count)."""
        k = self.flow_keys(cols, cat, params)
        fwd = k["cls"] == 0
        key = (k["site"][fwd].astype(np.uint64) << np.uint64(32)) | k["host"][fwd].astype(np.uint64)
        bucket = k["bucket"][fwd]
        order = np.lexsort((bucket, key))
        key, bucket = key[order], bucket[order]
        rate, lo, hi = k["rate"][fwd][order], k["ubps_lo"][fwd][order], k["ubps_hi"][fwd][order]
        uk, start, cnt = np.unique(key, return_index=True, return_counts=True)
        n = len(uk)
        out = {"site": (uk >> np.uint64(32)).astype(np.uint32), "host": (uk & np.uint64(0xFFFFFFFF)).astype(np.uint32),
               "count": cnt.astype(np.uint64), "ubps_lo": np.zeros(n, np.uint64), "ubps_hi": np.zeros(n, np.uint64),
               "min": np.zeros(n), "max": np.zeros(n), "avg": np.zeros(n), "median": np.zeros(n)}
        if n == 0:
            return out
        m32 = np.uint64(0xFFFFFFFF)
        l0 = np.add.reduceat(lo & m32, start)
        l1 = np.add.reduceat(lo >> np.uint64(32), start)
        l2 = np.add.reduceat(hi, start)
        out["min"] = np.minimum.reduceat(rate, start)
        out["max"] = np.maximum.reduceat(rate, start)
        kmed = bucket[start + (cnt + 1) // 2 - 1]
        med = np.where(kmed == BUCKETS - 1, 100000000.0, kmed.astype(np.float64) * 10000.0 + 5000.0)
        out["median"] = np.minimum(np.maximum(med, out["min"]), out["max"])  # std::clamp
        for i in range(n):
            u = int(l0[i]) + (int(l1[i]) << 32) + (int(l2[i]) << 64)
            out["ubps_lo"][i] = u & (2**64 - 1)
            out["ubps_hi"][i] = u >> 64
            out["avg"][i] = (self.u128_to_double(u) / 1e6) / float(cnt[i])
        if hist:
            row = np.repeat(np.arange(n), cnt)
            pair = row.astype(np.uint64) << np.uint64(14) | bucket.astype(np.uint64)
            up, pc = np.unique(pair, return_counts=True)
            out["hist_row"] = (up >> np.uint64(14)).astype(np.uint32)
            out["hist_bucket"] = (up & np.uint64(0x3FFF)).astype(np.uint32)
            out["hist_count"] = pc.astype(np.uint32)
        return out

    def evaluate_warnings(self, count, median, streak: np.ndarray, threshold: float = 1e6):
        cnt = np.ascontiguousarray(count, np.uint64)
        med = np.ascontiguousarray(median, np.float64)
        warn = np.zeros(len(cnt), np.uint8)
        self.L.orc_evaluate_warnings(len(cnt), _p(cnt), _p(med), streak.ctypes.data, threshold,
                                     warn.ctypes.data)
        return warn

    def u128_to_double(self, v: int) -> float:
        return self.L.orc_u128_to_double(v & (2**64 - 1), v >> 64)


class OrcCatalog:
    def __init__(self, L, h):
        self.L, self.h = L, h

    def __del__(self):
        if self.h:
            self.L.orc_catalog_destroy(self.h)
            self.h = None


def reference_available() -> bool:
    return os.path.exists(REF_PATH)


class Reference:
    """The unmodified reference (flowmon) compiled in place, via ref_driver.cpp."""

    def __init__(self):
        if not os.path.exists(REF_PATH):
            raise ImportError(f"{REF_PATH} missing: run `make -C oracle ref` where "
                              "/root/reference exists")
        L = C.CDLL(REF_PATH)
        V, U32, U64, D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_flow_record_size": (C.c_size_t, []),
            "ref_catalog_create": (V, []),
            "ref_catalog_destroy": (None, [V]),
            "ref_catalog_register": (C.c_longlong, [V, C.c_char_p, C.c_char_p]),
            "ref_catalog_register_raw": (C.c_longlong, [V, C.c_char_p, V, V, C.c_size_t]),
            "ref_cidr_parse": (C.c_int, [C.c_char_p, V, V]),
            "ref_catalog_lookup": (U32, [V, U32]),
            "ref_catalog_sequential_lookup": (U32, [V, U32]),
            "ref_catalog_entry_count": (C.c_size_t, [V]),
            "ref_catalog_site_count": (C.c_size_t, [V]),
            "ref_catalog_entries": (C.c_size_t, [V, V, V, C.c_size_t]),
            "ref_records_create": (V, [V] * 6 + [C.c_size_t]),
            "ref_records_destroy": (None, [V]),
            "ref_records_size": (C.c_size_t, [V]),
            "ref_records_data": (V, [V]),
            "ref_generate": (V, [U32, U64, U64, C.c_size_t, V, V, V, V, V, V, V, V, V]),
            "ref_records_columns": (None, [V] * 7),
            "ref_classify": (C.c_int, [U32, U32, U32, U32, U64, U64, U32, U32, U32, V, C.c_int]),
            "ref_flow_rate": (C.c_int, [U32, U64, U64, V, V, V]),
            "ref_bucket_index": (C.c_size_t, [D]),
            "ref_attribute": (U32, [U32, U32, V, C.c_int, V]),
            "ref_hist_create": (V, []),
            "ref_hist_destroy": (None, [V]),
            "ref_hist_add": (None, [V, D, U64, U64]),
            "ref_hist_median": (C.c_int, [V, V]),
            "ref_aggregate": (V, [V, V, U32, U32, U32, U32, C.c_int, U64, U64, V]),
            "ref_aggregate_time_range": (D, [V, C.c_size_t, C.c_size_t, V, U32]),
            "ref_aggregate_partitioned": (V, [V, V, U32, U32, U32, V, C.c_size_t]),
            "ref_result_destroy": (None, [V]),
            "ref_result_equal": (C.c_int, [V, V]),
            "ref_result_tallies": (None, [V, V]),
            "ref_result_site_ids": (C.c_size_t, [V, V, C.c_size_t]),
            "ref_result_site": (C.c_int, [V, U32, V, V, V, V, V]),
            "ref_result_hosts": (C.c_size_t, [V, U32, V, C.c_size_t]),
            "ref_ingest_batch": (C.c_size_t, [V, V, C.c_size_t, V, V]),
            "ref_result_host": (C.c_int, [V, U32, U32, V, V, V, V]),
            "ref_site_sums": (None, [V, V, U32, U32, U32, U32, V, V, V]),
            "ref_wstate_create": (V, []),
            "ref_wstate_destroy": (None, [V]),
            "ref_wstate_streak": (U32, [V, U32]),
            "ref_evaluate_warnings": (C.c_size_t, [V, V, V, D, V, V, V, C.c_size_t]),
            "ref_ingest_datagram": (C.c_int, [V, C.c_size_t, V, V, V]),
            "ref_encode_packet": (C.c_size_t, [V, V, C.c_size_t, V]),
            "ref_raw_record_size": (C.c_size_t, []),
            "ref_archive_write": (C.c_int, [V, C.c_char_p]),
            "ref_archive_load": (V, [C.c_char_p, V]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    # -- NetFlow v5 (netflow.cpp, collector.cpp:101-129) -------------------------
    def ingest_datagram(self, datagram: bytes):
        """(status 0 | 1+CodecError::Kind, FlowRecord rows as bytes, rejected)."""
        buf = np.frombuffer(datagram, np.uint8) if len(datagram) else np.zeros(1, np.uint8)
        out = np.zeros(30 * 64, np.uint8)
        n = C.c_size_t()
        rej = C.c_uint32()
        st = self.L.ref_ingest_datagram(buf.ctypes.data, len(datagram), out.ctypes.data, C.byref(n),
                                        C.byref(rej))
        return st, out[: n.value * 64].tobytes(), rej.value

    def write_archive(self, rows: np.ndarray, path: str) -> None:
        """FlowStore::write_archive of FlowRecord rows (64-byte structured or
        uint8 array)."""
        b = np.ascontiguousarray(rows).view(np.uint8).reshape(-1, 64)
        import ctypes as _C
        n = len(b)
        cols = [np.ascontiguousarray(b[:, o:o + w]).view(t).ravel() for o, w, t in
                ((0, 4, np.uint32), (4, 4, np.uint32), (16, 4, np.uint32), (20, 4, np.uint32),
                 (48, 8, np.uint64), (56, 8, np.uint64))]
        h = self.L.ref_records_create(*[c.ctypes.data for c in cols], n)
        # ref_records_create fills only the hot fields: overwrite with the full rows
        if n:
            _C.memmove(self.L.ref_records_data(h), b.ctypes.data, n * 64)
        try:
            if self.L.ref_archive_write(h, path.encode()) != 0:
                raise RuntimeError(self.err())
        finally:
            self.L.ref_records_destroy(h)

    def load_archive(self, path: str):
        """FlowStore::load -> (FlowRecord rows as uint8 bytes, error kind or -1)."""
        kind = C.c_int()
        h = self.L.ref_archive_load(path.encode(), C.byref(kind))
        if not h:
            return None, kind.value
        try:
            n = self.L.ref_records_size(h)
            buf = (C.c_uint8 * (n * 64)).from_address(self.L.ref_records_data(h)) if n else b""
            return bytes(buf), -1
        finally:
            self.L.ref_records_destroy(h)

    def ingest_batch(self, buf: np.ndarray, offsets: np.ndarray, out: np.ndarray):
        """The collector's decode loop over n datagrams, timed in C:
        (accepted records written to `out` (64-byte rows), elapsed ms)."""
        b = np.ascontiguousarray(buf, np.uint8)
        o = np.ascontiguousarray(offsets, np.uint64)
        ms = C.c_double()
        k = self.L.ref_ingest_batch(_p(b), _p(o), len(o) - 1, out.ctypes.data, C.byref(ms))
        return k, ms.value

    def encode_packet(self, header: Sequence[int], raw: np.ndarray) -> bytes:
        """encode_packet(ExportHeader{header...}, raw RawFlowRecord rows)."""
        h = np.asarray(header, np.uint32)
        r = np.ascontiguousarray(raw)
        out = np.zeros(24 + 48 * 30, np.uint8)
        n = self.L.ref_encode_packet(h.ctypes.data, r.ctypes.data, len(r) // 48 if r.dtype == np.uint8 else len(r),
                                     out.ctypes.data)
        return out[:n].tobytes()

    # -- catalog ---------------------------------------------------------------
    def catalog(self, sites: Sequence[Sequence[str]] = ()) -> "RefHandle":
        h = RefHandle(self.L, self.L.ref_catalog_create(), "ref_catalog_destroy")
        for i, cidrs in enumerate(sites):
            r = self.register(h, f"site{i}", cidrs)
            if r < 0:
                raise ValueError(f"register failed: {self.err()}")
        return h

    def register(self, cat: "RefHandle", name: str, cidrs: Sequence[str]) -> int:
        return self.L.ref_catalog_register(cat.h, name.encode(), ",".join(cidrs).encode())

    def register_raw(self, cat: "RefHandle", name: str, addrs, lens) -> int:
        a = np.ascontiguousarray(addrs, np.uint32)
        ln = np.ascontiguousarray(lens, np.int32)
        return self.L.ref_catalog_register_raw(cat.h, name.encode(), _p(a), _p(ln), len(a))

    def cidr_parse(self, text: str):
        a, ln = C.c_uint32(), C.c_int32()
        rc = self.L.ref_cidr_parse(text.encode(), C.byref(a), C.byref(ln))
        return None if rc else (a.value, ln.value)

    def lookup(self, cat, ip: int) -> Optional[int]:
        s = self.L.ref_catalog_lookup(cat.h, ip)
        return None if s == NO_SITE else s

    def sequential_lookup(self, cat, ip: int) -> Optional[int]:
        s = self.L.ref_catalog_sequential_lookup(cat.h, ip)
        return None if s == NO_SITE else s

    def entries(self, cat):
        n = self.L.ref_catalog_entry_count(cat.h)
        p = np.zeros(n, np.uint32)
        s = np.zeros(n, np.uint32)
        self.L.ref_catalog_entries(cat.h, _p(p), _p(s), n)
        return p, s

    # -- records ---------------------------------------------------------------
    def records(self, cols) -> "RefHandle":
        c = _cols(cols)
        return RefHandle(self.L, self.L.ref_records_create(*[_p(x) for x in c], len(c[0])),
                         "ref_records_destroy", keep=c)

    def record_columns(self, rec: "RefHandle"):
        n = self.L.ref_records_size(rec.h)
        out = (np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.uint32),
               np.zeros(n, np.uint32), np.zeros(n, np.uint64), np.zeros(n, np.uint64))
        self.L.ref_records_columns(rec.h, *[_p(x) for x in out])
        return out

    def generate(self, sites: list[dict], duration_hours=1, base_wall_ms=1_600_000_000_000,
                 seed=1) -> "RefHandle":
        """toolkit::generate over a ScenarioSpec (toolkit.hpp:48-65)."""
        n = len(sites)
        cidrs = (C.c_char_p * n)(*[s["cidr"].encode() for s in sites])
        hosts = np.array([s.get("hosts", 1) for s in sites], np.uint32)
        logn = np.array([1 if "mu" in s else 0 for s in sites], np.int32)
        fixed = np.array([s.get("fixed_bps", 1e6) for s in sites], np.float64)
        mu = np.array([s.get("mu", 0.0) for s in sites], np.float64)
        sigma = np.array([s.get("sigma", 1.0) for s in sites], np.float64)
        fph = np.array([s.get("flows_per_hour", 1000) for s in sites], np.uint32)
        ack = np.array([s.get("ack", 0.0) for s in sites], np.float64)
        adm = np.array([s.get("admin", 0.0) for s in sites], np.float64)
        h = self.L.ref_generate(duration_hours, base_wall_ms, seed, n, C.cast(cidrs, C.c_void_p),
                                *[_p(x) for x in (hosts, logn, fixed, mu, sigma, fph, ack, adm)])
        if not h:
            raise ValueError(self.err())
        return RefHandle(self.L, h, "ref_records_destroy")

    # -- analysis ----------------------------------------------------------------
    def aggregate(self, rec, cat, params=DEFAULT_PARAMS, workers=1, sequential=False,
                  ws=0, we=0) -> "RefHandle":
        ms = C.c_double()
        h = self.L.ref_aggregate(rec.h, cat.h, *params, workers, 1 if sequential else 0, ws, we,
                                 C.byref(ms))
        r = RefHandle(self.L, h, "ref_result_destroy")
        r.elapsed_ms = ms.value
        return r

    def aggregate_partitioned(self, rec, cat, boundaries, params=DEFAULT_PARAMS) -> "RefHandle":
        b = np.ascontiguousarray(boundaries, np.uint64)
        return RefHandle(self.L, self.L.ref_aggregate_partitioned(rec.h, cat.h, *params, _p(b), len(b)),
                         "ref_result_destroy")

    def time_range(self, rec, cat, begin: int, end: int, workers: int) -> float:
        return self.L.ref_aggregate_time_range(rec.h, begin, end, cat.h, workers)

    def equal(self, a, b) -> bool:
        return bool(self.L.ref_result_equal(a.h, b.h))

    def result(self, res, hist: bool = True, hosts: bool = False) -> dict:
        """AnalysisResult -> {"tallies": [f, ack, admin, unm], "sites": {id: {...}}}."""
        t = np.zeros(4, np.uint64)
        self.L.ref_result_tallies(res.h, _p(t))
        n = self.L.ref_result_site_ids(res.h, None, 0)
        ids = np.zeros(n, np.uint32)
        self.L.ref_result_site_ids(res.h, _p(ids), n)
        sites = {}
        for s in ids.tolist():
            cnt, st, sb, nh = C.c_uint64(), np.zeros(4), C.c_double(), C.c_uint64()
            b = np.zeros(BUCKETS, np.uint32) if hist else None
            self.L.ref_result_site(res.h, s, C.byref(cnt), _p(st), C.byref(sb),
                                   None if b is None else b.ctypes.data, C.byref(nh))
            d = {"count": cnt.value, "min": st[0], "max": st[1], "avg": st[2], "median": st[3],
                 "sum_bps": sb.value, "hist": b, "n_hosts": nh.value}
            if hosts:
                ips = np.zeros(nh.value, np.uint32)
                self.L.ref_result_hosts(res.h, s, _p(ips), nh.value)
                hd = {}
                for ip in ips.tolist():
                    hb = np.zeros(BUCKETS, np.uint32) if hist else None
                    hc, hst, hsb = C.c_uint64(), np.zeros(4), C.c_double()
                    self.L.ref_result_host(res.h, s, ip, C.byref(hc), _p(hst), C.byref(hsb),
                                           None if hb is None else hb.ctypes.data)
                    hd[ip] = {"count": hc.value, "min": hst[0], "max": hst[1], "avg": hst[2],
                              "median": hst[3], "sum_bps": hsb.value, "hist": hb}
                d["hosts"] = hd
            sites[s] = d
        return {"tallies": t, "sites": sites}

    def site_sums(self, rec, cat, n_sites: int, params=DEFAULT_PARAMS):
        lo = np.zeros(n_sites, np.uint64)
        hi = np.zeros(n_sites, np.uint64)
        octs = np.zeros(n_sites, np.uint64)
        self.L.ref_site_sums(rec.h, cat.h, *params, n_sites, _p(lo), _p(hi), _p(octs))
        return lo, hi, octs

    # -- scalar functions --------------------------------------------------------
    def classify(self, src, dst, pkts, octets, start, end, cat, params=DEFAULT_PARAMS, seq=False):
        return self.L.ref_classify(src, dst, pkts, octets, start, end, *params, cat.h, 1 if seq else 0)

    def flow_rate(self, octets: int, start: int, end: int):
        """(rate, ubps) or None when RateError::ZeroDuration was thrown."""
        r, lo, hi = C.c_double(), C.c_uint64(), C.c_uint64()
        if self.L.ref_flow_rate(octets, start, end, C.byref(r), C.byref(lo), C.byref(hi)):
            return None
        return r.value, hi.value << 64 | lo.value

    def bucket_index(self, rate: float) -> int:
        return self.L.ref_bucket_index(rate)

    def attribute(self, src: int, dst: int, cat, seq=False):
        host = C.c_uint32()
        s = self.L.ref_attribute(src, dst, cat.h, 1 if seq else 0, C.byref(host))
        return None if s == NO_SITE else (s, host.value)

    def hist(self) -> "RefHandle":
        return RefHandle(self.L, self.L.ref_hist_create(), "ref_hist_destroy")

    def hist_add(self, h, rate: float, ubps: int) -> None:
        self.L.ref_hist_add(h.h, rate, ubps & (2**64 - 1), ubps >> 64)

    def hist_median(self, h) -> Optional[float]:
        out = C.c_double()
        return None if self.L.ref_hist_median(h.h, C.byref(out)) else out.value

    # -- monitor -------------------------------------------------------------------
    def wstate(self) -> "RefHandle":
        return RefHandle(self.L, self.L.ref_wstate_create(), "ref_wstate_destroy")

    def streak(self, ws, site: int) -> int:
        return self.L.ref_wstate_streak(ws.h, site)

    def evaluate_warnings(self, res, cat, ws, threshold=1e6):
        cap = 1 << 16
        sites = np.zeros(cap, np.uint32)
        hours = np.zeros(cap, np.uint32)
        meds = np.zeros(cap)
        n = self.L.ref_evaluate_warnings(res.h, cat.h, ws.h, threshold, _p(sites), _p(hours),
                                         _p(meds), cap)
        return [(int(sites[i]), int(hours[i]), float(meds[i])) for i in range(min(n, cap))]


class RefHandle:
    def __init__(self, L, h, dtor: str, keep=None):
        self.L, self.h, self.dtor, self.keep = L, h, dtor, keep

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.L, self.dtor)(self.h)
            self.h = None
