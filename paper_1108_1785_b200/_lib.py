"""ctypes binding of the C-ABI in include/gnetmon.h (libgnetmon.so).

The shared library is built in-tree by ``make`` / ``__graft_entry__.build()``
into ``paper_1108_1785_b200/lib/``. There is no fallback: if the library is
missing, importing this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
# GNM_LIB: measurement builds only (tools/ablation.sh); the product and the
# tests load the in-tree library.
LIB_PATH = os.environ.get("GNM_LIB") or os.path.join(LIB_DIR, "libgnetmon.so")

BUCKET_COUNT = 10001
NO_SITE = 0xFFFFFFFF
FLOW_RECORD_BYTES = 64

# status codes (gnm_status)
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_OVERLAP = 2
ERR_INVALID_CIDR = 3
ERR_CUDA = 4
ERR_OUT_OF_MEMORY = 5
ERR_ZERO_DURATION = 6
ERR_EMPTY_HISTOGRAM = 7
ERR_NO_DEVICE = 8
ERR_CAPACITY = 9
ERR_BAD_MAGIC = 10
ERR_BAD_VERSION = 11
ERR_TRUNCATED = 12
ERR_COMM = 13

COMM_ID_BYTES = 128
GROUP_NCCL = 0
GROUP_LOOPBACK = 1

HOT_OFF = 0
HOT_AUTO = 1
HOT_FORCE = 2

MEM_HOST = 0
MEM_DEVICE = 1


class gnm_filter_params(C.Structure):
    _fields_ = [("ack_avg_size_max", C.c_uint32), ("min_packets", C.c_uint32),
                ("min_duration_ms", C.c_uint32), ("workers", C.c_uint32)]


class gnm_cidr(C.Structure):
    _fields_ = [("addr", C.c_uint32), ("prefix_len", C.c_int32)]


class gnm_batch_soa(C.Structure):
    _fields_ = [("src_addr", C.c_void_p), ("dst_addr", C.c_void_p), ("d_pkts", C.c_void_p),
                ("d_octets", C.c_void_p), ("start_ms", C.c_void_p), ("end_ms", C.c_void_p),
                ("n", C.c_uint64), ("mem", C.c_int32)]


class gnm_batch_aos(C.Structure):
    _fields_ = [("records", C.c_void_p), ("n", C.c_uint64), ("mem", C.c_int32)]


class gnm_tallies(C.Structure):
    _fields_ = [("forward", C.c_uint64), ("pure_ack", C.c_uint64),
                ("administrative", C.c_uint64), ("unmatched", C.c_uint64)]


class gnm_result(C.Structure):
    _fields_ = [("window_start_ms", C.c_uint64), ("window_end_ms", C.c_uint64),
                ("threshold_bps", C.c_double), ("sites_capacity", C.c_uint32),
                ("sites", C.c_void_p), ("histograms", C.c_void_p), ("n_sites", C.c_uint32),
                ("tallies", gnm_tallies)]


class gnm_partials(C.Structure):
    _fields_ = [("sums", C.c_void_p), ("min_bps", C.c_void_p), ("max_bps", C.c_void_p),
                ("coarse", C.c_void_p), ("fine", C.c_void_p), ("n_sites", C.c_uint64),
                ("sums_count", C.c_uint64), ("coarse_count", C.c_uint64),
                ("fine_count", C.c_uint64)]


class gnm_host_partials(C.Structure):
    _fields_ = [("sums", C.c_void_p), ("min", C.c_void_p), ("max", C.c_void_p), ("coarse", C.c_void_p),
                ("fine", C.c_void_p), ("n", C.c_uint64)]


class gnm_netflow_stats(C.Structure):
    _fields_ = [("datagrams", C.c_uint64), ("decode_errors", C.c_uint64),
                ("records_rejected", C.c_uint64), ("records_accepted", C.c_uint64)]


class gnm_timing(C.Structure):
    _fields_ = [("accumulate_ms", C.c_double), ("finalize_ms", C.c_double),
                ("h2d_ms", C.c_double), ("k2_launches", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("records", C.c_uint64),
                ("plan_ms", C.c_double), ("total_plan_ms", C.c_double),
                ("total_accumulate_ms", C.c_double), ("total_finalize_ms", C.c_double),
                ("total_finalizes", C.c_uint64), ("total_k2_launches", C.c_uint64),
                ("h2d_bytes", C.c_uint64)]


class gnm_warning(C.Structure):
    _fields_ = [("site", C.c_uint32), ("consecutive_bad_hours", C.c_uint32),
                ("median_bps", C.c_double)]


# gnm_site_stats as a numpy structured dtype (72 bytes, C layout).
SITE_STATS_DTYPE = np.dtype([
    ("flow_count", "<u8"), ("octets", "<u8"), ("rate_ubps_lo", "<u8"), ("rate_ubps_hi", "<u8"),
    ("min_bps", "<f8"), ("max_bps", "<f8"), ("avg_bps", "<f8"), ("median_bps", "<f8"),
    ("below_threshold", "<u4"), ("reserved", "<u4"),
])
assert SITE_STATS_DTYPE.itemsize == 72

# gnm_host_stats (64 bytes, C layout).
HOST_STATS_DTYPE = np.dtype([
    ("site", "<u4"), ("host", "<u4"), ("flow_count", "<u8"), ("rate_ubps_lo", "<u8"),
    ("rate_ubps_hi", "<u8"), ("min_bps", "<f8"), ("max_bps", "<f8"), ("avg_bps", "<f8"),
    ("median_bps", "<f8"),
])
assert HOST_STATS_DTYPE.itemsize == 64

# The 64-byte flowmon::FlowRecord (netflow.hpp:32-67).
FLOW_RECORD_DTYPE = np.dtype({
    "names": ["src_addr", "dst_addr", "next_hop", "input_if", "output_if", "d_pkts", "d_octets",
              "first", "last", "src_port", "dst_port", "pad1", "tcp_flags", "protocol", "tos",
              "src_as", "dst_as", "src_mask", "dst_mask", "pad2", "start_ms", "end_ms"],
    "formats": ["<u4", "<u4", "<u4", "<u2", "<u2", "<u4", "<u4", "<u4", "<u4", "<u2", "<u2",
                "u1", "u1", "u1", "u1", "<u2", "<u2", "u1", "u1", "<u2", "<u8", "<u8"],
    "offsets": [0, 4, 8, 12, 14, 16, 20, 24, 28, 32, 34, 36, 37, 38, 39, 40, 42, 44, 45, 46, 48, 56],
    "itemsize": 64,
})

# Every symbol include/gnetmon.h declares: (name, restype, argtypes).
_P = C.c_void_p
_SIGS = [
    ("gnm_last_error", C.c_char_p, []),
    ("gnm_abi_version", C.c_int, []),
    ("gnm_filter_params_default", None, [C.POINTER(gnm_filter_params)]),
    ("gnm_cidr_parse", C.c_int, [C.c_char_p, C.POINTER(gnm_cidr)]),
    ("gnm_ipv4_parse", C.c_int, [C.c_char_p, C.POINTER(C.c_uint32)]),
    ("gnm_registry_create", C.c_int, [C.POINTER(_P)]),
    ("gnm_registry_destroy", None, [_P]),
    ("gnm_registry_register_site", C.c_int,
     [_P, C.c_char_p, C.POINTER(gnm_cidr), C.c_size_t, C.POINTER(C.c_uint32)]),
    ("gnm_registry_lookup", C.c_uint32, [_P, C.c_uint32]),
    ("gnm_registry_sequential_lookup", C.c_uint32, [_P, C.c_uint32]),
    ("gnm_registry_site_count", C.c_size_t, [_P]),
    ("gnm_registry_entry_count", C.c_size_t, [_P]),
    ("gnm_registry_entries", C.c_size_t, [_P, _P, _P, C.c_size_t]),
    ("gnm_registry_site_name", C.c_char_p, [_P, C.c_uint32]),
    ("gnm_registry_version", C.c_uint64, [_P]),
    ("gnm_ctx_create", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("gnm_ctx_destroy", None, [_P]),
    ("gnm_ctx_set_stream", C.c_int, [_P, _P]),
    ("gnm_ctx_stream", _P, [_P]),
    ("gnm_ctx_set_chunk_records", C.c_int, [_P, C.c_uint64]),
    ("gnm_ctx_set_hot_mode", C.c_int, [_P, C.c_int]),
    ("gnm_ctx_set_hosts", C.c_int, [_P, C.c_int]),
    ("gnm_ctx_set_graphs", C.c_int, [_P, C.c_int]),
    ("gnm_host_count", C.c_uint64, [_P]),
    ("gnm_host_results", C.c_int, [_P, _P, C.c_uint64, _P]),
    ("gnm_host_histogram_entries", C.c_int, [_P, _P, _P, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    ("gnm_hosts_local_keys", C.c_int, [_P, _P, C.POINTER(_P), C.POINTER(C.c_uint64)]),
    ("gnm_hosts_set_keys", C.c_int, [_P, _P, C.c_uint64, C.POINTER(gnm_host_partials)]),
    ("gnm_hosts_prepare_median", C.c_int, [_P]),
    ("gnm_analyze", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa), C.POINTER(gnm_result)]),
    ("gnm_analyze_aos", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_aos), C.POINTER(gnm_result)]),
    ("gnm_accumulate", C.c_int, [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa)]),
    ("gnm_accumulate_window", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa), C.c_uint64, C.c_uint64]),
    ("gnm_accumulate_window_aos", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_aos), C.c_uint64, C.c_uint64]),
    ("gnm_analyze_window", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa), C.POINTER(gnm_result)]),
    ("gnm_accumulate_aos", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_aos)]),
    ("gnm_finalize", C.c_int, [_P, _P, C.POINTER(gnm_result)]),
    ("gnm_reset", C.c_int, [_P]),
    ("gnm_get_partials", C.c_int, [_P, _P, C.POINTER(gnm_partials)]),
    ("gnm_prepare_median", C.c_int, [_P, _P]),
    ("gnm_decode_archive", C.c_int, [_P, _P, C.c_uint64, C.c_int32, _P, C.c_uint64, C.c_int32, _P]),
    ("gnm_accumulate_archive", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), _P, C.c_uint64, C.c_int32]),
    ("gnm_analyze_archive", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), _P, C.c_uint64, C.c_int32, C.POINTER(gnm_result)]),
    ("gnm_decode_netflow", C.c_int,
     [_P, _P, C.c_uint64, _P, C.c_uint64, C.c_int32, _P, C.c_uint64, C.c_int32, _P,
      C.POINTER(gnm_netflow_stats)]),
    ("gnm_classify", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa), _P, C.c_int32]),
    ("gnm_ctx_timing", C.c_int, [_P, C.POINTER(gnm_timing)]),
    ("gnm_ctx_enable_timing", C.c_int, [_P, C.c_int]),
    ("gnm_warning_state_create", C.c_int, [C.POINTER(_P)]),
    ("gnm_warning_state_destroy", None, [_P]),
    ("gnm_warning_state_streak", C.c_uint32, [_P, C.c_uint32]),
    ("gnm_evaluate_warnings", C.c_int,
     [C.POINTER(gnm_result), _P, C.c_double, C.POINTER(gnm_warning), C.c_size_t,
      C.POINTER(C.c_size_t)]),
    ("gnm_comm_unique_id", C.c_int, [_P]),
    ("gnm_ctx_comm_init", C.c_int, [_P, C.c_int, C.c_int, _P]),
    ("gnm_ctx_comm_destroy", C.c_int, [_P]),
    ("gnm_ctx_comm_size", C.c_int, [_P]),
    ("gnm_group_create", C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(_P)]),
    ("gnm_group_destroy", None, [_P]),
    ("gnm_group_size", C.c_int, [_P]),
    ("gnm_group_ctx", _P, [_P, C.c_int]),
    ("gnm_group_analyze", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_soa), C.POINTER(gnm_result)]),
    ("gnm_group_analyze_aos", C.c_int,
     [_P, _P, C.POINTER(gnm_filter_params), C.POINTER(gnm_batch_aos), C.POINTER(gnm_result)]),
    ("gnm_group_host_count", C.c_uint64, [_P]),
    ("gnm_group_host_results", C.c_int, [_P, _P, C.c_uint64]),
    ("gnm_group_host_histogram_entries", C.c_int, [_P, _P, _P, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
]
SYMBOLS = [s[0] for s in _SIGS]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(). "
            "There is no CPU fallback for the analysis path.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.gnm_last_error()
    return msg.decode() if msg else ""
