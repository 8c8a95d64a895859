"""Synthetic NetFlow v5 export datagrams for the ingest tests (test helper).

The wire format is the reference's (netflow.cpp:115-143, encode_packet): a
24-byte big-endian header, then 48-byte big-endian records. `encode` is
pinned to the reference's encode_packet in tests/test_netflow.py."""
import numpy as np

HEADER = np.dtype([("version", ">u2"), ("count", ">u2"), ("sys_uptime", ">u4"), ("unix_secs", ">u4"),
                   ("unix_nsecs", ">u4"), ("flow_sequence", ">u4"), ("engine_type", "u1"),
                   ("engine_id", "u1"), ("sampling_interval", ">u2")])
RECORD_BE = np.dtype([("src_addr", ">u4"), ("dst_addr", ">u4"), ("next_hop", ">u4"), ("input_if", ">u2"),
                      ("output_if", ">u2"), ("d_pkts", ">u4"), ("d_octets", ">u4"), ("first", ">u4"),
                      ("last", ">u4"), ("src_port", ">u2"), ("dst_port", ">u2"), ("pad1", "u1"),
                      ("tcp_flags", "u1"), ("protocol", "u1"), ("tos", "u1"), ("src_as", ">u2"),
                      ("dst_as", ">u2"), ("src_mask", "u1"), ("dst_mask", "u1"), ("pad2", ">u2")])
# RawFlowRecord in host memory (netflow.hpp:32-57), same field order.
RECORD_LE = np.dtype([(n, RECORD_BE.fields[n][0].newbyteorder("<")) for n in RECORD_BE.names])
assert HEADER.itemsize == 24 and RECORD_BE.itemsize == 48 and RECORD_LE.itemsize == 48


def random_records(rng, n):
    r = np.zeros(n, RECORD_LE)
    for name in RECORD_LE.names:
        t = RECORD_LE.fields[name][0]
        r[name] = rng.integers(0, np.iinfo(t).max, n, dtype=np.uint64, endpoint=True).astype(t)
    # realistic-ish counters with the collector's reject cases mixed in
    r["d_pkts"] = rng.integers(0, 5000, n)
    r["d_octets"] = r["d_pkts"].astype(np.uint64) * rng.integers(0, 1600, n) + rng.integers(0, 100, n)
    return r


def header(rng, count, version=5):
    h = np.zeros(1, HEADER)
    h["version"], h["count"] = version, count
    h["sys_uptime"] = rng.integers(0, 2**32)
    h["unix_secs"] = rng.integers(1_500_000_000, 1_800_000_000)
    h["unix_nsecs"] = rng.integers(0, 1_000_000_000)
    h["flow_sequence"] = rng.integers(0, 2**32)
    h["engine_type"], h["engine_id"] = rng.integers(0, 256, 2)
    h["sampling_interval"] = rng.integers(0, 2**16)
    return h


def header_tuple(h):
    return [int(h[f][0]) for f in HEADER.names]


def encode(h, raw_le) -> bytes:
    """Header (HEADER row) + records (RECORD_LE rows) -> datagram bytes."""
    return h.tobytes() + raw_le.astype(RECORD_BE).tobytes()


def make_stream(rng, n_packets, corrupt=True):
    """Datagrams (list of bytes): mostly valid, with every CodecError kind
    and reject cases; records' first/last near the header's uptime so
    resolve_times exercises wrap_diff both ways."""
    out = []
    for i in range(n_packets):
        cnt = int(rng.integers(1, 31))
        h = header(rng, cnt)
        raw = random_records(rng, cnt)
        up = int(h["sys_uptime"][0])
        raw["first"] = (up - rng.integers(0, 4_000_000, cnt)) % 2**32
        raw["last"] = (up - rng.integers(-1000, 3_000_000, cnt)) % 2**32
        d = encode(h, raw)
        kind = i % 17 if corrupt else 0
        if kind == 1:    # bad version
            d = np.frombuffer(d, np.uint8).copy(); d[1] = 9; d = d.tobytes()
        elif kind == 2:  # truncated (one byte short)
            d = d[:-1]
        elif kind == 3:  # bad count 0
            d = np.frombuffer(d, np.uint8).copy(); d[2] = d[3] = 0; d = d.tobytes()
        elif kind == 4:  # header only
            d = d[:10]
        elif kind == 5:  # count 31 (and wrong length)
            d = np.frombuffer(d, np.uint8).copy(); d[2], d[3] = 0, 31; d = d.tobytes()
        out.append(d)
    return out


def pack(datagrams):
    offsets = np.zeros(len(datagrams) + 1, np.uint64)
    offsets[1:] = np.cumsum([len(d) for d in datagrams])
    buf = np.frombuffer(b"".join(datagrams), np.uint8) if datagrams else np.zeros(0, np.uint8)
    return buf, offsets
