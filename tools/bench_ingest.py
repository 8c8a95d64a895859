"""Throughput of the §8(f) rows around the hot path, on one GPU, with the
unmodified reference's CPU loop timed beside each (one JSON line per row):

  netflow_decode   gnm_decode_netflow, datagrams resident in HBM -> FlowRecord
                   rows in HBM (N1 validate, N2 scan, N3 decode)
  archive_decode   gnm_decode_archive, FLOWARC1 bytes in HBM -> FlowRecord rows
  archive_analyze  gnm_analyze_archive: K2 reads the archive entries in place
                   (aggregate(FlowStore::load(...)) without the decode pass)

    python tools/bench_ingest.py [--records N] [--reps R]

Inputs are larger than L2 (no flush needed). Times are CUDA events on the
engine stream around whole public calls (each call synchronises once).
The CPU arms: the reference's decode_packet + reject rule + resolve_times
loop over the same datagrams (oracle/_ref, ref_ingest_batch) and
FlowStore::load of the same archive written to /tmp by the reference.
"""
import argparse
import ctypes as C
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RAW_BE = np.dtype([("src_addr", ">u4"), ("dst_addr", ">u4"), ("next_hop", ">u4"), ("input_if", ">u2"),
                   ("output_if", ">u2"), ("d_pkts", ">u4"), ("d_octets", ">u4"), ("first", ">u4"),
                   ("last", ">u4"), ("src_port", ">u2"), ("dst_port", ">u2"), ("pad1", "u1"),
                   ("tcp_flags", "u1"), ("protocol", "u1"), ("tos", "u1"), ("src_as", ">u2"),
                   ("dst_as", ">u2"), ("src_mask", "u1"), ("dst_mask", "u1"), ("pad2", ">u2")])
HDR_BE = np.dtype([("version", ">u2"), ("count", ">u2"), ("sys_uptime", ">u4"), ("unix_secs", ">u4"),
                   ("unix_nsecs", ">u4"), ("flow_sequence", ">u4"), ("engine_type", "u1"),
                   ("engine_id", "u1"), ("sampling_interval", ">u2")])
ENTRY_BE = np.dtype([("start_ms", ">u8"), ("end_ms", ">u8"), ("raw", RAW_BE)])
assert RAW_BE.itemsize == 48 and HDR_BE.itemsize == 24 and ENTRY_BE.itemsize == 64


def make_datagrams(cols, per=30):
    """NetFlow v5 export datagrams (30 records each) carrying the D3 records."""
    src, dst, pkts, octs, start, end = cols
    n = len(src) // per * per
    g = n // per
    dg = np.zeros(g, np.dtype([("h", HDR_BE), ("r", RAW_BE, (per,))]))
    wall = 1_700_000_000_000
    dg["h"]["version"] = 5
    dg["h"]["count"] = per
    dg["h"]["sys_uptime"] = 4_000_000_000
    dg["h"]["unix_secs"] = wall // 1000
    r = dg["r"]  # (g, per) view; a reshape would copy
    r["src_addr"], r["dst_addr"] = src[:n].reshape(g, per), dst[:n].reshape(g, per)
    r["d_pkts"], r["d_octets"] = pkts[:n].reshape(g, per), octs[:n].reshape(g, per)
    # uptime-relative first/last so resolve_times gives end - start = duration
    dur = (end[:n] - start[:n]).astype(np.uint64) % np.uint64(3_000_000_000)
    last = np.uint64(4_000_000_000) - (np.arange(n, dtype=np.uint64) % np.uint64(1000))
    r["last"] = last.reshape(g, per)
    r["first"] = (last - dur).reshape(g, per)
    buf = dg.view(np.uint8).reshape(-1)
    offs = np.arange(g + 1, dtype=np.uint64) * np.uint64(HDR_BE.itemsize + per * RAW_BE.itemsize)
    return buf, offs, n


def make_archive(cols):
    src, dst, pkts, octs, start, end = cols
    e = np.zeros(len(src), ENTRY_BE)
    e["start_ms"], e["end_ms"] = start, end
    e["raw"]["src_addr"], e["raw"]["dst_addr"] = src, dst
    e["raw"]["d_pkts"], e["raw"]["d_octets"] = pkts, octs
    head = np.frombuffer(b"FLOWARC1" + (1).to_bytes(4, "big") + len(src).to_bytes(8, "big"), np.uint8)
    return np.concatenate([head, e.view(np.uint8).reshape(-1)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=30_000_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cpu-records", type=int, default=3_000_000)
    args = ap.parse_args()

    import torch
    from paper_1108_1785_b200 import Engine, SiteCatalog, synth, _lib
    from paper_1108_1785_b200._lib import lib, gnm_netflow_stats
    from paper_1108_1785_b200.flowmon import _check

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs") or peaks.get("hbm_GBps") or 6446.3)
    w = synth.workload("D3")
    cols = synth.generate(w, args.records)
    cat = SiteCatalog()
    w.sites.register(cat)
    eng = Engine(0)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    try:
        from oracle import Reference
        ref = Reference()
    except ImportError:
        ref = None

    # ---- NetFlow v5 decode -----------------------------------------------------
    buf, offs, n = make_datagrams(cols)
    d_buf = torch.from_numpy(buf).cuda()
    d_off = torch.from_numpy(offs.view(np.int64)).cuda()
    g = len(offs) - 1
    d_out = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
    status = np.zeros(g, np.uint8)
    st = gnm_netflow_stats()

    def nf():
        _check(lib.gnm_decode_netflow(eng.handle, d_buf.data_ptr(), buf.size, d_off.data_ptr(), g, _lib.MEM_DEVICE,
                                      d_out.data_ptr(), n, _lib.MEM_DEVICE, status.ctypes.data, C.byref(st)))
    ms = timed(nf, args.reps)
    moved = buf.size + st.records_accepted * 64 + g * (8 + 8 + 4 + 1)
    line = {"row": "netflow_decode", "records": n, "datagrams": g, "ms": ms, "records_per_s": n / (ms / 1e3),
            "accepted": st.records_accepted,
            "roofline": {"bound": "hbm", "bytes": moved, "achieved_gbs": moved / (ms / 1e3) / 1e9,
                         "peak_gbs": hbm, "frac": moved / (ms / 1e3) / 1e9 / hbm}}
    if ref is not None:
        k = min(g, args.cpu_records // 30)
        out = np.empty(k * 30 * 64, np.uint8)
        _, cms = ref.ingest_batch(buf[:int(offs[k])], offs[:k + 1], out)
        line["cpu_reference"] = {"records_per_s": k * 30 / (cms / 1e3), "cores": 1,
                                 "sample": f"{k} datagrams, decode_packet + reject + resolve_times loop"}
    print(json.dumps(line), flush=True)
    del d_buf, d_off, d_out

    # ---- FLOWARC1 decode and in-place analysis -----------------------------------
    arc = make_archive(cols)
    d_arc = torch.from_numpy(arc).cuda()
    d_rows = torch.empty(args.records * 64, dtype=torch.uint8, device="cuda")
    nout = C.c_uint64()

    def ad():
        _check(lib.gnm_decode_archive(eng.handle, d_arc.data_ptr(), arc.size, _lib.MEM_DEVICE, d_rows.data_ptr(),
                                      args.records, _lib.MEM_DEVICE, C.byref(nout)))
    ms = timed(ad, args.reps)
    moved = 2 * 64 * args.records
    line = {"row": "archive_decode", "records": args.records, "ms": ms, "records_per_s": args.records / (ms / 1e3),
            "roofline": {"bound": "hbm", "bytes": moved, "achieved_gbs": moved / (ms / 1e3) / 1e9,
                         "peak_gbs": hbm, "frac": moved / (ms / 1e3) / 1e9 / hbm}}
    if ref is not None:
        import time
        k = min(args.records, args.cpu_records)
        path = os.path.join(tempfile.gettempdir(), "gnm_bench.flowarc")
        ref.write_archive(synth.to_aos(tuple(c[:k] for c in cols)), path)
        kind = C.c_int()
        ref.L.ref_records_destroy(ref.L.ref_archive_load(path.encode(), C.byref(kind)))  # warm the page cache
        t0 = time.perf_counter()
        h = ref.L.ref_archive_load(path.encode(), C.byref(kind))
        cms = (time.perf_counter() - t0) * 1e3
        ref.L.ref_records_destroy(h)
        os.remove(path)
        line["cpu_reference"] = {"records_per_s": k / (cms / 1e3), "cores": 1,
                                 "sample": f"FlowStore::load of a {k}-record archive (page-cached file)"}
    print(json.dumps(line), flush=True)
    del d_rows

    res = {}

    def aa():
        res["r"] = eng.aggregate_archive(d_arc, cat)
    ms = timed(aa, args.reps)
    moved = 64 * args.records  # the entry sectors holding start/end/src/dst/pkts/octets
    line = {"row": "archive_analyze", "records": args.records, "ms": ms,
            "records_per_s": args.records / (ms / 1e3),
            "tallies_total": res["r"].tallies.total(),
            "roofline": {"bound": "hbm", "bytes": moved, "achieved_gbs": moved / (ms / 1e3) / 1e9,
                         "peak_gbs": hbm, "frac": moved / (ms / 1e3) / 1e9 / hbm,
                         "note": "whole analysis step (K1+K2+finalize) over 64 B entries"}}
    print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
