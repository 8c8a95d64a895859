"""NetFlow v5 ingest: the test encoder is pinned to the reference's
encode_packet (CPU), and the GPU batch decode (gnm_decode_netflow) equals
the reference's Collector::ingest_datagram path (decode_packet, the reject
rule, resolve_times; collector.cpp:101-129) byte for byte, including every
CodecError kind."""
import numpy as np
import pytest

import netflow_gen as NG
import golden_io as G


def test_encoder_matches_reference_encode_packet(ref):
    rng = np.random.default_rng(3)
    for cnt in (1, 7, 30):
        h = NG.header(rng, cnt)
        raw = NG.random_records(rng, cnt)
        assert NG.encode(h, raw) == ref.encode_packet(NG.header_tuple(h), raw.view(np.uint8))


def test_reference_ingest_kinds(ref):
    """The reference's own verdicts on the corrupted datagrams (sanity of the
    harness): every CodecError kind occurs, and valid datagrams decode."""
    rng = np.random.default_rng(5)
    ds = NG.make_stream(rng, 120)
    kinds = {ref.ingest_datagram(d)[0] for d in ds}
    assert kinds == {0, 1, 2, 3}


def test_golden_netflow_fixture_matches_reference(ref):
    z = G.load("netflow")
    buf, offs = z["datagrams"], z["offsets"]
    for i in range(len(offs) - 1):
        st, rows, rej = ref.ingest_datagram(buf[offs[i]:offs[i + 1]].tobytes())
        assert st == z["status"][i]
    # all rows of the fixture, concatenated
    rows = b"".join(ref.ingest_datagram(buf[offs[i]:offs[i + 1]].tobytes())[1] for i in range(len(offs) - 1))
    assert rows == z["records"].tobytes()


def _expected(ref_or_fixture, datagrams):
    rows, status, rej = [], [], 0
    for d in datagrams:
        st, r, k = ref_or_fixture.ingest_datagram(d)
        rows.append(r)
        status.append(st)
        rej += k
    return b"".join(rows), np.array(status, np.uint8), rej


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_gpu_decode_matches_reference(engine, ref, on_device):
    rng = np.random.default_rng(11)
    ds = NG.make_stream(rng, 2000)
    buf, offs = NG.pack(ds)
    want, want_status, want_rej = _expected(ref, ds)
    if on_device:
        import torch
        recs, status, stats = engine.decode_netflow(torch.from_numpy(buf.copy()).cuda(), offs, out_device=True)
        got = recs.cpu().numpy().tobytes()
    else:
        recs, status, stats = engine.decode_netflow(buf, offs)
        got = recs.tobytes()
    assert got == want
    np.testing.assert_array_equal(status, want_status)
    assert stats["decode_errors"] == int((want_status != 0).sum())
    assert stats["records_rejected"] == want_rej
    assert stats["records_accepted"] == len(want) // 64


@pytest.mark.gpu
def test_gpu_decode_golden_fixture(engine):
    z = G.load("netflow")
    recs, status, stats = engine.decode_netflow(z["datagrams"], z["offsets"])
    assert recs.tobytes() == z["records"].tobytes()
    np.testing.assert_array_equal(status, z["status"])


@pytest.mark.gpu
def test_gpu_decode_unaligned_and_empty(engine, ref):
    """Datagrams at odd byte offsets (a 3-byte prefix) and an empty batch."""
    rng = np.random.default_rng(13)
    ds = NG.make_stream(rng, 300)
    buf, offs = NG.pack(ds)
    buf2 = np.concatenate([np.array([7, 7, 7], np.uint8), buf])
    recs, status, _ = engine.decode_netflow(buf2, offs + np.uint64(3))
    want, want_status, _ = _expected(ref, ds)
    assert recs.tobytes() == want
    np.testing.assert_array_equal(status, want_status)
    recs, status, stats = engine.decode_netflow(np.zeros(0, np.uint8), np.zeros(1, np.uint64))
    assert len(recs) == 0 and stats["datagrams"] == 0


@pytest.mark.gpu
def test_decoded_records_feed_aggregate(engine, orc):
    """Ingest -> analysis end to end: decoded rows analysed on the GPU equal
    the oracle on the same rows."""
    import parity
    from paper_1108_1785_b200 import FlowRecords, SiteCatalog
    rng = np.random.default_rng(17)
    ds = NG.make_stream(rng, 1500, corrupt=False)
    buf, offs = NG.pack(ds)
    recs, _, _ = engine.decode_netflow(buf, offs)
    cat = SiteCatalog()
    cat.register_site("a", ["0.0.0.0/2"])
    cat.register_site("b", ["128.0.0.0/3"])
    cols = tuple(np.ascontiguousarray(recs[c]) for c in ("src_addr", "dst_addr", "d_pkts", "d_octets",
                                                          "start_ms", "end_ms"))
    res = engine.aggregate(FlowRecords(recs.view(np.uint8)), cat, histograms=True)
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))
