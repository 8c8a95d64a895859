"""The site registry behind the C-ABI (host side, no GPU) against the
reference: catalog_test.cpp known answers and the golden catalog fixture
(random /16../26 registrations, overlaps, invalid CIDRs, boundary probes)."""
import numpy as np
import pytest

import golden_io as G
from paper_1108_1785_b200 import CatalogError, Cidr, SiteCatalog, parse_ipv4


def test_slash22_expands_to_four_entries():
    c = SiteCatalog()
    c.register_site("SiteA", ["192.168.4.0/22"])
    assert c.entry_count() == 4
    for third in (4, 5, 6, 7):
        assert c.lookup(192 << 24 | 168 << 16 | third << 8 | 1) is not None
    assert c.lookup(192 << 24 | 168 << 16 | 3 << 8 | 1) is None
    assert c.lookup(192 << 24 | 168 << 16 | 8 << 8 | 1) is None


def test_longer_prefixes_round_up():
    c = SiteCatalog()
    c.register_site("SiteC", ["10.1.2.128/26"])
    assert c.entry_count() == 1
    assert c.lookup(parse_ipv4("10.1.2.1")) is not None
    assert c.lookup(parse_ipv4("10.1.2.200")) is not None


def test_expansion_law():
    for k in range(16, 25):
        c = SiteCatalog()
        c.register_site("s", [f"10.32.0.0/{k}"])
        assert c.entry_count() == 1 << (24 - k)
        expected = parse_ipv4("10.32.0.0")
        for prefix, site in c.entries():
            assert prefix == expected and site == 0
            expected += 256


def test_overlap_is_an_error_and_leaves_catalog_unchanged():
    c = SiteCatalog()
    c.register_site("A", ["10.0.0.0/23"])
    with pytest.raises(CatalogError) as e:
        c.register_site("B", ["10.0.1.0/24"])
    assert e.value.kind == "Overlap"
    assert "already belongs to site 'A'" in str(e.value)
    assert c.site_count() == 1 and c.entry_count() == 2
    with pytest.raises(CatalogError) as e:
        c.register_site("C", ["10.5.0.0/24", "10.5.0.0/25"])  # duplicate within one call
    assert e.value.kind == "Overlap"
    assert c.site_count() == 1


@pytest.mark.parametrize("bad", ["10.0.0.0", "10.0.0/24", "10.0.0.256/24", "10.0.0.0/33",
                                 "10.0.0.0/0", "banana", "10.0.0.0/2x", "1.2.3.4/", "1.2.3.04444/8",
                                 " 1.2.3.4/8"])
def test_invalid_cidrs(bad):
    with pytest.raises(CatalogError) as e:
        Cidr.parse(bad)
    assert e.value.kind == "InvalidCidr"


def test_empty_catalog_resolves_nothing():
    c = SiteCatalog()
    rng = np.random.default_rng(1)
    for ip in rng.integers(0, 2**32, 100).tolist():
        assert c.lookup(ip) is None and c.sequential_lookup(ip) is None


def test_golden_catalog_fixture():
    z = G.load("catalog")
    c = SiteCatalog()
    for text, outcome in zip(z["regs"].tolist(), z["outcomes"].tolist()):
        if outcome >= 0:
            assert c.register_site(f"s{outcome}", [text]) == outcome
        else:
            with pytest.raises(CatalogError) as e:
                c.register_site("x", [text])
            assert e.value.kind == ("Overlap" if outcome == -1 else "InvalidCidr")
    p, s = c.entries_arrays()
    np.testing.assert_array_equal(p, z["entry_prefix"])
    np.testing.assert_array_equal(s, z["entry_site"])
    look = np.array([c.lookup(int(ip)) if c.lookup(int(ip)) is not None else 0xFFFFFFFF
                     for ip in z["ips"]], np.uint32)
    np.testing.assert_array_equal(look, z["lookup"])


def test_hash_and_sequential_agree_everywhere():
    """catalog_test.cpp:93-121 on this registry."""
    c = SiteCatalog()
    rng = np.random.default_rng(2)
    for i in range(50):
        ln = int(rng.integers(20, 27))
        base = int(rng.integers(0, 2**32)) & 0xFFFFFF00
        try:
            c.register_site(f"s{i}", [(base, ln)])
        except CatalogError:
            pass
    assert c.entry_count() > 0
    for ip in rng.integers(0, 2**32, 20000).tolist():
        assert c.lookup(ip) == c.sequential_lookup(ip)
    for i in range(c.site_count()):
        for cd in c.site_cidrs(i):
            for ip in (cd.first_prefix24(), cd.first_prefix24() + 255, cd.last_prefix24(),
                       cd.last_prefix24() + 255, cd.first_prefix24() - 1, cd.last_prefix24() + 256):
                ip &= 0xFFFFFFFF
                assert c.lookup(ip) == c.sequential_lookup(ip)


def test_load_save_round_trip():
    """SiteCatalog::load/save (site_catalog.cpp:150-203) and rebuild idempotence."""
    text = "one 10.1.0.0/22,10.9.0.0/24  # comment\n\n# only a comment\ntwo 172.20.5.0/24\n"
    a = SiteCatalog.load(text)
    b = SiteCatalog.load(a.save())
    assert a.entries() == b.entries()
    assert [a.site(i) for i in range(a.site_count())] == ["one", "two"]
    rng = np.random.default_rng(3)
    for ip in rng.integers(0, 2**32, 2000).tolist() + [parse_ipv4("10.1.3.7"), parse_ipv4("172.20.5.1")]:
        assert a.lookup(ip) == b.lookup(ip)


def test_version_bumps_on_registration_only():
    c = SiteCatalog()
    v0 = c.version()
    c.register_site("a", ["10.0.0.0/24"])
    v1 = c.version()
    with pytest.raises(CatalogError):
        c.register_site("b", ["10.0.0.0/24"])
    assert v1 == v0 + 1 and c.version() == v1
