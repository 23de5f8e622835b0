"""The oracle's restatement of the shipped reference headers, pinned against
known-answer vectors produced by the reference code itself
(tests/golden/make_golden.py) and SURVEY Appendix B."""
import numpy as np
import pytest

import oracle_lib as O


def test_appendix_b_rng():
    L = O.lib()
    assert [hex(int(x)) for x in O.splitmix(0, 3)] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]
    assert int(O.splitmix(1234567, 1)[0]) == 0x599ED017FB08FC85
    assert L.txo_mix_seed(0, 0, 0) == 0xA706DD2F4D197E6F
    assert L.txo_mix_seed(42, 0, 0) == 0x57E1FABA65107204
    assert L.txo_mix_seed(42, 1, 0) == 0x42B544C0F309A887
    assert L.txo_mix_seed(42, 0, 1) == 0x932F43447F959E57
    s = L.txo_mix_seed(42, 500, 500)
    assert list(O.splitmix(s, 2, 1, 201)) == [185, 95]
    d = O.splitmix(s, 3, 2)[2].view(np.float64)
    assert d == 0.19086892760999641


def test_appendix_b_walk():
    t, r, c, k = O.walk(0, 0, 3, 7, False)
    assert len(t) == 8
    assert t[0] == 1 / 7 and r[0] == 0.42857142857142855 and c[0] == 1 and k[0] == 1
    assert t[2] == 1 / 3 and r[2] == 1 and c[2] == 2.333333333333333 and k[2] == 0
    t, r, c, k = O.walk(0, 0, 2, 4, True)
    assert list(t) == [0.25, 0.5, 0.75, 1.0] and list(k) == [1, 2, 1, 2]
    assert list(r) == [0.5, 1, 1.5, 2] and list(c) == [1, 2, 3, 4]
    assert O.walk_hash(46000, 46000, 45900, 46071, False)[1] == 169
    assert O.chunks(10, 3) == [(0, 4), (4, 7), (7, 10)]


def test_rng_against_reference_vectors(kat):
    for s, vals in kat["splitmix_next"].items():
        assert [str(int(x)) for x in O.splitmix(int(s), len(vals))] == vals
    for key, vals in kat["splitmix_next_below"].items():
        s, n = (int(x) for x in key.split("/"))
        assert [str(int(x)) for x in O.splitmix(s, len(vals), 1, n)] == vals
    for s, vals in kat["splitmix_next_double_bits"].items():
        assert [str(int(x)) for x in O.splitmix(int(s), len(vals), 2)] == vals
    for a, b, c, v in kat["mix_seed"]:
        assert O.lib().txo_mix_seed(int(a), int(b), int(c)) == int(v)


def test_walk_lists_against_reference(kat):
    for e in kat["walk_lists"]:
        t, r, c, k = O.walk(*e["seg"])
        assert t.tolist() == e["t"] and r.tolist() == e["row"] and c.tolist() == e["col"]
        assert k.tolist() == e["kind"]


def test_walk_hashes_against_reference(kat):
    """600 segments with absolute coordinates up to 46400 and spans up to
    2000: the (t,row,col,kind) bit patterns hash identically."""
    for r0, c0, r1, c1, e, h, n in kat["walk_hashes"]:
        assert O.walk_hash(r0, c0, r1, c1, e) == (int(h), n), (r0, c0, r1, c1, e)


def test_chunks_against_reference(kat):
    for n, t, ch in kat["chunks"]:
        assert O.chunks(n, t) == [tuple(x) for x in ch]


def test_live_reference_shim_random_segments():
    """Where the reference headers were compiled (this container), compare the
    restated walk with the real walk_crossings on fresh random segments."""
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built (reference absent on this host)")
    rng = np.random.default_rng(1)
    for _ in range(3000):
        r0, c0 = (int(x) for x in rng.integers(0, 46400, 2))
        dr, dc = (int(x) for x in rng.integers(-300, 301, 2))
        e = int(rng.integers(0, 2))
        assert O.walk_hash(r0, c0, r0 + dr, c0 + dc, e) == O.walk_hash(r0, c0, r0 + dr, c0 + dc, e, R)
