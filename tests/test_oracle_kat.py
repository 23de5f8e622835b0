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


# ---- SPEC.md:147 fp64 formula: the oracle's fp64 mode pinned to the reference walk ----
def _tie_terrain():
    zq = (O.generate_fractal(80, 80, 0.6, 31, 0, 600) // 50 * 50).astype(np.int16)
    zq[30:40, :] = 100
    return zq


def test_fp64_los_pinned_on_tie_heavy_terrain(kat):
    """Golden fp64 decisions of the REFERENCE walk_crossings (oracle/ref_shim.cpp)
    on a terrain built to produce grazing ties: the oracle's fp64 is_visible and
    estimate_vix match bit for bit; the exact predicate differs only at ties."""
    zq = _tie_terrain()
    g = kat["los_fp64_ties"]
    pairs = np.array(g["pairs"], np.int32).reshape(-1, 4)
    f = O.is_visible_batch(zq, pairs, g["ht"], g["hr"])
    assert np.array_equal(f, np.array(g["visible"], np.uint8))
    e = O.is_visible_batch(zq, pairs, g["ht"], g["hr"], arith="exact")
    diff = np.nonzero(f != e)[0]
    assert len(diff) > 0                                      # the fixture exercises ties
    for i in diff:
        a, b, c, d = (int(x) for x in pairs[i])
        assert e[i] == 1 and O.los_class(zq, a, b, 0, c, d, 0) == 0
    v = kat["vix_fp64_ties"]
    s = O.estimate_vix(zq, v["roi"], v["ht"], v["hr"], v["samples"], v["seed"])
    assert np.array_equal(s.ravel(), np.array(v["scores"], np.uint8))


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (no /root/reference here)")
def test_fp64_vix_live_against_reference_walk():
    """Fresh terrains, live: oracle fp64 estimate_vix == SPEC.md:147 on the
    compiled reference walk_crossings (ref_estimate_vix_fp64)."""
    R = O.ref()
    for seed, (n, rough, roi, h, S) in enumerate([(120, 0.5, 30, 10, 10), (90, 0.6, 45, 20, 20), (100, 0.3, 12, 0, 8)]):
        z = O.generate_fractal(n, n, rough, 500 + seed, 0, 4000)
        if seed == 2:
            z = (z // 100 * 100).astype(np.int16)
        ref = np.zeros((n, n), np.uint8)
        R.ref_estimate_vix_fp64(O._p(z), n, n, roi, h, h, S, 77 + seed, 0, O._p(ref), 0, n)
        assert np.array_equal(O.estimate_vix(z, roi, h, h, S, 77 + seed), ref), seed


def test_viewshed_fp64_differs_from_exact_only_at_ties():
    """The fp64 R2 formula (oracle compute_viewshed_fp64) and the exact one agree
    on every cell whose tangent is not EXACTLY its horizon."""
    z = O.generate_fractal(300, 300, 0.5, 2006, 0, 4000)
    rng = np.random.default_rng(3)
    rows, cols = rng.integers(0, 300, 60).astype(np.int32), rng.integers(0, 300, 60).astype(np.int32)
    for roi, h in ((40, 10), (100, 10), (60, 50)):
        wf, vf = O.viewsheds(z, roi, h, h, rows, cols)
        nties = nflip = 0
        for i in range(len(rows)):
            ve, vt = O.viewshed_ties(z, roi, h, h, int(rows[i]), int(cols[i]))
            x = ve ^ vf[i]
            assert not (x & ~vt).any(), (roi, i)              # differences only at tie cells
            nties += int(np.unpackbits(vt.view(np.uint8)).sum())
            nflip += int(np.unpackbits(x.view(np.uint8)).sum())
        assert nflip <= nties
        print(f"roi {roi}: {nties} tie cells, {nflip} decided differently by fp64")


@pytest.mark.parametrize("roi,h,rough,zmax", [(100, 10, 0.5, 4000), (200, 20, 0.6, 3000), (250, 50, 0.5, 4000)])
def test_viewshed_fp64_vs_d4_euclid_within_tolerance(roi, h, rough, zmax):
    """SURVEY Appendix A D4 verbatim takes a cell's own Euclidean run
    sqrt(a^2 + b^2); the engine's fp64 formula runs a cell along its owner ray
    (D5, dot / |(p,q)|), which equals the exact predicate away from ties.  The
    bits the choice moves are counted at the BASELINE ROIs / heights on
    interior observers: <= 1e-5 of window bits (north_star tolerance)."""
    z = O.generate_fractal(900, 900, rough, 2006 + roi, 0, zmax)
    rng = np.random.default_rng(roi)
    rows = rng.integers(roi, 900 - roi, 150).astype(np.int32)
    cols = rng.integers(roi, 900 - roi, 150).astype(np.int32)
    wf, vf = O.viewsheds(z, roi, h, h, rows, cols)
    _, vd = O.viewsheds(z, roi, h, h, rows, cols, arith="fp64-euclid")
    area = int((wf[:, 2] * wf[:, 3]).sum())
    d4 = int(np.unpackbits((vf ^ vd).view(np.uint8)).sum())
    print(f"roi {roi}: D4-euclid moves {d4} of {area} bits ({d4 / area:.2e})")
    assert d4 <= 1e-5 * area
