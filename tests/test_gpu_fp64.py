"""SPEC.md:147 fp64 parity on the GPU (DESIGN.md §2 D2).

The engine's default LOS arithmetic (txs_params.los_arith = fp64) must give
the decisions of SPEC.md:147's fp64 formula bit for bit: the exact integer
walks find every grazing tie (terrain exactly ON the LOS / a cell exactly on
its horizon) and only those are re-decided in fp64 on the device.  The oracle's
fp64 mode is pinned to the reference walk_crossings (tests/test_oracle_kat.py);
where oracle/_ref is present the reference formula is also compared live.
Tie-heavy terrains (elevations quantized to 50, a flat band) make ties common;
the exact mode is checked against the oracle's exact mode on the same inputs."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _T():
    import paper_2006_16783_b200 as T
    return T


def _tie_terrain(n=80, m=80, seed=31, zmax=600):
    z = (O.generate_fractal(n, m, 0.6, seed, 0, zmax) // 50 * 50).astype(np.int16)
    z[3 * n // 8:n // 2, :] = 100
    return z


@pytest.mark.parametrize("arith", ["fp64", "exact"])
def test_los_batch_tie_terrain(engine, kat, arith):
    z = _tie_terrain()
    g = kat["los_fp64_ties"]
    pairs = np.array(g["pairs"], np.int32).reshape(-1, 4)
    engine.set_terrain(z)
    got = engine.is_visible_batch(pairs, g["ht"], g["hr"], los_arith=arith)
    assert np.array_equal(got, O.is_visible_batch(z, pairs, g["ht"], g["hr"], arith=arith))
    if arith == "fp64":
        assert np.array_equal(got, np.array(g["visible"], np.uint8))     # the reference walk's fp64
    e = O.is_visible_batch(z, pairs, g["ht"], g["hr"], arith="exact")
    assert (e != O.is_visible_batch(z, pairs, g["ht"], g["hr"])).sum() > 0   # ties are exercised


@pytest.mark.parametrize("path", ["smem", "pairs", "zt"])
@pytest.mark.parametrize("skip", ["1", "2", "0"])
@pytest.mark.parametrize("arith", ["fp64", "exact"])
def test_vix_tie_terrain_every_path(engine, monkeypatch, path, skip, arith):
    """Every VIX kernel / skip mode on a tie-heavy terrain, both arithmetics."""
    if path != "pairs" and skip != "1":
        pytest.skip("skip modes exist on the quad path only")
    T = _T()
    z = _tie_terrain(300, 280, 7, 800)
    engine.set_terrain(z)
    monkeypatch.setenv("TXS_VIX_PATH", path)
    monkeypatch.setenv("TXS_VIX_SKIP", skip)
    for roi, S, h, group in [(40, 12, 0, "4"), (60, 16, 0, "16"), (160, 10, 0, "4")]:
        monkeypatch.setenv("TXS_VIX_GROUP", group)
        g = engine.estimate_vix(T.make_params(roi, h, h, samples=S, seed=5, los_arith=arith))
        o = O.estimate_vix(z, roi, h, h, S, 5, arith=arith)
        assert np.array_equal(g, o), (roi, int((g != o).sum()))
    if arith == "fp64":
        assert engine.stats()["vix_fp64_ties"] > 0


def test_vix_c1_full_vs_reference_formula(engine, c1_terrain):
    """BASELINE config 1 in full (1000x1000, roi 100, h 10, S 10): 0 differing
    LOS-derived scores against SPEC.md:147's fp64 (the oracle's fp64 mode, and
    the compiled reference walk where oracle/_ref exists)."""
    T = _T()
    z = c1_terrain
    engine.set_terrain(z)
    g = engine.estimate_vix(T.make_params(100, 10, 10, samples=10, seed=1))
    o = O.estimate_vix(z, 100, 10, 10, 10, 1)
    assert np.array_equal(g, o), int((g != o).sum())
    st = engine.stats()
    e = O.estimate_vix(z, 100, 10, 10, 10, 1, arith="exact")
    print(f"c1: fp64 ties re-tested {st['vix_fp64_ties']}, flipped {st['vix_fp64_flips']}, "
          f"exact-vs-fp64 differing decisions {int((e.astype(int) - o).sum())}")
    R = O.ref()
    if R is not None:
        ref = np.zeros_like(o)
        R.ref_estimate_vix_fp64(O._p(z), 1000, 1000, 100, 10, 10, 10, 1, 0, O._p(ref), 0, 1000)
        assert np.array_equal(g, ref)


@pytest.mark.parametrize("roi,h,k", [(40, 0, "2"), (40, 0, "3"), (100, 10, "1"), (250, 0, "2"), (300, 5, "1")])
@pytest.mark.parametrize("arith", ["fp64", "exact"])
def test_viewsheds_tie_terrain(engine, monkeypatch, roi, h, k, arith):
    """Viewsheds on a tie-heavy terrain, interior and edge observers, the K-observer
    sweeps and the generic roi > 250 kernel: bit-exact vs the oracle's same
    arithmetic (fp64: every tied ray re-decided on the device)."""
    T = _T()
    z = _tie_terrain(700, 650, 11, 900)
    rng = np.random.default_rng(roi + len(arith))
    n = 3000
    rows, cols = rng.integers(0, 700, n).astype(np.int32), rng.integers(0, 650, n).astype(np.int32)
    rows[:6], cols[:6] = [0, 699, 0, 699, 41, 658], [0, 649, 649, 0, 41, 608]
    monkeypatch.setenv("TXS_VS_K", k)
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(roi, h, h, los_arith=arith))
    gw, gv, gp = engine.viewsheds(roi)
    sel = np.unique(np.concatenate([np.arange(6), np.arange(0, n, 7)])) if roi >= 250 else np.arange(n)
    ow, ov = O.viewsheds(z, roi, h, h, rows[sel], cols[sel], arith=arith)
    bad = np.nonzero((gv[sel] != ov).any(1))[0]
    assert len(bad) == 0, f"{len(bad)} viewsheds differ, first {sel[bad[:5]]}"
    assert np.array_equal(gp[sel], np.unpackbits(ov.view(np.uint8), axis=1).sum(1))
    if arith == "fp64":
        st = engine.stats()
        print(f"roi {roi}: fp64 tied rays {st['vs_fp64_ties']}, flipped bits {st['vs_fp64_flips']}")
