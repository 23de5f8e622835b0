"""The VIX crossing statistic (txs_stats.vix_crossings_full, the roofline's
algorithmic LOS count) is a function of grid, band, roi, S and seed only:
k_vix_lanes counts it on the first launch with a given key and adds the cached
count afterwards -- the figure must not change between the two, and a new key
recounts."""
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def test_vix_crossing_statistic_cached(engine):
    import paper_2006_16783_b200 as T
    z = O.generate_fractal(700, 600, 0.5, 3, 0, 2000)
    engine.set_terrain(z)
    got = []
    for seed in (5, 5, 6, 5):
        engine.reset_stats()
        engine.estimate_vix(T.make_params(60, 10, 10, samples=8, seed=seed))
        st = engine.stats()
        got.append(st["vix_crossings_full"])
        assert st["vix_los"] == 700 * 600 * 8
    assert got[0] == got[1] == got[3] > 0
    assert got[2] != got[0] and got[2] > 0
