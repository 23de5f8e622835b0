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


def test_vix_crossing_statistic_upload_bands(engine, monkeypatch):
    """txs_run_pipeline_host's banded VIX (one launch per upload chunk) sums to
    the same statistic as the single launch, counted (a fresh key) or cached,
    with uniform and geometrically growing chunks; the VixMap is the same."""
    import numpy as np
    import paper_2006_16783_b200 as T
    z = O.generate_fractal(900, 640, 0.5, 4, 0, 2000)
    engine.set_terrain(z)
    p = T.make_params(60, 10, 10, samples=9, per_block=2, block_width=64, seed=11, max_selected=5)
    engine.reset_stats()
    ref_map = engine.estimate_vix(p)
    ref = engine.stats()["vix_crossings_full"]
    first = None
    for seed, mode in ((12, "uniform"), (12, "grow"), (11, "grow"), (13, "grow")):
        # counted over the bands, cached, cached from the single launch, counted over growing bands
        monkeypatch.delenv("TXS_UPLOAD_CHUNK_ROWS", raising=False)
        monkeypatch.delenv("TXS_UPLOAD_BANDS", raising=False)
        if mode == "uniform":
            monkeypatch.setenv("TXS_UPLOAD_CHUNK_ROWS", "128")
        else:
            monkeypatch.setenv("TXS_UPLOAD_BANDS", "grow")
            monkeypatch.setenv("TXS_UPLOAD_FIRST_ROWS", "64")   # chunks 64, 64, 128, 256 (a quarter), 256, 132
        q = T.make_params(60, 10, 10, samples=9, per_block=2, block_width=64, seed=seed, max_selected=5)
        engine.reset_stats()
        engine.run_pipeline_host(z, q)
        st = engine.stats()
        assert st["vix_los"] == 900 * 640 * 9
        if seed == 11:
            assert st["vix_crossings_full"] == ref
            assert np.array_equal(engine.vix(), ref_map)
        elif seed == 12:
            first = st["vix_crossings_full"] if first is None else first
            assert st["vix_crossings_full"] == first > 0
        else:
            engine.reset_stats()
            m13 = engine.estimate_vix(q)   # the cached count from the growing bands, and the single launch's map
            assert engine.stats()["vix_crossings_full"] == st["vix_crossings_full"] > 0
            monkeypatch.setenv("TXS_UPLOAD_BANDS", "grow")
            engine.run_pipeline_host(z, q)
            assert np.array_equal(engine.vix(), m13)
