"""txs_run_pipeline_host: run_pipeline straight from a host terrain, the upload
in chunks on a copy stream overlapping VIX band by band (the 16-step
terrain-walk path), else the whole terrain first -- same picks, VixMap and cum
as txs_set_terrain + txs_run_pipeline, and the oracle's."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _ref(e, z, p):
    e.set_terrain(z)
    r = e.run_pipeline(p)
    return r, e.vix(), e.cumulative()


@pytest.mark.parametrize("shape,roi,bw,k,S,water", [((1000, 1000), 100, 100, 10, 10, 0),     # config 1
                                                    ((2300, 700), 100, 100, 4, 6, 300),      # banded, water rows
                                                    ((900, 800), 30, 40, 3, 8, 0),           # many small bands
                                                    ((1100, 900), 160, 128, 4, 5, 0)])       # quad planes: no bands
@pytest.mark.parametrize("chunk", [None, "64", "grow"])   # default (one chunk below 128 MB) / forced bands / growing chunks
def test_host_pipeline_matches(engine, monkeypatch, shape, roi, bw, k, S, water, chunk):
    import torch
    if chunk == "grow":   # chunks of 64, 64, 128, 256 ... rows, at most a quarter of the grid each
        monkeypatch.setenv("TXS_UPLOAD_BANDS", "grow")
        monkeypatch.setenv("TXS_UPLOAD_FIRST_ROWS", "64")
    elif chunk:
        monkeypatch.setenv("TXS_UPLOAD_CHUNK_ROWS", chunk)
    import paper_2006_16783_b200 as T
    nr, nc = shape
    z = O.generate_fractal(nr, nc, 0.55, 17, 0, 3500)
    z[:water] = 0
    zp = torch.empty((nr, nc), dtype=torch.int16, pin_memory=True).numpy()
    zp[:] = z
    p = T.make_params(roi, 10, 10, samples=S, per_block=k, block_width=bw, target=0.98, max_selected=150, seed=3)
    ref, vix, cum = _ref(engine, z, p)
    for src in (zp, z):   # pinned (overlapped) and pageable host memory
        got = engine.run_pipeline_host(src, p)
        assert got["stop"] == ref["stop"] and np.array_equal(got["index"], ref["index"])
        assert np.array_equal(got["gain"], ref["gain"]) and np.array_equal(got["coverage"], ref["coverage"])
        assert np.array_equal(engine.vix(), vix) and np.array_equal(engine.cumulative(), cum)
        assert np.array_equal(engine.terrain(), z)
    if roi == 100 and nr == 1000:
        o = O.estimate_vix(z, roi, 10, 10, S, 3)
        assert np.array_equal(vix, o)


def test_host_pipeline_rejects_nodata(engine):
    import paper_2006_16783_b200 as T
    z = O.generate_fractal(600, 500, 0.5, 2, 0, 2000)
    z[599, 3] = -32768
    with pytest.raises(T.TxsError) as e:
        engine.run_pipeline_host(z, T.make_params(40, 10, 10, samples=4, per_block=2, block_width=50))
    assert e.value.status == "NODATA"
