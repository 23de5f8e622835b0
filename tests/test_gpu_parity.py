"""GPU parity: every stage through the C-ABI against the CPU oracle on the
same seeded inputs — bit-exact (integer/byte/index work: VixMap bytes,
candidate lists, packed viewshed words, selection sequence, cumulative bitmap).
Full BASELINE config-1 size here; larger configs by sampled rows/observers."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _T():
    import paper_2006_16783_b200 as T
    return T


@pytest.fixture(scope="module")
def c1(engine):
    """BASELINE config 1: 1000x1000, roughness 0.5, 0..4000 m."""
    z = O.generate_fractal(1000, 1000, 0.5, 1, 0, 4000)
    return z


# ---- terrain -------------------------------------------------------------------
@pytest.mark.parametrize("nr,nc,rough,seed,zmin,zmax", [
    (1000, 1000, 0.5, 1, 0, 4000), (257, 300, 0.6, 9, -100, 3000), (2, 2, 1.0, 3, 0, 10),
    (4096, 4096, 0.6, 2, 0, 3000), (33, 1025, 0.5, 4, 0, 4000)])
def test_generator_bit_exact(engine, nr, nc, rough, seed, zmin, zmax):
    engine.generate_fractal(nr, nc, rough, seed, zmin, zmax)
    assert np.array_equal(engine.terrain(), O.generate_fractal(nr, nc, rough, seed, zmin, zmax))


def test_fill_rows_and_set_terrain(engine):
    z = O.generate_fractal(300, 200, 0.5, 5, 0, 4000)
    engine.set_terrain(z)
    assert np.array_equal(engine.terrain(), z)
    engine.fill_rows(0, 37, 0)
    z2 = z.copy(); z2[:37] = 0
    assert np.array_equal(engine.terrain(), z2)
    bad = z.copy(); bad[5, 5] = -32768
    with pytest.raises(_T().TxsError) as e:
        engine.set_terrain(bad)
    assert e.value.status == "NODATA"


# ---- los -----------------------------------------------------------------------
def test_is_visible_batch_bit_exact(engine):
    rng = np.random.default_rng(11)
    for seed, (nr, nc) in [(1, (200, 200)), (2, (64, 700)), (3, (1000, 1000))]:
        z = O.generate_fractal(nr, nc, 0.6, seed, 0, 4000)
        engine.set_terrain(z)
        pairs = np.stack([rng.integers(0, nr, 20000), rng.integers(0, nc, 20000),
                          rng.integers(0, nr, 20000), rng.integers(0, nc, 20000)], 1).astype(np.int32)
        pairs[:50, 2:] = pairs[:50, :2]                       # zero-length
        pairs[50:100, 2] = pairs[50:100, 0]                   # axis aligned
        for ht, hr in [(10, 10), (0, 0), (50, 3)]:
            assert np.array_equal(engine.is_visible_batch(pairs, ht, hr), O.is_visible_batch(z, pairs, ht, hr))
    with pytest.raises(_T().TxsError) as e:
        engine.is_visible_batch(np.array([[0, 0, 5000, 0]], np.int32), 1, 1)
    assert e.value.status == "OFF_GRID"


def test_is_visible_ridge_and_graze(engine):
    z = np.zeros((3, 5), np.int16)
    z[1] = [0, 0, 50, 0, 0]
    engine.set_terrain(z)
    assert list(engine.is_visible_batch([[1, 0, 1, 4]], 1, 1)) == [0]
    z[1] = [0, 0, 1, 0, 0]
    engine.set_terrain(z)
    assert list(engine.is_visible_batch([[1, 0, 1, 4]], 1, 1)) == [1]


# ---- vix -----------------------------------------------------------------------
def test_vix_c1_bit_exact(engine, c1):
    """Config 1 in full: 1000x1000, roi 100, h 10, 10 samples (shared-memory tile path)."""
    T = _T()
    engine.set_terrain(c1)
    p = T.make_params(100, 10, 10, samples=10, seed=12345)
    g = engine.estimate_vix(p)
    o = O.estimate_vix(c1, 100, 10, 10, 10, 12345)
    assert np.array_equal(g, o), int((g != o).sum())
    st = engine.stats()
    assert st["vix_los"] >= 1000 * 1000 * 10


@pytest.mark.parametrize("roi,samples,ht,hr", [(7, 20, 0, 0), (150, 10, 20, 20), (200, 20, 20, 20)])
def test_vix_rows_bit_exact(engine, roi, samples, ht, hr):
    """Global-memory path (roi >= 150) and small-roi smem path on sampled rows."""
    T = _T()
    z = O.generate_fractal(1200, 900, 0.6, 8, 0, 3000)
    engine.set_terrain(z)
    g = engine.estimate_vix(T.make_params(roi, ht, hr, samples=samples, seed=77))
    for rb, re in [(0, 24), (590, 610), (1176, 1200)]:
        o = O.estimate_vix(z, roi, ht, hr, samples, 77, rows=(rb, re))
        assert np.array_equal(g[rb:re], o[rb:re]), (rb, int((g[rb:re] != o[rb:re]).sum()))


@pytest.mark.parametrize("path", ["smem", "pairs", "zt"])
@pytest.mark.parametrize("roi,samples,ht,hr", [(60, 24, 15, 5), (141, 33, 0, 30), (255, 9, 20, 20)])
def test_vix_paths_bit_exact(engine, monkeypatch, path, roi, samples, ht, hr):
    """Every VIX kernel path (shared-memory tile, quad planes, column-major copy),
    forced with TXS_VIX_PATH, against the oracle -- including roi 255, where the
    quad path's dp2a weights reach 255; rows at both grid edges."""
    T = _T()
    z = O.generate_fractal(700, 610, 0.7, 21, -500, 3000)
    engine.set_terrain(z)
    monkeypatch.setenv("TXS_VIX_PATH", path)
    g = engine.estimate_vix(T.make_params(roi, ht, hr, samples=samples, seed=31))
    for rb, re in [(0, 6), (300, 306), (694, 700)]:
        o = O.estimate_vix(z, roi, ht, hr, samples, 31, rows=(rb, re))
        assert np.array_equal(g[rb:re], o[rb:re]), (path, rb, int((g[rb:re] != o[rb:re]).sum()))


@pytest.mark.parametrize("nr,nc,rough,zmin,zmax,roi,samples,ht,hr", [
    (700, 610, 0.7, -500, 3000, 60, 24, 15, 5),      # rough, negative elevations
    (513, 777, 0.5, 0, 4000, 100, 10, 10, 10),       # smooth (most groups skipped)
    (400, 401, 0.9, -32000, 32000, 255, 9, 0, 0),    # near-full int16 range, roi 255
    (300, 300, 0.3, 0, 50, 200, 20, 1, 1),           # low relief, grazing LOS
    (37, 1000, 0.6, 0, 3000, 150, 16, 20, 20),       # thin grid: windows off both edges
])
def test_vix_skip_map_matches_full_walk(engine, monkeypatch, nr, nc, rough, zmin, zmax, roi, samples, ht, hr):
    """The quad path's conservative skip test (TXS_VIX_SKIP, default on) gives
    the full walk's VixMap bit for bit over the whole grid, and the oracle's on
    edge rows."""
    T = _T()
    z = O.generate_fractal(nr, nc, rough, 5, zmin, zmax)
    engine.set_terrain(z)
    p = T.make_params(roi, ht, hr, samples=samples, seed=9)
    monkeypatch.setenv("TXS_VIX_PATH", "pairs")
    monkeypatch.setenv("TXS_VIX_SKIP", "0")
    full = engine.estimate_vix(p)
    # per-segment / flattened (default) skip tests, 4- and 16-step groups, every unit size
    for mode, group, unit in [("2", "4", ""), ("2", "16", ""), ("1", "4", "4"), ("1", "4", "8"),
                              ("1", "16", "1"), ("1", "16", "2")]:
        monkeypatch.setenv("TXS_VIX_SKIP", mode)
        monkeypatch.setenv("TXS_VIX_GROUP", group)
        monkeypatch.setenv("TXS_VIX_UNIT", unit or "8")
        skip = engine.estimate_vix(p)
        assert np.array_equal(full, skip), (mode, group, unit, int((full != skip).sum()))
    monkeypatch.delenv("TXS_VIX_GROUP")
    monkeypatch.delenv("TXS_VIX_UNIT")
    monkeypatch.setenv("TXS_VIX_SKIP", "1")
    skip = engine.estimate_vix(p)   # the defaults
    assert np.array_equal(full, skip)
    for rb, re in [(0, 3), (nr - 3, nr)]:
        o = O.estimate_vix(z, roi, ht, hr, samples, 9, rows=(rb, re))
        assert np.array_equal(skip[rb:re], o[rb:re]), rb


@pytest.mark.parametrize("samples", [1, 2, 3, 64])
def test_vix_sample_counts_queue_paths(engine, monkeypatch, samples):
    """Receiver-queue bookkeeping of the quad path: S = 1 and 2 fill the
    16-post ring (drained with partial batches), S = 3 just fits it, S = 64
    spreads each post over several 32-segment batches."""
    T = _T()
    z = O.generate_fractal(90, 77, 0.6, 13, 0, 2000)
    engine.set_terrain(z)
    monkeypatch.setenv("TXS_VIX_PATH", "pairs")
    p = T.make_params(30, 5, 5, samples=samples, seed=17)
    g = engine.estimate_vix(p)
    o = O.estimate_vix(z, 30, 5, 5, samples, 17)
    assert np.array_equal(g, o), int((g != o).sum())


def test_vix_flat_and_tiny(engine):
    T = _T()
    engine.set_terrain(np.full((70, 45), 3, np.int16))
    assert (engine.estimate_vix(T.make_params(30, 10, 10, samples=13)) == 13).all()
    z = O.generate_fractal(5, 3, 0.5, 1, 0, 100)
    engine.set_terrain(z)
    assert np.array_equal(engine.estimate_vix(T.make_params(40, 1, 2, samples=7, seed=5)),
                          O.estimate_vix(z, 40, 1, 2, 7, 5))


# ---- findmax -------------------------------------------------------------------
@pytest.mark.parametrize("nr,nc,bw,k,levels", [(1000, 1000, 100, 10, 11), (1000, 1000, 128, 16, 21),
                                               (300, 257, 40, 2000, 3), (96, 96, 7, 5, 1), (128, 128, 64, 32, 256)])
def test_findmax_bit_exact(engine, nr, nc, bw, k, levels):
    T = _T()
    rng = np.random.default_rng(nr + bw)
    s = rng.integers(0, levels, (nr, nc)).astype(np.uint8)
    engine.set_terrain(np.zeros((nr, nc), np.int16))
    engine.set_vix(s)
    rows, cols, sc = engine.find_candidates(T.make_params(max(3, bw), per_block=k, block_width=bw))
    orow, ocol, osc = O.find_candidates(s, bw, k)
    assert np.array_equal(rows, orow) and np.array_equal(cols, ocol) and np.array_equal(sc, osc)


def test_random_observers_bit_exact(engine):
    engine.set_terrain(np.zeros((16384, 16384 // 64), np.int16))
    engine.random_observers(100000, 424242)
    r, c, _ = engine.candidates()
    orow, ocol = O.random_observers(16384, 16384 // 64, 100000, 424242)
    assert np.array_equal(r, orow) and np.array_equal(c, ocol)


# ---- viewshed ----------------------------------------------------------------------
def _vs_compare(engine, z, roi, ht, hr, rows, cols):
    T = _T()
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(roi, ht, hr))
    gw, gv, gp = engine.viewsheds(roi)
    ow, ov = O.viewsheds(z, roi, ht, hr, rows, cols)
    assert np.array_equal(gw, ow)
    bad = np.nonzero((gv != ov).any(1))[0]
    assert len(bad) == 0, f"{len(bad)} viewsheds differ, first {bad[:5]}"
    pops = np.unpackbits(ov.view(np.uint8), axis=1).sum(1)
    assert np.array_equal(gp, pops)


def test_viewsheds_c1_bit_exact(engine, c1):
    """Config-1 observers (a FINDMAX candidate list) at roi 100."""
    T = _T()
    engine.set_terrain(c1)
    p = T.make_params(100, 10, 10, samples=10, per_block=10, block_width=100, seed=1)
    engine.estimate_vix(p, copy=False)
    rows, cols, _ = engine.find_candidates(p)
    assert len(rows) == 1000
    _vs_compare(engine, c1, 100, 10, 10, rows, cols)


@pytest.mark.parametrize("k,pairs,step", [(1, 0, 2), (2, 0, 2), (2, 1, 2), (4, 1, 2), (2, 1, 4), (3, 1, 2)])
def test_viewsheds_k_paths_bit_exact(engine, monkeypatch, k, pairs, step):
    """Every VIEWSHED sweep: K observers per CTA (1/2/3/4, TXS_VS_K), int16 posts
    or H/V pair planes (TXS_VS_PAIRS), 2 or 4 events per sweep iteration
    (TXS_VS_STEP), tile-sorted order (n >= 4096), CTAs mixing interior and edge
    observers (corners, edges) -- all against the oracle."""
    rng = np.random.default_rng(100 + k)
    z = O.generate_fractal(700, 650, 0.6, 33, -200, 2500)
    n = 5000
    rows, cols = rng.integers(0, 700, n).astype(np.int32), rng.integers(0, 650, n).astype(np.int32)
    rows[:6], cols[:6] = [0, 699, 0, 699, 41, 658], [0, 649, 649, 0, 41, 608]
    monkeypatch.setenv("TXS_VS_K", str(k))
    monkeypatch.setenv("TXS_VS_PAIRS", str(pairs))
    monkeypatch.setenv("TXS_VS_STEP", str(step))
    _vs_compare(engine, z, 40, 15, 5, rows, cols)


def test_viewsheds_c5_default_path(engine):
    """The C5 production sweep with no overrides: roi 250 >= 225 selects K = 2
    observers per CTA, 4 events per iteration and the interleaved pair planes
    (>= 2 * SMs * 4 observers); interior, edge and corner observers of a grid
    only a little larger than the window, compared in full."""
    rng = np.random.default_rng(250)
    z = O.generate_fractal(900, 1000, 0.5, 35, 0, 4000)
    n = 2 * 148 * 4 + 321
    rows, cols = rng.integers(0, 900, n).astype(np.int32), rng.integers(0, 1000, n).astype(np.int32)
    rows[:8], cols[:8] = [0, 899, 0, 899, 251, 648, 450, 0], [0, 999, 999, 0, 251, 748, 0, 500]
    _vs_compare(engine, z, 250, 50, 50, rows, cols)


@pytest.mark.parametrize("roi,h", [(200, 20), (250, 50), (1, 0), (3, 5), (300, 10), (100, 10)])
def test_viewsheds_sampled_bit_exact(engine, roi, h):
    z = O.generate_fractal(1100, 1300, 0.5, 31, 0, 4000)
    rng = np.random.default_rng(roi)
    rows = np.concatenate([rng.integers(0, 1100, 120), [0, 1099, 0, 1099, 550]]).astype(np.int32)
    cols = np.concatenate([rng.integers(0, 1300, 120), [0, 1299, 1299, 0, 3]]).astype(np.int32)
    _vs_compare(engine, z, roi, h, h, rows, cols)


def test_viewshed_flat_disk_and_small_grid(engine):
    T = _T()
    z = np.full((100, 100), 100, np.int16)
    engine.set_terrain(z)
    engine.set_candidates([50], [50])
    engine.compute_all_viewsheds(T.make_params(30, 10, 10))
    _, _, pops = engine.viewsheds(30)
    assert pops[0] == 2821
    small = O.generate_fractal(9, 14, 0.7, 2, 0, 500)
    _vs_compare(engine, small, 40, 3, 3, [0, 8, 4, 4], [0, 13, 7, 7])


# ---- site ------------------------------------------------------------------------
def _site_compare(engine, roi, rows, cols, nr, nc, target, max_sel, mode):
    T = _T()
    wins, words, _ = engine.viewsheds(roi)
    g = engine.site(T.make_params(roi, target=target, max_selected=max_sel, site_mode=mode))
    o = O.site(rows, cols, wins, words, nr, nc, target, max_sel)
    assert g["stop"] == o["stop"]
    assert np.array_equal(g["index"], o["index"]), (g["index"][:10], o["index"][:10])
    assert np.array_equal(g["gain"], o["gain"]) and np.array_equal(g["coverage"], o["coverage"])
    assert np.array_equal(g["row"], o["row"]) and np.array_equal(g["col"], o["col"])
    assert np.array_equal(engine.cumulative(), o["cum"])
    return g


@pytest.mark.parametrize("mode", [0, 1])
def test_site_c1_bit_exact(engine, c1, mode):
    """Config 1: until 95% or 200 observers; both device strategies."""
    T = _T()
    engine.set_terrain(c1)
    p = T.make_params(100, 10, 10, samples=10, per_block=10, block_width=100, seed=1)
    engine.estimate_vix(p, copy=False)
    rows, cols, _ = engine.find_candidates(p)
    engine.compute_all_viewsheds(p)
    _site_compare(engine, 100, rows, cols, 1000, 1000, 0.95, 200, mode)


@pytest.mark.parametrize("mode", [0, 1])
def test_site_random_dense_bit_exact(engine, mode):
    """Many overlapping candidates, run to exhaustion/zero gain (target 1.0)."""
    T = _T()
    z = O.generate_fractal(300, 420, 0.6, 17, 0, 4000)
    rng = np.random.default_rng(3 + mode)
    rows, cols = rng.integers(0, 300, 700).astype(np.int32), rng.integers(0, 420, 700).astype(np.int32)
    rows[5], cols[5] = rows[4], cols[4]                     # a duplicate (zero second gain)
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(25, 10, 10))
    g = _site_compare(engine, 25, rows, cols, 300, 420, 1.0, 0, mode)
    assert (np.diff(g["gain"]) <= 0).all()


@pytest.mark.parametrize("mode", [0, 1])
def test_site_bucket_tiled_bit_exact(engine, mode):
    """>= 64 candidates per roi-sized bucket: mode 1 takes the bucket-tiled gain
    kernel (cum region staged in shared memory); grid edges included."""
    T = _T()
    z = O.generate_fractal(200, 256, 0.5, 5, 0, 2000)
    rng = np.random.default_rng(11)
    n = 9500
    rows, cols = rng.integers(0, 200, n).astype(np.int32), rng.integers(0, 256, n).astype(np.int32)
    rows[:4], cols[:4] = [0, 199, 0, 199], [0, 255, 255, 0]
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(20, 5, 5))
    _site_compare(engine, 20, rows, cols, 200, 256, 1.0, 0, mode)


@pytest.mark.parametrize("kind,shape", [("full", None), ("tiled", None), ("t8", None), ("t8", "pf0"), ("t8", "pf7"),
                                        ("strips", None), ("strips", "8x1"), ("strips", "40x3")])
def test_site_full_rescan_gain_pass_forms(engine, monkeypatch, kind, shape):
    """Mode-1 rounds through every gain-pass kernel (per-candidate, bucket-tiled,
    the 8x8-tile shadow layout with its own cum, strip-tile task list with bulk
    copies; A/B knob TXS_GAIN_PASS) and strip
    shapes whose tiles cut windows at many rows and bucket columns; grid edges
    and a duplicate included."""
    T = _T()
    z = O.generate_fractal(230, 300, 0.6, 13, 0, 3000)
    rng = np.random.default_rng(5)
    n = 900
    rows, cols = rng.integers(0, 230, n).astype(np.int32), rng.integers(0, 300, n).astype(np.int32)
    rows[:5], cols[:5] = [0, 229, 0, 229, 0], [0, 299, 299, 0, 0]
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(33, 10, 10))
    monkeypatch.setenv("TXS_GAIN_PASS", kind)
    if shape and shape.startswith("pf"):   # the tile-cum L2 prefetch of grids whose cum exceeds L2
        monkeypatch.setenv("TXS_GAIN_PF_AHEAD", shape[2:])
        monkeypatch.setenv("TXS_GAIN_GRID", "1")   # several candidates per warp
    elif shape:
        sh, tx = shape.split("x")
        monkeypatch.setenv("TXS_STRIP_ROWS", sh)
        monkeypatch.setenv("TXS_STRIP_TX", tx)
    _site_compare(engine, 33, rows, cols, 230, 300, 0.99, 0, 1)
    ms, nbytes = engine.time_gain_pass(2)
    assert ms > 0 and nbytes == sum(8 * ((int(w[2]) * int(w[3]) + 63) // 64) for w in engine.viewsheds(33)[0])


@pytest.mark.parametrize("ctas", ["", "1", "3"])
def test_site_persistent_loop_widths(engine, monkeypatch, ctas):
    """Persistent SITE loop with 400-1000 expected neighbours per round (4 CTAs
    per SM by default) and forced widths, against the oracle."""
    T = _T()
    z = O.generate_fractal(300, 300, 0.6, 9, 0, 2500)
    rng = np.random.default_rng(21)
    n = 6000
    rows, cols = rng.integers(0, 300, n).astype(np.int32), rng.integers(0, 300, n).astype(np.int32)
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(20, 8, 4))
    if ctas:
        monkeypatch.setenv("TXS_SITE_LOOP_CTAS", ctas)
    _site_compare(engine, 20, rows, cols, 300, 300, 0.97, 0, 0)


@pytest.mark.parametrize("cs", ["16", "8", "0"])
@pytest.mark.parametrize("case", ["sparse", "tiny", "maxsel"])
def test_site_cluster_loop(engine, monkeypatch, cs, case):
    """The SITE loop inside one thread-block cluster (cluster barrier, partial
    winners through distributed shared memory; A/B knob TXS_SITE_CLUSTER) at
    both cluster sizes and off, against the oracle:
    sparse candidates with grid corners and a duplicate run to exhaustion, fewer
    candidates than CTAs, and a max_selected stop."""
    T = _T()
    nr, nc, roi = 420, 380, 25
    z = O.generate_fractal(nr, nc, 0.6, 31, 0, 3000)
    rng = np.random.default_rng(77)
    n = {"sparse": 700, "tiny": 5, "maxsel": 300}[case]
    rows, cols = rng.integers(0, nr, n).astype(np.int32), rng.integers(0, nc, n).astype(np.int32)
    if n > 5:
        rows[:5], cols[:5] = [0, nr - 1, 0, nr - 1, 0], [0, nc - 1, nc - 1, 0, 0]
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(roi, 10, 10))
    monkeypatch.setenv("TXS_SITE_CLUSTER", cs)
    before = engine.stats()["site_launches"]
    _site_compare(engine, roi, rows, cols, nr, nc, 1.0 if case != "maxsel" else 0.9, 40 if case == "maxsel" else 0, 0)
    assert engine.stats()["site_launches"] == before + 1   # one persistent kernel either way


@pytest.mark.parametrize("case", ["dense", "maxsel", "target", "flat-ties", "cap1", "cap3", "wide", "tiny", "single", "exhaust"])
def test_site_batched_greedy(engine, monkeypatch, case):
    """The batched exact greedy (site.cu run_site_batched: every local maximum of
    the key per round, the greedy order recovered by sorting the committed picks)
    against the oracle's serial greedy: to zero gain with a duplicate and the
    grid corners; a max_selected stop and a target stop (picks committed past
    the stop are cut and the cum rebuilt); flat terrain (every gain ties, lowest
    index wins); one and three winner slots per round; a grid wide enough that
    the batched form is the default; fewer candidates than buckets; one
    candidate; every candidate picked (exhausted)."""
    T = _T()
    nr, nc, roi, n, target, max_sel, rough = 300, 420, 25, 700, 1.0, 0, 0.6
    if case == "maxsel":
        target, max_sel = 1.0, 60
    elif case == "target":
        target = 0.55
    elif case == "flat-ties":
        nr, nc, roi, n = 200, 260, 10, 1500
    elif case == "wide":
        nr, nc, roi, n, max_sel = 1100, 1300, 10, 6000, 900
    elif case == "tiny":
        n = 5
    elif case == "single":
        n = 1
    elif case == "exhaust":
        nr, nc, roi, n = 400, 400, 6, 40
    z = np.zeros((nr, nc), np.int16) if case == "flat-ties" else O.generate_fractal(nr, nc, rough, 19, 0, 3500)
    rng = np.random.default_rng(101)
    rows, cols = rng.integers(0, nr, n).astype(np.int32), rng.integers(0, nc, n).astype(np.int32)
    if case == "exhaust":   # pairwise disjoint windows: every candidate keeps its whole gain and is picked
        k = np.arange(n)
        rows, cols = (20 + 40 * (k // 8)).astype(np.int32), (20 + 40 * (k % 8)).astype(np.int32)
    elif n > 5:
        rows[:5], cols[:5] = [0, nr - 1, 0, nr - 1, 0], [0, nc - 1, nc - 1, 0, 0]
        rows[7], cols[7] = rows[6], cols[6]
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(roi, 10, 10))
    if case != "wide":
        monkeypatch.setenv("TXS_SITE_BATCH", "1")
    if case.startswith("cap"):
        monkeypatch.setenv("TXS_SITE_BATCH_CAP", case[3:])
    before = engine.stats()["site_launches"]
    g = _site_compare(engine, roi, rows, cols, nr, nc, target, max_sel, 0)
    assert (engine.stats()["site_launches"] - before) % 40 == 0   # graphs of 8 rounds x 5 kernels: the batched form ran
    if case == "exhaust":
        assert g["stop"] == "exhausted" and len(g["index"]) == n
    if case == "maxsel":
        assert g["stop"] == "max-selected" and len(g["index"]) == 60
    if case == "target":
        assert g["stop"] == "target-reached"


def test_site_edge_cases(engine):
    T = _T()
    z = O.generate_fractal(64, 64, 0.5, 2, 0, 4000)
    engine.set_terrain(z)
    engine.set_candidates([], [])
    engine.compute_all_viewsheds(T.make_params(10))
    g = engine.site(T.make_params(10, target=0.5))
    assert g["stop"] == "exhausted" and len(g["index"]) == 0
    engine.set_candidates([10, 10, 40], [10, 10, 40])
    engine.compute_all_viewsheds(T.make_params(10))
    g = _site_compare(engine, 10, np.array([10, 10, 40]), np.array([10, 10, 40]), 64, 64, 1.0, 0, 0)
    assert g["stop"] == "zero-gain"
    g = _site_compare(engine, 10, np.array([10, 10, 40]), np.array([10, 10, 40]), 64, 64, 1.0, 1, 0)
    assert g["stop"] == "max-selected"


def test_marginal_gains_vs_oracle(engine):
    T = _T()
    z = O.generate_fractal(200, 333, 0.5, 6, 0, 4000)
    rng = np.random.default_rng(1)
    rows, cols = rng.integers(0, 200, 300).astype(np.int32), rng.integers(0, 333, 300).astype(np.int32)
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(30, 10, 10))
    wins, words, _ = engine.viewsheds(30)
    for density in (0.0, 0.3, 0.9):
        cum = O.pack_dense(rng.random((200, 333)) < density)
        gains = engine.marginal_gains(cum)
        exp = [O.marginal_gain(wins[i], words[i], cum, 200, 333) for i in range(300)]
        assert list(gains) == exp


def test_set_viewsheds_then_site(engine):
    """SITE on injected (oracle) viewsheds, the drop-in path for a caller that
    already holds packed viewsheds."""
    T = _T()
    z = O.generate_fractal(256, 256, 0.5, 12, 0, 4000)
    rng = np.random.default_rng(9)
    rows, cols = rng.integers(0, 256, 400).astype(np.int32), rng.integers(0, 256, 400).astype(np.int32)
    ow, ov = O.viewsheds(z, 20, 10, 10, rows, cols)
    engine.set_terrain(z)
    engine.set_viewsheds(20, rows, cols, ow, ov)
    g = engine.site(T.make_params(20, target=0.9))
    o = O.site(rows, cols, ow, ov, 256, 256, 0.9)
    assert np.array_equal(g["index"], o["index"]) and g["stop"] == o["stop"]
    assert np.array_equal(engine.cumulative(), o["cum"])


def test_set_viewsheds_rejects_malformed_windows(engine):
    """Injected windows must be the origin's clipped roi box (the
    SITE neighbour search relies on it) with zero padding bits."""
    T = _T()
    z = O.generate_fractal(128, 128, 0.5, 3, 0, 1000)
    rows, cols = np.array([5, 64], np.int32), np.array([70, 64], np.int32)
    ow, ov = O.viewsheds(z, 10, 5, 5, rows, cols)
    engine.set_terrain(z)
    engine.set_viewsheds(10, rows, cols, ow, ov)          # well-formed: accepted
    shifted = ow.copy()
    shifted[1, 1] += 1                                     # off-centre window
    with pytest.raises(T.TxsError, match="clipped roi box"):
        engine.set_viewsheds(10, rows, cols, shifted, ov)
    dirty = ov.copy()
    nbits = int(ow[0, 2]) * int(ow[0, 3])
    assert nbits % 64
    dirty[0, nbits // 64] |= np.uint64(1) << np.uint64(63)   # a padding bit past h*w
    with pytest.raises(T.TxsError, match="padding bits"):
        engine.set_viewsheds(10, rows, cols, ow, dirty)
    with pytest.raises(T.TxsError, match="off the grid"):
        engine.set_viewsheds(10, np.array([128], np.int32), np.array([3], np.int32), ow[:1], ov[:1])


# ---- pipeline ---------------------------------------------------------------------
def test_run_pipeline_c1_matches_oracle(engine, c1):
    """run_pipeline on config 1 end to end vs the oracle stages."""
    T = _T()
    engine.set_terrain(c1)
    p = T.make_params(100, 10, 10, samples=10, per_block=10, block_width=100, target=0.95,
                      max_selected=200, seed=2024)
    res = engine.run_pipeline(p)
    s = O.estimate_vix(c1, 100, 10, 10, 10, 2024)
    rows, cols, _ = O.find_candidates(s, 100, 10)
    ow, ov = O.viewsheds(c1, 100, 10, 10, rows, cols)
    o = O.site(rows, cols, ow, ov, 1000, 1000, 0.95, 200)
    assert np.array_equal(res["index"], o["index"]) and res["stop"] == o["stop"]
    assert np.array_equal(engine.cumulative(), o["cum"])
    assert set(res["stage_ms"]) == {"vix", "findmax", "viewshed", "site"}


def test_errors_are_stage_tagged(engine):
    T = _T()
    engine.set_terrain(np.zeros((10, 10), np.int16))
    with pytest.raises(T.TxsError) as e:
        engine.estimate_vix(T.make_params(0))
    assert e.value.status == "INVALID_ARGUMENT" and "[vix]" in str(e.value)
    with pytest.raises(T.TxsError) as e:
        engine.set_candidates([11], [0])
    assert e.value.status == "OFF_GRID"


# ---- C++ host API + CLI (the reference's tools/txsite_main.cpp flags) ----------
def test_cli_matches_oracle_and_is_deterministic(tmp_path):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "paper_2006_16783_b200", "bin", "txsite")
    args = [exe, "--synth", "--nrows", "300", "--ncols", "260", "--seed", "5", "--roughness", "0.5",
            "--roi", "20", "--tx-height", "10", "--rx-height", "10", "--samples", "10", "--per-block", "4",
            "--block-width", "30", "--coverage", "0.9", "--vix-seed", "7", "--snapshots", "1,2,4"]
    outs = []
    for k in range(2):
        d = tmp_path / f"run{k}"
        d.mkdir()
        r = subprocess.run(args + ["--out-dir", str(d)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append({f: (d / f).read_bytes() for f in ("result.csv", "cumshed.pgm", "cumshed_1.pgm",
                                                         "cumshed_2.pgm", "cumshed_4.pgm")})
    assert outs[0] == outs[1]
    z = O.generate_fractal(300, 260, 0.5, 5, 0, 4000)
    s = O.estimate_vix(z, 20, 10, 10, 10, 7)
    rows, cols, _ = O.find_candidates(s, 30, 4)
    ow, ov = O.viewsheds(z, 20, 10, 10, rows, cols)
    o = O.site(rows, cols, ow, ov, 300, 260, 0.9)
    lines = outs[0]["result.csv"].decode().strip().splitlines()
    assert lines[0] == "rank,row,col,marginal_gain,cumulative_coverage"
    got = [tuple(int(x) for x in l.split(",")[1:4]) for l in lines[1:]]
    exp = list(zip(o["row"].tolist(), o["col"].tolist(), o["gain"].tolist()))
    assert got == exp
    pgm = outs[0]["cumshed.pgm"]
    assert pgm.startswith(b"P5\n260 300\n255\n")
    img = np.frombuffer(pgm[len(b"P5\n260 300\n255\n"):], np.uint8).reshape(300, 260)
    assert np.array_equal(img == 255, O.dense_bits(o["cum"], 300, 260) == 1)
    a1 = np.frombuffer(outs[0]["cumshed_1.pgm"][15:], np.uint8)
    a2 = np.frombuffer(outs[0]["cumshed_2.pgm"][15:], np.uint8)
    assert ((a1 <= a2)).all()


# ---- row-band shards on one device (virtual ranks) ---------------
@pytest.mark.parametrize("device_rounds", [False, "gather", "reduce", "replicate"])
@pytest.mark.parametrize("kind,nb", [("findmax", 1), ("findmax", 2), ("findmax", 3), ("observers", 2),
                                     ("observers", 4)])
def test_sharded_engine_matches_single(monkeypatch, kind, nb, device_rounds):
    """Row bands on virtual ranks (one device) == the single-context run, with
    the SITE rounds host-driven or device-resident (txs_site_shard_*_dev), the
    latter with the one-allgather or the two-allreduce exchange per round, or
    replicated (one allgather of the packed viewsheds, then the single-GPU loop)."""
    T = _T()
    if device_rounds:
        monkeypatch.setenv("TXS_SHARD_EXCHANGE", device_rounds)
    from paper_2006_16783_b200.configs import Config, params_for, run, setup_terrain
    from paper_2006_16783_b200.shard import LocalComm, run_sharded
    if kind == "findmax":
        cfg = Config("s1", 600, 500, 0.5, 0, 4000, 20, 10, 10, 50, 4, 0.9, 0, 5, 6, water_rows=37)
    else:
        cfg = Config("s2", 512, 480, 0.6, 0, 3000, 30, 20, 0, 0, 0, 1.0, 40, 8, 9,
                     random_observers=2000, observer_seed=77)
    params = params_for(cfg)
    engines = [T.Engine(0) for _ in range(nb)]
    res = run_sharded([(e, k) for k, e in enumerate(engines)], LocalComm(), cfg, params, nb,
                      device_rounds=bool(device_rounds))
    with T.Engine(0) as e:
        setup_terrain(e, cfg)
        single = run(e, cfg, params)
        cum = e.cumulative()
    for x in engines:
        x.close()
    assert res["stop"] == single["stop"]
    assert np.array_equal(res["index"], single["index"])
    assert np.array_equal(res["gain"], single["gain"]) and np.array_equal(res["coverage"], single["coverage"])
    assert np.array_equal(res["cum"], cum)


def test_bounds_checked_build_edge_workloads():
    """compute-sanitizer is closed on the B200 pool: run edge-heavy workloads
    (global-path VIX at roi 150 on a 1024^2 grid whose terrain ends on an
    allocation boundary, corner observers at roi 250, both SITE modes, shards)
    on the bounds-checked build, where any out-of-range terrain load traps."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TXS_CHECKED="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "memcheck_run.py")], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sharded" in r.stdout


def test_sharded_bench_torchrun_world1():
    """bench.py's row-band path under torchrun (NCCL, world 1): device-resident
    SITE rounds captured as a CUDA graph with the NCCL collectives, one JSON
    line on stdout, and the same picks as the single-context bench line."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"), "--gpus", "1",
           "--sharded", "--config", "c1", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    par = d["result"]["parallelism"]
    assert ("replicated" in par or "graph" in par) and d["roofline"] and d["stages"]["site"]["ms"] > 0
    r1 = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "c1", "--steps", "1",
                         "--warmup", "1", "--no-cpu-baseline"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    d1 = json.loads(r1.stdout.strip().splitlines()[-1])
    assert d["result"]["sited"] == d1["result"]["sited"] and d["result"]["stop"] == d1["result"]["stop"]


def test_time_gain_pass_counts_packed_bytes(engine):
    """txs_time_gain_pass: the timed full gain pass streams exactly the packed
    (SPEC-layout) bytes of every candidate window, and leaves exact gains."""
    T = _T()
    z = O.generate_fractal(300, 300, 0.6, 19, 0, 2000)
    rng = np.random.default_rng(4)
    rows, cols = rng.integers(0, 300, 500).astype(np.int32), rng.integers(0, 300, 500).astype(np.int32)
    engine.set_terrain(z)
    engine.set_candidates(rows, cols)
    engine.compute_all_viewsheds(T.make_params(30, 10, 10))
    wins, words, _ = engine.viewsheds(30)
    engine.site(T.make_params(30, target=0.5, max_selected=5))
    ms, nbytes = engine.time_gain_pass(3)
    assert ms > 0
    assert nbytes == int(sum(8 * ((int(h) * int(w) + 63) // 64) for _, _, h, w in wins))
    cum = engine.cumulative()
    exp = [O.marginal_gain(wins[i], words[i], cum, 300, 300) for i in range(len(rows))]
    assert np.array_equal(engine.marginal_gains(cum), np.array(exp))


def test_bench_json_contract_and_cache_read(engine):
    """bench.py's default-arm JSON line carries every key of the driver
    contract (roofline, cpu_baseline, e2e with copy bytes, clocks sampled
    during the timed region, launches); txs_measure_cache_read reports a
    positive L2-resident read bandwidth."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "c1", "--steps", "2",
                        "--warmup", "3"], cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["clocks"] and d["clocks"]["samples"] >= 1 and d["clocks"]["sm_mhz"] > 0
    assert engine.measure_l2(16 << 20, 4) > 100.0


def test_graft_entry_smoke():
    """__graft_entry__.smoke(): one small pipeline on cuda:0, every stage
    checked bit-exactly against the oracle (the driver's round-end check)."""
    import importlib
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    g = importlib.import_module("__graft_entry__")
    g.smoke()
