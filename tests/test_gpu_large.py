"""BASELINE configurations 2-5 at full size on the GPU against the CPU oracle
(the reference contract: SITE output identical to naive
greedy).

- C2: every stage in full -- terrain, VixMap, candidate list, all 16,384
  viewsheds, the whole SITE sequence, stop reason and cumulative bitmap.
- C3 / C4: terrain (C3 in full), VIX on every 64th row, FINDMAX in full on the
  GPU VixMap, viewsheds of every candidate with index % 64 == 0, then the FULL
  SITE sequence, stop reason and cumulative bitmap of the oracle's lazy greedy
  (== naive greedy, tests/test_oracle_spec.py) fed with the downloaded GPU
  viewsheds of every candidate.
- C5: the 1,048,576 observer draws in full, viewsheds at index % 64 == 0, and
  the full SITE (8,192 picks) on all 1M downloaded viewsheds (32.9 GB).
All with the default arithmetic (SPEC.md:147 fp64)."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def _site_vs_oracle(e, cfg, p, rows, cols, wins, words):
    """GPU SITE on the resident viewsheds vs the oracle's greedy on the same
    (downloaded) viewsheds: sequence, gains, coverage, stop reason, cum."""
    res = e.site(p, cap=cfg.max_selected + 1)
    cum = e.cumulative()
    o = O.site(rows, cols, wins, words, cfg.nrows, cfg.ncols, cfg.target, cfg.max_selected)
    assert res["stop"] == o["stop"], (res["stop"], o["stop"])
    assert np.array_equal(res["index"], o["index"]), (len(res["index"]), len(o["index"]))
    assert np.array_equal(res["gain"], o["gain"])
    assert np.array_equal(res["coverage"], o["coverage"])
    assert np.array_equal(res["row"], o["row"]) and np.array_equal(res["col"], o["col"])
    assert np.array_equal(cum, o["cum"])
    print(f"{cfg.name}: SITE {len(res['index'])} picks, stop {res['stop']}, "
          f"coverage {res['coverage'][-1]:.6f} == oracle")
    return res


def _viewsheds_every_64th(e, cfg, z, rows, cols):
    """Downloads every viewshed (SPEC layout) and checks index % 64 == 0 against
    the oracle; returns (wins, words, pops) for the SITE check."""
    gw, gv, gp = e.viewsheds(cfg.roi)
    idx = np.arange(0, len(rows), 64)
    ow, ov = O.viewsheds(z, cfg.roi, cfg.height, cfg.height, rows[idx], cols[idx])
    assert np.array_equal(gw[idx], ow)
    bad = np.nonzero((gv[idx] != ov).any(1))[0]
    assert len(bad) == 0, f"{len(bad)} viewsheds differ, first {idx[bad[:5]]}"
    assert np.array_equal(gp[idx], O.popcounts(ov))
    print(f"{cfg.name}: {len(idx)} viewsheds (index % 64 == 0) bit-exact")
    return gw, gv


def _setup(e, name):
    from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain
    cfg = CONFIGS[name]
    setup_terrain(e, cfg)
    return cfg, params_for(cfg)


def _terrain_check(z, cfg):
    zo = O.generate_fractal(cfg.nrows, cfg.ncols, cfg.roughness, cfg.terrain_seed, cfg.zmin, cfg.zmax)
    if cfg.water_rows:
        zo[:cfg.water_rows] = 0
    assert np.array_equal(z, zo)


def test_config2_full_end_to_end():
    """C2 (the headline single-GPU pipeline of round 1) with every stage in full."""
    import paper_2006_16783_b200 as T
    with T.Engine(0) as e:
        cfg, p = _setup(e, "c2")
        z = e.terrain()
        _terrain_check(z, cfg)
        vix = e.estimate_vix(p)
        ovix = O.estimate_vix(z, cfg.roi, cfg.height, cfg.height, cfg.samples, cfg.vix_seed)
        assert np.array_equal(vix, ovix), int((vix != ovix).sum())
        rows, cols, sc = e.find_candidates(p)
        orow, ocol, osc = O.find_candidates(ovix, cfg.block, cfg.per_block)
        assert np.array_equal(rows, orow) and np.array_equal(cols, ocol) and np.array_equal(sc, osc)
        assert len(rows) == 16384
        e.compute_all_viewsheds(p)
        gw, gv, gp = e.viewsheds(cfg.roi)
        ow, ov = O.viewsheds(z, cfg.roi, cfg.height, cfg.height, orow, ocol)
        assert np.array_equal(gw, ow)
        bad = np.nonzero((gv != ov).any(1))[0]
        assert len(bad) == 0, f"{len(bad)} viewsheds differ"
        del gv
        res = e.site(p, cap=cfg.max_selected + 1)
        o = O.site(orow, ocol, ow, ov, cfg.nrows, cfg.ncols, cfg.target, cfg.max_selected)
        assert res["stop"] == o["stop"]
        assert np.array_equal(res["index"], o["index"]) and np.array_equal(res["gain"], o["gain"])
        assert np.array_equal(res["coverage"], o["coverage"])
        assert np.array_equal(e.cumulative(), o["cum"])
        st = e.stats()
        print(f"c2: {len(res['index'])} sited, stop {res['stop']}; fp64 ties: VIX {st['vix_fp64_ties']} "
              f"(flipped {st['vix_fp64_flips']}), VIEWSHED rays {st['vs_fp64_ties']} (bits {st['vs_fp64_flips']})")
        # the one-call pipeline gives the same result
        pp = e.run_pipeline(p, cap=cfg.max_selected + 1)
        assert np.array_equal(pp["index"], res["index"]) and pp["stop"] == res["stop"]


def _vix_findmax_rows(e, cfg, p, z, step=64):
    vix = e.estimate_vix(p)
    sel = np.arange(0, cfg.nrows, step)
    o = O.estimate_vix_rows(z, cfg.roi, cfg.height, cfg.height, cfg.samples, cfg.vix_seed, sel)
    bad = np.nonzero((vix[sel] != o).any(1))[0]
    assert len(bad) == 0, f"VIX rows differ: {sel[bad[:5]]}"
    print(f"{cfg.name}: VIX rows 0, {step}, 2*{step}, ... ({len(range(0, cfg.nrows, step))} rows) bit-exact")
    rows, cols, sc = e.find_candidates(p)
    orow, ocol, osc = O.find_candidates(vix, cfg.block, cfg.per_block)
    assert np.array_equal(rows, orow) and np.array_equal(cols, ocol) and np.array_equal(sc, osc)
    del vix
    return rows, cols


def test_config3_full_size():
    import paper_2006_16783_b200 as T
    with T.Engine(0) as e:
        cfg, p = _setup(e, "c3")
        z = e.terrain()
        _terrain_check(z, cfg)
        rows, cols = _vix_findmax_rows(e, cfg, p, z)
        assert len(rows) == 131072
        e.compute_all_viewsheds(p)
        wins, words = _viewsheds_every_64th(e, cfg, z, rows, cols)
        res = _site_vs_oracle(e, cfg, p, rows, cols, wins, words)
        assert res["stop"] == "max-selected" and len(res["index"]) == 4096


def test_config4_full_size():
    import paper_2006_16783_b200 as T
    with T.Engine(0) as e:
        cfg, p = _setup(e, "c4")
        z = e.terrain()
        rows, cols = _vix_findmax_rows(e, cfg, p, z)
        assert len(rows) == 116 * 116 * 16
        e.compute_all_viewsheds(p)
        wins, words = _viewsheds_every_64th(e, cfg, z, rows, cols)
        del z
        res = _site_vs_oracle(e, cfg, p, rows, cols, wins, words)
        assert res["stop"] == "max-selected" and len(res["index"]) == 4096


def test_config5_full_size():
    import paper_2006_16783_b200 as T
    with T.Engine(0) as e:
        cfg, p = _setup(e, "c5")
        z = e.terrain()
        _terrain_check(z, cfg)
        e.random_observers(cfg.random_observers, cfg.observer_seed)
        rows, cols, _ = e.candidates()
        orow, ocol = O.random_observers(cfg.nrows, cfg.ncols, cfg.random_observers, cfg.observer_seed)
        assert np.array_equal(rows, orow) and np.array_equal(cols, ocol)
        e.compute_all_viewsheds(p)
        wins, words = _viewsheds_every_64th(e, cfg, z, rows, cols)
        res = _site_vs_oracle(e, cfg, p, rows, cols, wins, words)
        # with roi 250 and h 50 the picks reach full coverage (target 1.0) before the 8,192 cap
        assert res["stop"] == "target-reached" and res["coverage"][-1] == 1.0 and len(res["index"]) < 8192
