"""The native multi-GPU group (txs_group_*, csrc/group.cu) driven on CPU: the
C++ orchestration -- band plan, per-rank stage fan-out on worker threads,
global candidate ids by the band-count prefix, host-staged SITE rounds with
the D9 stop rules, and the whole-grid cum assembled from every band's rows --
runs over 2 and 3 ranks of the oracle-backed stand-in engine
(oracle/fake_engine.cpp) and must reproduce the single-process oracle
pipeline exactly (block order ids, naive-greedy picks)."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
import paper_2006_16783_b200 as T
from paper_2006_16783_b200.shard import plan_bands as py_plan_bands


def _fake_ops():
    L = O.lib()
    L.txo_fake_engine_ops.restype = C.c_void_p
    return L.txo_fake_engine_ops()


@pytest.mark.parametrize("nrows,block,world", [(1000, 100, 1), (1000, 100, 3), (1000, 100, 10), (4096, 128, 8),
                                               (16384, 256, 8), (46400, 400, 8), (97, 10, 4)])
def test_plan_bands_matches_python(nrows, block, world):
    assert T.plan_bands(nrows, block, world) == py_plan_bands(nrows, block, world)


def test_plan_bands_rejects_empty_bands():
    with pytest.raises(T.TxsError):
        T.plan_bands(1000, 100, 11)   # 10 block rows, 11 ranks: a rank would own nothing
    with pytest.raises(ValueError):
        py_plan_bands(1000, 100, 11)   # shard.py refuses it too (its peers would block in the collectives)


def _oracle_pipeline(z, roi, h, S, bw, k, target, max_sel, seed, observers=None):
    nr, nc = z.shape
    if observers is None:
        vix = O.estimate_vix(z, roi, h, h, S, seed)
        rows, cols, _ = O.find_candidates(vix, bw, k)
    else:
        rows, cols = O.random_observers(nr, nc, observers[0], observers[1])
    wins, words = O.viewsheds(z, roi, h, h, rows, cols)
    return O.site(rows, cols, wins, words, nr, nc, target, max_selected=max_sel)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["findmax", "observers"])
def test_group_host_rounds_match_oracle(world, mode):
    nr, nc, roi, h, S, bw, k = 96, 80, 9, 5, 6, 12, 3
    z = O.generate_fractal(nr, nc, 0.55, 11, 0, 900)
    obs = (150, 77) if mode == "observers" else None
    ref = _oracle_pipeline(z, roi, h, S, bw, k, 0.97, 25, 4, obs)
    p = T.make_params(roi, h, h, samples=S, per_block=k, block_width=bw, target=0.97, max_selected=25, seed=4)
    with T.Group(devices=[0] * world, ops=_fake_ops()) as g:
        g.set_grid(nr, nc, p)
        assert [g.band(r) for r in range(world)] == py_plan_bands(nr, bw, world)
        g.generate_fractal(0.55, 11, 0, 900)
        if obs:
            g.random_observers(*obs)
        res = g.run_pipeline(p)
        cum = g.cumulative()
    assert np.array_equal(res["index"], ref["index"])
    assert np.array_equal(res["row"], ref["row"]) and np.array_equal(res["col"], ref["col"])
    assert np.array_equal(res["gain"], ref["gain"])
    assert res["stop"] == ref["stop"]
    assert np.array_equal(cum, ref["cum"])


def test_group_host_terrain_and_water_rows():
    """Terrain from the host (each rank copies its band + halo rows) plus a
    config-3-style water clamp, 3 ranks, stop on target coverage."""
    nr, nc, roi, h, S, bw, k = 90, 70, 8, 4, 5, 10, 2
    z = O.generate_fractal(nr, nc, 0.5, 5, 0, 700)
    z[:20] = 0
    ref = _oracle_pipeline(z, roi, h, S, bw, k, 0.5, 0, 9)
    p = T.make_params(roi, h, h, samples=S, per_block=k, block_width=bw, target=0.5, seed=9)
    with T.Group(devices=[0, 0, 0], ops=_fake_ops()) as g:
        g.set_grid(nr, nc, p)
        g.set_terrain(O.generate_fractal(nr, nc, 0.5, 5, 0, 700))
        g.fill_rows(0, 20, 0)
        res = g.run_pipeline(p)
        cum = g.cumulative()
    assert res["stop"] == ref["stop"] == "target-reached"
    assert np.array_equal(res["index"], ref["index"]) and np.array_equal(cum, ref["cum"])


def test_group_errors_are_stage_tagged():
    p = T.make_params(9, 5, 5, samples=4, per_block=2, block_width=12)
    with T.Group(devices=[0, 0], ops=_fake_ops()) as g:
        with pytest.raises(T.TxsError, match="set_grid"):
            g.run_pipeline(p)
        with pytest.raises(T.TxsError, match="host exchange only"):
            g.set_exchange("p2p")
    with T.Group(devices=[0, 0, 0], ops=_fake_ops()) as g:
        with pytest.raises(T.TxsError, match="block rows"):
            g.set_grid(20, 50, p)        # 2 block rows of 12 posts, 3 ranks
