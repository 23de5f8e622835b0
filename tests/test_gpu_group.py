"""Native multi-GPU group (txs_group_*, csrc/group.cu) on the B200: N row-band
contexts in one process, SITE rounds exchanged over peer memory (P2P mailboxes
read by a select kernel, multi-device CUDA graph of 16 rounds), NCCL
(ncclCommInitAll + one allgather per round) or the host.  The pool exposes one
GPU, so several ranks share device 0 ("virtual ranks": the same kernels, peer
pointers that happen to be local, cross-stream event ordering); every variant
must reproduce the single-context pick sequence and cumulative bitmap exactly
(SPEC.md:372,395), which the single context itself matches against the oracle
(test_gpu_parity.py)."""
import numpy as np
import pytest

import paper_2006_16783_b200 as T
from paper_2006_16783_b200.configs import CONFIGS, params_for

pytestmark = pytest.mark.gpu


def _single(nr, nc, rough, tseed, p, water=0, observers=None, zmax=4000):
    with T.Engine(0) as e:
        e.generate_fractal(nr, nc, rough, tseed, 0, zmax)
        if water:
            e.fill_rows(0, water, 0)
        if observers:
            e.random_observers(*observers)
            e.compute_all_viewsheds(p)
            res = e.site(p)
        else:
            res = e.run_pipeline(p)
        return res, e.cumulative()


def _group(devs, xchg, nr, nc, rough, tseed, p, water=0, observers=None, zmax=4000):
    with T.Group(devices=devs, exchange=xchg) as g:
        g.set_grid(nr, nc, p)
        g.generate_fractal(rough, tseed, 0, zmax)
        if water:
            g.fill_rows(0, water, 0)
        if observers:
            g.random_observers(*observers)
        res = g.run_pipeline(p)
        return res, g.cumulative()


def _same(a, b):
    ra, ca = a
    rb, cb = b
    assert ra["stop"] == rb["stop"]
    for k in ("index", "row", "col", "gain"):
        assert np.array_equal(ra[k], rb[k]), k
    assert np.array_equal(ra["coverage"], rb["coverage"])
    assert np.array_equal(ca, cb)


@pytest.mark.parametrize("devs,xchg", [([0], "p2p"), ([0, 0], "p2p"), ([0, 0, 0], "p2p"), ([0, 0, 0, 0], "p2p"),
                                       ([0, 0], "host"), ([0, 0, 0], "host"), ([0], "nccl"), ([0], "replicate"),
                                       ([0, 0, 0], "replicate")])
def test_group_matches_single_context(devs, xchg):
    p = T.make_params(30, 10, 10, samples=8, per_block=6, block_width=40, target=0.9, max_selected=120, seed=5)
    ref = _single(480, 400, 0.5, 3, p)
    assert len(ref[0]["index"]) > 40
    _same(_group(devs, xchg, 480, 400, 0.5, 3, p), ref)


@pytest.mark.parametrize("devs,xchg", [([0, 0], "p2p"), ([0, 0, 0], "p2p"), ([0, 0], "replicate"),
                                       ([0, 0, 0, 0], "replicate")])
def test_group_random_observers_and_water(devs, xchg):
    p = T.make_params(40, 20, 10, target=1.0, max_selected=200, block_width=48)
    ref = _single(512, 448, 0.6, 8, p, water=60, observers=(3000, 17))
    _same(_group(devs, xchg, 512, 448, 0.6, 8, p, water=60, observers=(3000, 17)), ref)


def test_group_config2_four_ranks():
    """BASELINE config 2 (4096^2, R200, 16384 candidates, 1024 picks max) on 4
    row bands, exchanging winners over peer memory or gathering the viewsheds
    once (replicated SITE) == the single context."""
    cfg = CONFIGS["c2"]
    p = params_for(cfg)
    ref = _single(cfg.nrows, cfg.ncols, cfg.roughness, cfg.terrain_seed, p, zmax=cfg.zmax)
    for xchg in ("p2p", "replicate"):
        got = _group([0, 0, 0, 0], xchg, cfg.nrows, cfg.ncols, cfg.roughness, cfg.terrain_seed, p, zmax=cfg.zmax)
        _same(got, ref)
        assert got[0]["stage_ms"]["site"] > 0


def test_group_rejects_bad_use():
    p = T.make_params(30, 10, 10, block_width=40)
    with T.Group(devices=[0, 0]) as g:
        with pytest.raises(T.TxsError, match="NCCL needs one rank per device"):
            g.set_exchange("nccl")
        with pytest.raises(T.TxsError, match="block rows"):
            T.Group(devices=[0] * 5).set_grid(120, 100, p)   # 3 block rows, 5 ranks
        g.set_grid(200, 100, p)
        g.generate_fractal(0.5, 1, 0, 1000)
        with pytest.raises(T.TxsError, match="roi"):
            g.run_pipeline(T.make_params(31, 10, 10, block_width=40))
