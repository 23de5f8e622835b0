"""Multi-rank row-band orchestration (paper_2006_16783_b200/shard.py) across
two real processes over torch.distributed gloo, each driving two bands with
the oracle-backed fake engine; the SITE sequence and cumulative bitmap must
equal the single-process oracle pipeline bit for bit."""
import os
import socket

import numpy as np
import pytest

import oracle_lib as O

NB = 4   # bands; 2 processes x 2 bands


def _cfgs():
    from paper_2006_16783_b200.configs import Config
    return {
        "findmax": Config("t1", 240, 200, 0.5, 0, 4000, 12, 10, 8, 30, 3, 0.97, 0, 7, 3),
        "observers": Config("t2", 200, 170, 0.6, 0, 3000, 10, 10, 0, 0, 0, 1.0, 25, 9, 4,
                            random_observers=300, observer_seed=11),
    }


def _params(cfg):
    from paper_2006_16783_b200.configs import params_for
    return params_for(cfg)


def _oracle(cfg):
    z = O.generate_fractal(cfg.nrows, cfg.ncols, cfg.roughness, cfg.terrain_seed, cfg.zmin, cfg.zmax)
    if cfg.random_observers:
        rows, cols = O.random_observers(cfg.nrows, cfg.ncols, cfg.random_observers, cfg.observer_seed)
    else:
        s = O.estimate_vix(z, cfg.roi, cfg.height, cfg.height, cfg.samples, cfg.vix_seed)
        rows, cols, _ = O.find_candidates(s, cfg.block, cfg.per_block)
    w, v = O.viewsheds(z, cfg.roi, cfg.height, cfg.height, rows, cols)
    return O.site(rows, cols, w, v, cfg.nrows, cfg.ncols, cfg.target, cfg.max_selected)


def _worker(rank, world, port, name, out):
    import torch.distributed as dist
    from fake_engine import FakeShardEngine
    from paper_2006_16783_b200.shard import TorchComm, run_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = _cfgs()[name]
    ranks = [(FakeShardEngine(), b) for b in range(rank * NB // world, (rank + 1) * NB // world)]
    res = run_sharded(ranks, TorchComm("cpu"), cfg, _params(cfg), NB)
    np.savez(os.path.join(out, f"r{rank}.npz"), index=res["index"], gain=res["gain"], cum=res["cum"],
             row=res["row"], col=res["col"], stop=np.array(res["stop"]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_bands():
    from paper_2006_16783_b200.shard import plan_bands
    # config 4: 116 block rows -> 15,15,15,15,14,14,14,14
    assert plan_bands(46400, 400, 8) == [(0, 6000), (6000, 12000), (12000, 18000), (18000, 24000),
                                        (24000, 29600), (29600, 35200), (35200, 40800), (40800, 46400)]
    assert plan_bands(1000, 100, 8)[-1] == (900, 1000)
    with pytest.raises(ValueError):           # a rank without a band is refused
        plan_bands(100, 100, 3)
    for nr, b, w in [(4096, 128, 8), (16384, 256, 5), (1000, 7, 6)]:
        bands = plan_bands(nr, b, w)
        assert bands[0][0] == 0 and bands[-1][1] == nr
        assert all(x[1] == y[0] for x, y in zip(bands, bands[1:]))
        assert all(x[0] % b == 0 for x in bands)


@pytest.mark.parametrize("name", ["findmax", "observers"])
def test_two_process_gloo_bit_exact(tmp_path, name):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2, join=True)
    exp = _oracle(_cfgs()[name])
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(got["index"], exp["index"])
        assert np.array_equal(got["gain"], exp["gain"])
        assert np.array_equal(got["row"], exp["row"]) and np.array_equal(got["col"], exp["col"])
        assert str(got["stop"]) == exp["stop"]
        assert np.array_equal(got["cum"], exp["cum"])
