import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2006_16783_b200 as T
from paper_2006_16783_b200.configs import Config, params_for, run, setup_terrain
# (run by tests/test_gpu_parity.py::test_bounds_checked_build_edge_workloads with TXS_CHECKED=1)
# global-path VIX (roi > 142) on a grid whose terrain ends at a 2 MB boundary, viewsheds, both SITE modes, shards
cfgs = [Config("m1", 1024, 1024, 0.6, 0, 3000, 150, 20, 6, 128, 4, 1.0, 64, 3, 4),
        Config("m2", 700, 512, 0.5, 0, 4000, 60, 10, 8, 64, 3, 0.95, 0, 5, 6),
        Config("m3", 512, 512, 0.5, 0, 4000, 250, 50, 0, 0, 0, 1.0, 40, 8, 9, random_observers=3000, observer_seed=1)]
with T.Engine(0) as e:
    for cfg in cfgs:
        setup_terrain(e, cfg)
        for mode in (0, 1):
            res = run(e, cfg, params_for(cfg, mode))
            e.cumulative()
            wins, words, pops = e.viewsheds(cfg.roi, 0, min(50, len(res["index"]) + 1))
        print(cfg.name, len(res["index"]), res["stop"])
from paper_2006_16783_b200.shard import LocalComm, run_sharded
engs = [T.Engine(0) for _ in range(3)]
r = run_sharded([(x, k) for k, x in enumerate(engs)], LocalComm(), cfgs[1], params_for(cfgs[1]), 3)
print("sharded", len(r["index"]))
