"""One VIEWSHED stage on a BASELINE config (for ncu captures): python profiles/scripts/vs_once.py c5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
e = Engine()
setup_terrain(e, cfg)
p = params_for(cfg)
if cfg.random_observers:
    e.random_observers(cfg.random_observers, cfg.observer_seed)
else:
    e.estimate_vix(p, copy=False)
    e.find_candidates(p, copy=False)
e.compute_all_viewsheds(p)
e.synchronize()
print("ms_viewshed", e.stats()["ms_viewshed"])
