"""SITE streaming gain pass on a BASELINE config after its incremental SITE
(for ncu captures of k_gain_full / k_gain_tiled): python profiles/scripts/gain_once.py c3"""
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
e.site(p, cap=(cfg.max_selected or 64) + 1)
ms, b = e.time_gain_pass(16)
print(f"gain pass {ms:.4f} ms, {b / (ms / 1e3) / 1e12:.2f} TB/s")
