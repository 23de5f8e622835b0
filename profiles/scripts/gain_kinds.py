"""SITE streaming gain pass: every kernel form (TXS_GAIN_PASS=full|tiled|strips|t8)
on a BASELINE config, timed alone (txs_time_gain_pass) and checked by running
64 full-rescan SITE rounds with it against the incremental SITE's picks.
python profiles/scripts/gain_kinds.py c3 [kinds...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine, make_params  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
kinds = sys.argv[2:] or ["full", "tiled", "strips", "t8"]
e = Engine()
setup_terrain(e, cfg)
p0 = params_for(cfg)
if cfg.random_observers:
    e.random_observers(cfg.random_observers, cfg.observer_seed)
else:
    e.estimate_vix(p0, copy=False)
    e.find_candidates(p0, copy=False)
e.compute_all_viewsheds(p0)
def capped(mode):
    return make_params(cfg.roi, cfg.height, cfg.height, samples=max(cfg.samples, 1), per_block=max(cfg.per_block, 1),
                       block_width=cfg.block, target=cfg.target, max_selected=64, seed=cfg.vix_seed, site_mode=mode)


ref = e.site(capped(0), cap=65)
p1 = capped(1)
for k in kinds:
    os.environ["TXS_GAIN_PASS"] = k
    r = e.site(p1, cap=65)
    n = min(64, len(ref["index"]), len(r["index"]))
    same = np.array_equal(np.asarray(ref["index"][:n]), np.asarray(r["index"][:n]))
    e.site(p0, cap=(cfg.max_selected or 64) + 1)   # a realistic cum for the timing
    ms, b = e.time_gain_pass(16)
    print(f"{cfg.name} {k:7s} picks_equal={same} ({n}) gain pass {ms:.4f} ms, {b / (ms / 1e3) / 1e12:.3f} TB/s", flush=True)
