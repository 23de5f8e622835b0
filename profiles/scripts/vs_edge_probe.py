"""How much of C5's VIEWSHED time do the CTAs with observers near the grid edge
take?  Times compute_all_viewsheds for (a) the C5 observers, (b) the same
observers clamped into the interior, (c) only the C5 observers within roi+1 of
an edge.   python profiles/scripts/vs_edge_probe.py [c5]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
R = cfg.roi
e = Engine()
setup_terrain(e, cfg)
p = params_for(cfg)
e.random_observers(cfg.random_observers, cfg.observer_seed)
rows, cols, _ = e.candidates()
edge = (rows < R + 1) | (rows > cfg.nrows - R - 2) | (cols < R + 1) | (cols > cfg.ncols - R - 2)


def t(r, c, label):
    e.set_candidates(r, c)
    best = 1e30
    for _ in range(3):
        e.reset_stats()
        e.compute_all_viewsheds(p)
        e.synchronize()
        best = min(best, e.stats()["ms_viewshed_kernel"])
    print(f"{label}: {len(r)} observers, sweep kernel {best:.1f} ms ({best / len(r) * 1e6:.1f} ns/observer)", flush=True)


t(rows, cols, "c5 observers")
t(np.clip(rows, R + 1, cfg.nrows - R - 2), np.clip(cols, R + 1, cfg.ncols - R - 2), "clamped interior")
t(rows[edge], cols[edge], f"edge only ({edge.mean() * 100:.1f} %)")
