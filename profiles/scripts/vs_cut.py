"""VIEWSHED A/B on one resident configuration: the sweep with and without the
horizon cut-off (TXS_VS_CUT), alternating, device-timed (stage + sweep
kernel), with the fraction of events cut and a check that both variants give
identical popcounts.   python vs_cut.py c5 [reps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1"]
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    p = params_for(cfg)
    if cfg.random_observers:
        e.random_observers(cfg.random_observers, cfg.observer_seed)
    else:
        e.estimate_vix(p, copy=False)
        e.find_candidates(p, copy=False)
    pops = {}
    for r in range(reps):
        for v in variants:
            os.environ["TXS_VS_CUT"] = v
            e.reset_stats()
            e.compute_all_viewsheds(p)
            st = e.stats()
            n = st["candidates"]
            total = st["viewshed_crossings"] + st["viewshed_cells"]
            print(f"{cfg.name} cut={v} stage {st['ms_viewshed']:.2f} ms kernel {st['ms_viewshed_kernel']:.2f} ms "
                  f"events_cut {st['viewshed_events_cut']} ({st['viewshed_events_cut'] / max(1, total):.3f} of "
                  f"{total} real events, incl. padding)", flush=True)
            if r == 0:
                _, _, pc = e.viewsheds(cfg.roi, 0, min(n, 200000))
                pops[v] = pc
    ref = pops[variants[0]]
    print("popcounts identical:", all(np.array_equal(ref, x) for x in pops.values()))
