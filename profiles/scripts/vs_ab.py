"""VIEWSHED A/B on one resident configuration: each variant is a set of
environment overrides ("K=V;K2=V2", "-" for none), timed device-side (stage +
sweep kernel), popcounts checked identical across variants.
    python vs_ab.py c5 "-" "TXS_VS_UNIFORM=1" "TXS_VS_UNIFORM=1;TXS_VS_K=3" """
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
variants = sys.argv[2:] or ["-"]
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    p = params_for(cfg)
    if cfg.random_observers:
        e.random_observers(cfg.random_observers, cfg.observer_seed)
    else:
        e.estimate_vix(p, copy=False)
        e.find_candidates(p, copy=False)
    ref = None
    keys = set()
    for v in variants:
        for kv in v.split(";"):
            if "=" in kv:
                keys.add(kv.split("=")[0])
    for rep in range(2):
        for v in variants:
            for k in keys:
                os.environ.pop(k, None)
            for kv in v.split(";"):
                if "=" in kv:
                    k, val = kv.split("=")
                    os.environ[k] = val
            e.reset_stats()
            e.compute_all_viewsheds(p)
            st = e.stats()
            ok = ""
            if rep == 0:
                _, _, pc = e.viewsheds(cfg.roi, 0, min(st["candidates"], 100000))
                if ref is None:
                    ref = pc
                ok = "popcounts " + ("identical" if np.array_equal(ref, pc) else "DIFFER")
            print(f"{cfg.name} [{v}] stage {st['ms_viewshed']:.2f} ms kernel {st['ms_viewshed_kernel']:.2f} ms "
                  f"ties {st['vs_fp64_ties']} {ok}", flush=True)
