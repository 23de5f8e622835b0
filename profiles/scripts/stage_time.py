"""Time single stages on a BASELINE configuration (device-side stage timers of
the C-ABI): python profiles/scripts/stage_time.py c2 vix [reps].  Used for
kernel A/B measurements (TXS_VIX_PATH / TXS_VS_K env overrides)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
stages = sys.argv[2].split(",")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
e = Engine()
setup_terrain(e, cfg)
p = params_for(cfg)
out = {}
for st in stages:
    ts = []
    for _ in range(reps + 1):
        e.reset_stats()
        if st == "vix":
            e.estimate_vix(p, copy=False)
        elif st == "viewshed":
            if cfg.random_observers:
                e.random_observers(cfg.random_observers, cfg.observer_seed)
            else:
                e.estimate_vix(p, copy=False)
                e.find_candidates(p, copy=False)
            e.reset_stats()
            e.compute_all_viewsheds(p)
        elif st == "site":    # incremental SITE (mode 0), the config's stop rules
            if _ == 0:
                if cfg.random_observers:
                    e.random_observers(cfg.random_observers, cfg.observer_seed)
                else:
                    e.estimate_vix(p, copy=False)
                    e.find_candidates(p, copy=False)
                e.compute_all_viewsheds(p)
            e.reset_stats()
            e.site(p, cap=cfg.max_selected + 1 if cfg.max_selected > 0 else 1 << 20)
        elif st == "site1":   # full-rescan SITE, 64 rounds (the streaming figure)
            if _ == 0:
                if cfg.random_observers:
                    e.random_observers(cfg.random_observers, cfg.observer_seed)
                else:
                    e.estimate_vix(p, copy=False)
                    e.find_candidates(p, copy=False)
                e.compute_all_viewsheds(p)
            e.reset_stats()
            p1 = params_for(cfg, site_mode=1)
            p1.max_selected = 64
            e.site(p1, cap=65)
        e.synchronize()
        s = e.stats()
        ts.append(s["ms_" + st.rstrip("1")])
        if st == "site1":
            out["site1_gbs"] = round(s["site_bytes"] / (s["ms_site"] / 1e3) / 1e9, 1)
            out["site1_rounds_ms"] = round(s["ms_site_rounds"], 3)
            out["site1_rounds_gbs"] = round(s["site_bytes"] / (s["ms_site_rounds"] / 1e3) / 1e9, 1)
    out[st] = min(ts[1:])
print(sys.argv[1], os.environ.get("TXS_VIX_PATH", ""), os.environ.get("TXS_VS_K", ""), out, flush=True)
