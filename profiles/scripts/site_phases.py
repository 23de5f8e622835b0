"""Per-phase device time of the one-barrier persistent SITE loop (k_site_loop1,
CTA 0's %globaltimer, TXS_SITE_PROFILE=1) on a BASELINE config:
    python site_phases.py c3"""
import os
import sys

os.environ["TXS_SITE_PROFILE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, run, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    p = params_for(cfg)
    for rep in range(3):
        e.reset_stats()
        res = run(e, cfg, p)
        st = e.stats()
        n = len(res["index"])
        ph = st["site_phase_ns"]
        names = ["winner", "commit", "update", "partial", "barrier"]
        tot = sum(ph)
        print(f"{cfg.name}: {n} rounds, SITE {st['ms_site']:.2f} ms, loop {tot / 1e6:.2f} ms, per round "
              + " ".join(f"{k} {v / max(1, n) / 1e3:.2f}us" for k, v in zip(names, ph)), flush=True)
