"""A/B of the full-rescan gain pass kernels on one resident configuration:
runs the config's pipeline once, then times txs_time_gain_pass (CUDA events,
8 passes) under each TXS_GAIN_* variant.   python gain_variants.py c3 [variants...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, run, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
variants = sys.argv[2:] or ["reg", "25", "26", "28", "45", "46", "48", "85"]
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    ref = run(e, cfg, params_for(cfg))
    for rep in range(2):
        for v in variants:
            for k in ("TXS_GAIN_REG", "TXS_GAIN_LEAN", "TXS_GAIN_V2", "TXS_GAIN_TILED_SMALL", "TXS_GAIN_REGION"):
                os.environ.pop(k, None)
            if v.startswith("rg"):
                os.environ["TXS_GAIN_REGION"] = v[2:]
            if v == "small":
                os.environ["TXS_GAIN_TILED_SMALL"] = "1"
            if v == "reg":
                os.environ["TXS_GAIN_REG"] = "1"
            elif v.startswith("v"):
                os.environ["TXS_GAIN_V2"] = v[1:]
            elif v != "default":
                os.environ["TXS_GAIN_LEAN"] = v
            ms, b = e.time_gain_pass(8)
            check = ""
            if rep == 0:   # mode-1 SITE (the gain pass every round) must pick what the incremental SITE picks
                p1 = params_for(cfg, 1)
                p1.max_selected = 48
                r1 = e.site(p1, cap=49)
                check = " picks " + ("ok" if np.array_equal(r1["index"], ref["index"][:len(r1["index"])]) else "DIFFER")
            print(f"{cfg.name} {v:8s} {ms:.4f} ms/pass {b / ms / 1e6:.1f} GB/s{check}", flush=True)
