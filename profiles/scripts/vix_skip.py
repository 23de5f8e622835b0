"""A/B of the VIX skip map (TXS_VIX_SKIP=0 full walk / 1 flattened / 2 per-segment): device time of the VIX stage
(min of reps) and a bit-exact comparison of the two VixMaps, per config.
python profiles/scripts/vix_skip.py c1,c2,c3 [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for name in sys.argv[1].split(","):
    cfg = CONFIGS[name]
    e = Engine()
    setup_terrain(e, cfg)
    p = params_for(cfg)
    res, maps = {}, {}
    modes = ("0", "1", "2")
    for skip in modes:
        os.environ["TXS_VIX_SKIP"] = skip
        ts = []
        for k in range(reps + 1):
            e.reset_stats()
            v = e.estimate_vix(p, copy=(k == 0))
            if k == 0:
                maps[skip] = v
            e.synchronize()
            ts.append(e.stats()["ms_vix"])
        res[skip] = min(ts[1:])
    same = all(np.array_equal(maps["0"], maps[m]) for m in modes)
    print(f"{name}: full {res['0']:.2f} ms  flattened skip {res['1']:.2f} ms  per-segment skip {res['2']:.2f} ms  "
          f"identical={same}", flush=True)
    assert same
    e.close()
