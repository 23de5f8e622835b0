"""One VIX stage on a BASELINE config (for ncu captures of k_vix_quads):
python profiles/scripts/vix_once.py c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_16783_b200 import Engine  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
e = Engine()
setup_terrain(e, cfg)
e.estimate_vix(params_for(cfg), copy=False)
e.synchronize()
print("ms_vix", e.stats()["ms_vix"])
