"""One siting run of a BASELINE config (plus one full-rescan gain pass), the
command profiles/scripts/kernel_counts.sh runs under ncu to record the main
kernels' per-launch counters for bench.py's roofline (profiles/kernel_counts.json).
  python profiles/scripts/one_run.py --config c3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, run, setup_terrain  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--l2", action="store_true", help="also measure the L2-resident read bandwidth (sizes sweep)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    p = params_for(cfg)
    if cfg.samples:   # the crossing statistic is counted on the first VIX launch per key and cached: the counters
        e.estimate_vix(p, copy=False)   # recorded for k_vix_lanes are the cached form's (the one the bench times)
    res = run(e, cfg, p)
    ms, b = e.time_gain_pass(1)
    st = e.stats()
    print(f"{cfg.name}: sited {len(res['index'])} stop {res['stop']} vix_kernel {st['ms_vix_kernel']:.2f} ms "
          f"vs_kernel {st['ms_viewshed_kernel']:.2f} ms gain pass {ms:.3f} ms {b} B", flush=True)
    if a.l2:
        for mb in (8, 16, 24, 32, 48, 64, 96):
            print(f"l2_read {mb} MB: {e.measure_l2(mb << 20, 40):.1f} GB/s", flush=True)
