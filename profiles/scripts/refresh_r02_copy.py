"""Copy a refresh_r02.sh (+ vs_ncu.sh) run from gpurun_out/ into profiles/ as the round-2 evidence:
per-config counters (+ kernel_counts.json), the c3 launch list, ncu --set full summaries of the top
kernels, ncu_traffic.json, the five bench lines and the reference arm.
  python profiles/scripts/refresh_r02_copy.py"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G, P, S = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles"), os.path.join(ROOT, "profiles", "scripts")


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


cfgs = [c for c in ("c1", "c2", "c3", "c4", "c5") if os.path.exists(os.path.join(G, f"counts_{c}.csv"))]
print(run(os.path.join(S, "counts_summary.py"), *cfgs))
for c in cfgs:
    shutil.copy(os.path.join(G, f"counts_{c}.csv"), os.path.join(P, f"r02_counts_{c}.csv"))
open(os.path.join(P, "r02_launches_c3.txt"), "w").write(run(os.path.join(S, "launch_list.py"), os.path.join(G, "launches_c3.csv")))
for src, dst in (("r02_vix_c3.ncu-rep", "r02_ncu_full_c3_vix.csv"),):
    if os.path.exists(os.path.join(G, src)):
        open(os.path.join(P, dst), "w").write(run(os.path.join(S, "ncu_summary.py"), os.path.join(G, src)))
for src, dst in (("gain_c3_t8.csv", "r02_ncu_full_c3_gain_t8.csv"), ("gain_c3_full.csv", "r02_ncu_full_c3_gain_rows.csv"),
                 ("gain_c4_t8.csv", "r02_ncu_full_c4_gain_t8.csv"), ("r02_vs_c5.csv", "r02_ncu_full_c5_viewshed.csv"),
                 ("r02_vs_c3.csv", "r02_ncu_full_c3_viewshed.csv"), ("batch_launches_c3.csv", "r02_batch_site_launches_c3.csv"),
                 ("batch_launches_c5.csv", "r02_batch_site_launches_c5.csv")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
for c in ("c1", "c2", "c3", "c4", "c5"):
    f = os.path.join(G, f"final_bench_{c}.log")
    if os.path.exists(f):
        lines = [l for l in open(f) if l.startswith("{")]
        if lines:
            open(os.path.join(P, f"r02_bench_{c}.json"), "w").write(lines[-1])
            j = json.loads(lines[-1])
            print(c, j["value"], j["e2e"]["value"], {k: v["ms"] for k, v in j["stages"].items() if "ms" in v},
                  j.get("cpu_baseline", {}).get("value"), j.get("differing_bits", {}).get("site"))
f = os.path.join(G, "final_ref_c3.log")
if os.path.exists(f):
    lines = [l for l in open(f) if l.startswith("{")]
    if lines:
        open(os.path.join(P, "r02_bench_reference_c3.json"), "w").write(lines[-1])
        print("reference", json.loads(lines[-1]).get("value"))
