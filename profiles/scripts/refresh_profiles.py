"""Copy a round_profile.sh run from gpurun_out/ into profiles/: the c2 launch
list summary, the ncu --set full summary of the top kernels and their DRAM
traffic per launch (profiles/ncu_traffic.json).  python profiles/scripts/refresh_profiles.py"""
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

raw = open(os.path.join(G, "launches_c2.csv")).read()
rows = list(csv.reader(io.StringIO("\n".join(l for l in raw.splitlines() if l.startswith('"')))))
hdr, data = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg, tot = collections.OrderedDict(), 0.0
for r in data:
    name = re.sub(r"^.*::", "", r[ik].split("(")[0].replace("void ", ""))
    v, u = float(r[iv].replace(",", "")), r[iu]
    ms = v / 1e6 if u == "ns" else v / 1e3 if u in ("us", "usecond") else v if u in ("ms", "msecond") else v / 1e6
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ms
    tot += ms
out = ["# c2 launch list (ncu --metrics gpu__time_duration.sum --clock-control none; bench.py --steps 1 --warmup 3 "
       "--no-cpu-baseline --e2e-steps 1)",
       "# cold-cache serialised per-launch times over the whole command (warm-up, timed step, e2e, site_stream): "
       "compare SHARES, not absolutes",
       f"# {len(data)} launches, {tot:.1f} ms total", "kernel,launches,total_ms,share"]
for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k.replace(',', ';')},{c},{ms:.3f},{ms / tot:.4f}")
open(os.path.join(P, "r01_launches_c2.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[2:8]))

summ = subprocess.run(["python", os.path.join(P, "scripts", "ncu_summary.py"), os.path.join(G, "prof_c2.ncu-rep")],
                      capture_output=True, text=True).stdout
open(os.path.join(P, "r01_ncu_full_c2.csv"), "w").write(summ)
rows = list(csv.reader(io.StringIO(summ)))
tr = json.load(open(os.path.join(P, "ncu_traffic.json")))


def to_bytes(v, key):
    v = float(v)
    return v * 1e9 if "Gbyte" in key else v * 1e6 if "Mbyte" in key else v * 1e3 if "Kbyte" in key else v


for row in rows[1:]:
    x = dict(zip(rows[0], row))
    kr = next(k for k in x if k.startswith("dram__bytes_read"))
    kw = next(k for k in x if k.startswith("dram__bytes_write"))
    try:
        b = int(to_bytes(x[kr], kr) + to_bytes(x[kw], kw))
    except ValueError:
        continue
    for kern in ("k_vix_quads", "k_site_loop"):
        if kern in row[0]:
            tr[kern] = b
    print(row[0], b)
json.dump(tr, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
