"""gpurun_out/counts_<cfg>.csv (kernel_counts.sh) -> profiles/kernel_counts.json:
per config and kernel the per-launch ncu counters bench.py's roofline uses
(warp instructions issued, DRAM bytes, L2 read bytes from L1/TEX, duration).
  python profiles/scripts/counts_summary.py c1 c2 c3 c4 c5"""
import csv
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "sector": 1, "inst": 1,
        "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1, "%": 1, "": 1}
KEY = {"gpu__time_duration.sum": "ns", "smsp__inst_executed.sum": "inst", "dram__bytes_read.sum": "dram_read",
       "dram__bytes_write.sum": "dram_write", "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
       "lts__t_sectors_srcunit_tex_op_write.sum": "l2_write_sectors",
       "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct"}
path = os.path.join(P, "kernel_counts.json")
out = json.load(open(path)) if os.path.exists(path) else {}
for cfg in sys.argv[1:]:
    raw = open(os.path.join(G, f"counts_{cfg}.csv")).read()
    rows = list(csv.reader(io.StringIO("\n".join(l for l in raw.splitlines() if l.startswith('"')))))
    hdr, data = rows[0], rows[1:]
    ik, iid, im, iv, iu = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    for r in data:
        name = re.sub(r"^.*::", "", r[ik].split("(")[0].replace("void ", "")).split("<")[0]
        d = per.setdefault(name, {}).setdefault(r[iid], {})
        try:
            d[KEY.get(r[im], r[im])] = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1)
        except ValueError:
            pass
    res = {}
    for name, launches in per.items():
        # the launch that dominates (the main pass; a few tiny launches share names)
        ids = sorted(launches, key=int)
        if name == "k_vix_lanes" and len(ids) >= 2:   # one_run.py's second VIX pass (crossing statistic cached)
            ids = ids[len(ids) // 2:]
        main = max((launches[i] for i in ids), key=lambda d: d.get("ns", 0))
        e = {k: main.get(k) for k in ("ns", "inst", "dram_read", "dram_write", "l2_read_sectors",
                                      "l2_write_sectors", "issue_active_pct", "sm_throughput_pct")}
        e["dram_bytes"] = (e["dram_read"] or 0) + (e["dram_write"] or 0)
        e["l2_read_bytes"] = 32 * (e["l2_read_sectors"] or 0)
        e["launches_in_capture"] = len(launches)
        res[name] = e
    out[cfg] = res
    print(cfg, {k: (round(v["ns"] / 1e6, 3), v["inst"]) for k, v in res.items()})
out["_source"] = ("ncu --metrics (see profiles/scripts/kernel_counts.sh) --clock-control none over "
                  "profiles/scripts/one_run.py --config <cfg>; per kernel the longest launch's counters")
json.dump(out, open(path, "w"), indent=1, sort_keys=True)
