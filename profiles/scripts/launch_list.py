"""ncu launch list CSV (--metrics gpu__time_duration.sum) -> per-kernel totals and
shares.  python profiles/scripts/launch_list.py gpurun_out/launches_c3.csv "header" > out.txt"""
import collections
import csv
import io
import sys

raw = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO("\n".join(l for l in raw.splitlines() if l.startswith('"')))))
hdr, data = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in data:
    name = r[ik].split("(")[0].replace("void ", "")
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[iu], 1)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(sys.argv[2] if len(sys.argv) > 2 else "per kernel total ns, launches, share")
for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ns:14.0f} ns {c:5d} {100 * ns / tot:6.1f}%  {k}")
