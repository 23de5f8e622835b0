"""Per-source-line instruction counts and stall samples from an ncu report
(`ncu -i REP --page source --csv --print-source=cuda,sass`): the CUDA source
lines ranked by warp instructions executed.
  python profiles/scripts/src_hotspots.py gpurun_out/vix_c3.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and r[2] == "-":     # a CUDA line aggregate (Address '-')
        d = dict(zip(hdr[4:], r[4:]))
        try:
            rows.append((int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"]), fname,
                         int(r[0]), r[1].strip()))
        except (KeyError, ValueError):
            pass
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
print("inst%   stall%  file:line  source")
for i, smp, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * i / tot_i:5.1f}  {100 * smp / tot_s:5.1f}  {f}:{ln}  {src[:110]}")
