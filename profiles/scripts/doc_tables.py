"""Fill DESIGN.md's and README.md's round-2 measurement tables from profiles/r02_bench_c*.json
(rows between the table header and the next blank line are replaced).  python profiles/scripts/doc_tables.py"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = {"c1": "c1 1000², R100", "c2": "c2 4096², R200", "c3": "c3 16384², R100 (default)", "c4": "c4 46400², R100",
         "c5": "c5 16384², R250, 1M obs."}
README = {"c1": "c1 1000², R100, 1k candidates", "c2": "c2 4096², R200, 16k candidates",
          "c3": "c3 16384², R100, 131k candidates (bench default)", "c4": "c4 46400² (4.3 GB), R100, 215k candidates",
          "c5": "c5 16384², R250, 1M random observers"}
d_rows, r_rows = [], []
for c in NAMES:
    j = json.loads(open(os.path.join(ROOT, "profiles", f"r02_bench_{c}.json")).read())
    st, cb = j["stages"], j.get("cpu_baseline", {})
    ss = st.get("site_stream", {})
    diff = 0
    for v in j.get("differing_bits", {}).values():
        if isinstance(v, dict):
            diff += sum(int(v.get(k, 0)) for k in ("bits_differing", "cum_bits_differing", "scores_differing", "posts_differing"))
    full = cb.get("sample", "").startswith("VIX in full") and "VIEWSHED in full" in cb.get("sample", "")
    cpu = f"{cb.get('value', 0):.3g} s ({'full' if full else 'sampled'})"
    vix = f"{st['vix']['ms']:.1f}" if "vix" in st else "—"
    stream = f"{ss['kernel_gbs'] / 1e3:.2f} TB/s ({100 * ss['kernel_frac_of_hbm']:.1f} %)" if ss.get("kernel_gbs") and c != "c1" else "—"
    d_rows.append(f"| {NAMES[c]} | **{j['value'] * 1e3:.1f}** | {j['e2e']['value'] * 1e3:.1f} | {vix} | {st['viewshed']['ms']:.1f} | "
                  f"{st['site']['ms']:.1f} | {stream} | {cpu} | {diff} |")
    val = f"{j['value'] * 1e3:.1f} ms" if j["value"] < 1 else f"{j['value']:.3f} s"
    e2e = f"{j['e2e']['value'] * 1e3:.1f} ms" if j["e2e"]["value"] < 1 else f"{j['e2e']['value']:.3f} s"
    r_rows.append(f"| {README[c]} | {val} | {e2e} | {cb.get('value', 0):.3g} s ({'full' if full else 'sampled, extrapolated'}) |")


def fill(path, header_re, rows):
    s = open(path).read()
    m = re.search(header_re + r"\n(\|[-| ]+\|\n)", s)
    start = m.end()
    end = s.index("\n\n", start) + 1
    open(path, "w").write(s[:start] + "\n".join(rows) + "\n" + s[end:])


fill(os.path.join(ROOT, "DESIGN.md"), r"\| config \| pipeline \(`value`\) \| e2e \|[^\n]*", d_rows)
fill(os.path.join(ROOT, "README.md"), r"\| config \| pipeline \| e2e[^\n]*", r_rows)
print("\n".join(d_rows + r_rows))
