"""Summarise ncu outputs into profiles/ (tracked):
  launches csv (--metrics gpu__time_duration.sum)  -> per-kernel share table
  full capture (.ncu-rep)                           -> per-kernel metric table + ncu_summary.json
usage: python tools/ncu_summary.py <tag> <scene> <launches.csv> <prof.ncu-rep>"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

tag, scene, launches, rep = sys.argv[1:5]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out, exist_ok=True)

# ---- launch list
text = open(launches).read()
start = text.find('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
total = 0.0
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    t = float(r[vi].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
    total += t
lines = [f"# {tag}: kernel launch list of `python bench.py --config {scene} --steps 2 --warmup 1` under",
         "`ncu --metrics gpu__time_duration.sum --clock-control none` (YS_PCG_GRAPH=none: the same kernels",
         "launched directly, because ncu cannot see kernel nodes of a conditional graph).",
         "Per-launch times are cold-cache and serialised; compare shares, not absolutes.", "",
         "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| `{name}` | {n} | {t/1e6:.3f} | {100*t/total:.1f}% |")
open(os.path.join(out, f"{tag}_launches_{scene}.md"), "w").write("\n".join(lines) + "\n")

# ---- full capture
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
want = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
        ("launch__registers_per_thread", "")]
idx = {w: h.index(w) for w, _ in want if w in h}
per = collections.OrderedDict()
for r in rr[2:]:
    name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "")
    per.setdefault(name, []).append({w: float(r[i].replace(",", "")) for w, i in idx.items()})
tl = [f"# {tag}: `ncu --set full --clock-control none` of the top kernels, scene {scene}",
      f"(command: `YS_PCG_GRAPH=none ncu --set full ... python tools/prof_driver.py {scene}`; mean over captured launches)", "",
      "| kernel | n | time us | DRAM rd MB | DRAM wr MB | DRAM % | L1 % | L2 % | warps % | FP64 pipe % | regs |",
      "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
summary = {}
for name, lst in per.items():
    m = {w: sum(d[w] for d in lst) / len(lst) for w in idx}
    tl.append(f"| `{name}` | {len(lst)} | " + " | ".join(
        f"{m.get(w, float('nan')):.1f}" for w, _ in want) + " |")
    summary[name] = {k: v for k, v in m.items()}
open(os.path.join(out, f"{tag}_ncu_top_{scene}.md"), "w").write("\n".join(tl) + "\n")
js = os.path.join(out, "ncu_summary.json")
d = json.load(open(js)) if os.path.exists(js) else {}
sp = [v for k, v in summary.items() if k.startswith("k_spmv33")]
d[scene] = {"tag": tag, "kernels": summary}
if sp:
    d[scene]["spmv_dram_bytes"] = 1e6 * (sp[0]["dram__bytes_read.sum"] + sp[0]["dram__bytes_write.sum"])
json.dump(d, open(js, "w"), indent=1)
print("\n".join(lines[:16]))
print("\n".join(tl))
