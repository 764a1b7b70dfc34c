"""Summarise ncu outputs into profiles/ (tracked):
  launches csv (--metrics gpu__time_duration.sum)  -> per-kernel share table
  full capture (.ncu-rep)                           -> per-kernel metric table + ncu_summary.json
  eval FLOP counts csv (--metrics ...dfma/dadd/dmul)  -> eval_flops_per_step in ncu_summary.json
usage: python tools/ncu_summary.py <tag> <scene> <launches.csv> <prof.ncu-rep> [prof_driver.log] [evalflops.csv]
(the log's "pcg iterations N" line converts the persistent PCG kernel's DRAM bytes to bytes per iteration)"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

tag, scene, launches, rep = sys.argv[1:5]
pcg_iters = None
evalflops = sys.argv[6] if len(sys.argv) > 6 else None
if len(sys.argv) > 5:
    m = re.search(r"pcg iterations (\d+)", open(sys.argv[5]).read())
    pcg_iters = int(m.group(1)) if m else None
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
lines = [f"# {tag}: kernel launch list of `python bench.py --config {scene} --steps 2 --warmup 1 --no-cpu-baseline`",
         "under `ncu --metrics gpu__time_duration.sum --clock-control none`.  The uniform-3x3 PCG is one",
         "cooperative launch per solve (`k_pcg33_stream`); the bench's own kernel-timing hooks",
         "(`ys_time_kernel`: SpMV x50, assembly x10, eval x5) run after the timed steps and appear here too.",
         "Per-launch times are cold-cache and serialised; compare shares, not absolutes.", "",
         "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| `{name}` | {n} | {t/1e6:.3f} | {100*t/total:.1f}% |")
open(os.path.join(out, f"{tag}_launches_{scene}.md"), "w").write("\n".join(lines) + "\n")

# ---- full capture
want = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
        ("launch__registers_per_thread", "")]
# to MB and us whatever unit each report chose for a column
_SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6,
          "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
          "s": 1e6, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
per = collections.OrderedDict()
idx = {}
for one in rep.split(","):  # several captures may be merged
    raw = subprocess.run(["ncu", "-i", one, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    part = list(csv.reader(io.StringIO(raw)))
    if len(part) < 3:
        continue
    h, units = part[0], part[1]
    idx = {w: h.index(w) for w, _ in want if w in h}
    for r in part[2:]:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "")
        vals = {}
        for w, i in idx.items():
            v = float(r[i].replace(",", "") or "nan")
            vals[w] = v * _SCALE.get(units[i], 1.0)
        per.setdefault(name, []).append(vals)
tl = [f"# {tag}: `ncu --set full --clock-control none` of the top kernels, scene {scene}",
      f"(command: `ncu --set full --import-source on ... python tools/prof_driver.py {scene}`; mean over captured launches)", "",
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
def base(k):
    return k.split("::")[-1]


sp = [v for k, v in summary.items() if base(k).startswith("k_spmv_sell")] or \
     [v for k, v in summary.items() if base(k).startswith("k_spmv33")]
prev = d.get(scene, {})
d[scene] = dict(prev, tag=tag, kernels=summary)
if sp:
    d[scene]["spmv_dram_bytes"] = 1e6 * (sp[0]["dram__bytes_read.sum"] + sp[0]["dram__bytes_write.sum"])
pp = [v for k, v in summary.items() if base(k).startswith("k_pcg33_stream") or base(k).startswith("k_pcg33_sell")] or \
     [v for k, v in summary.items() if base(k).startswith("k_pcg33_persistent")]
if pp and pcg_iters:
    d[scene]["pcg_iterations"] = pcg_iters
    d[scene]["pcg_dram_bytes_per_iteration"] = 1e6 * (pp[0]["dram__bytes_read.sum"] +
                                                       pp[0]["dram__bytes_write.sum"]) / pcg_iters
if evalflops and os.path.exists(evalflops):
    t2 = open(evalflops).read()
    rr = list(csv.reader(io.StringIO(t2[t2.find('"ID"'):])))
    h2 = rr[0]
    k2, m2, v2 = h2.index("Kernel Name"), h2.index("Metric Name"), h2.index("Metric Value")
    cnt = collections.Counter()
    for r in rr[1:]:
        if len(r) > v2:
            cnt[r[m2]] += float(r[v2].replace(",", ""))
    dfma = cnt["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
    dadd = cnt["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    dmul = cnt["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    d[scene]["eval_flops_per_step"] = 2 * dfma + dadd + dmul
    d[scene]["eval_fp64_inst"] = {"dfma": dfma, "dadd": dadd, "dmul": dmul}
    with open(os.path.join(out, f"{tag}_eval_flops_{scene}.md"), "w") as f:
        f.write(f"# {tag}: FP64 work of the local evaluation, scene {scene} (one Newton step, every k_eval* launch)\n\n"
                f"`ncu --metrics smsp__sass_thread_inst_executed_op_{{dfma,dadd,dmul}}_pred_on.sum -k regex:k_eval "
                f"python tools/one_step.py {scene} 1`\n\n"
                f"| DFMA | DADD | DMUL | FLOPs (2 DFMA + DADD + DMUL) |\n|---:|---:|---:|---:|\n"
                f"| {dfma:.4g} | {dadd:.4g} | {dmul:.4g} | {2 * dfma + dadd + dmul:.4g} |\n")
json.dump(d, open(js, "w"), indent=1)
print("\n".join(lines[:16]))
print("\n".join(tl))
