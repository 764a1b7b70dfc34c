"""Aggregates an ncu source page (cuda,sass view) by CUDA source line:
warp-stall samples and the top stall reasons per line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
header = None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = next(csv.reader(io.StringIO(line)))[1].split("/")[-1]
        continue
    if line.startswith('"Line No"'):
        header = next(csv.reader(io.StringIO(line)))
        continue
    if header is None or not line.startswith('"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) != len(header) or not r[0]:
        continue
    d = dict(zip(header, r))
    try:
        samples = int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    rows.append((samples, fname, r[0], r[1].strip()[:70], sorted(stalls.items(), key=lambda kv: -kv[1])[:3]))
tot = sum(r[0] for r in rows) or 1
rows.sort(key=lambda r: -r[0])
print(f"total samples {tot}")
for s, f, ln, src, st in rows[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:5} {src:70} {' '.join(f'{k[6:]}={v}' for k, v in st)}")
