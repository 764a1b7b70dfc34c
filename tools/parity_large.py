"""GPU vs the oracle restatement on a large scene (C4 cloth, C5 pile) from the
bench's prepared state (development aid for tests/test_gpu_large.py; prints
every comparison).  usage: python tools/parity_large.py c5 [rollout|jitter]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from bench import oracle_from, prepare  # noqa: E402
from fixtures import rel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
state = sys.argv[2] if len(sys.argv) > 2 else "rollout"
t0 = time.time()
g = prepare(name, True, "gpu", state=state)
t1 = time.time()
o = oracle_from(g, name, True) if state == "rollout" else prepare(name, True, "oracle", state=state)
t2 = time.time()
print(f"{name}: build+pairs gpu {t1-t0:.1f}s oracle {t2-t1:.1f}s", flush=True)
eg, eo = g.eng, o.eng
pg, po = eg.get_pairs(g.contact_pairset), eo.get_pairs(o.contact_pairset)
print("pairs", len(pg), "equal", np.array_equal(pg, po), flush=True)
for e in (eg, eo):
    e.refresh_dynamic()
    e.assemble(True, True)
for w in (0, 1):
    hg, ho = eg.hessian(w), eo.hessian(w)
    print(f"group {w}: checksum equal {hg.checksum == ho.checksum} coords equal "
          f"{np.array_equal(hg.row, ho.row) and np.array_equal(hg.col, ho.col)} values rel {rel(hg.values, ho.values):.2e}",
          flush=True)
print(f"gradient rel {rel(eg.gradient(), eo.gradient()):.2e}  energy rel "
      f"{abs(eg.total_energy() - eo.total_energy()) / abs(eo.total_energy()):.2e}", flush=True)
dg = np.concatenate([b.ravel() for b in eg.diag_blocks()])
do = np.concatenate([b.ravel() for b in eo.diag_blocks()])
print(f"diag rel {rel(dg, do):.2e}", flush=True)
rng = np.random.default_rng(3)
x = rng.standard_normal(eg.s)
print(f"apply_hessian rel {rel(eg.apply_hessian(x), eo.apply_hessian(x)):.2e}", flush=True)
tol = g.config.pcg_tol
for t in (tol, 1e-8, 1e-10):
    sg = eg.minimize_step(t)
    res = {}
    for thr in ("1", "16"):
        os.environ["YO_SPMV_THREADS"] = thr
        t3 = time.time()
        so = eo.minimize_step(t)
        res[thr] = (so, time.time() - t3)
    os.environ["YO_SPMV_THREADS"] = "1"
    s1, s16 = res["1"][0], res["16"][0]
    print(f"tol {t:g}: iterations gpu {sg.pcg_iterations} oracle serial {s1.pcg_iterations} "
          f"oracle 16-shard {s16.pcg_iterations} | residual gpu {sg.pcg_residual:.3e} oracle {s1.pcg_residual:.3e} | "
          f"dx rel gpu-oracle {rel(sg.dx, s1.dx):.2e}, oracle serial-vs-16 {rel(s16.dx, s1.dx):.2e} | "
          f"oracle solve {res['1'][1]:.1f}s", flush=True)
