"""Per-CTA clocks of the symmetric band PCG (load balance diagnostics).
usage: python tools/sym_ctas.py c5"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig, Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = SimConfig.from_dict(configs.CONFIGS[name]())
sim = Simulation(cfg)
configs.jitter_targets(sim, 0.1 * (0.025 if name == "c1" else 0.01))
sim.begin_frame()
sim.refresh_dynamic_pairs()
for _ in range(2):
    sim.eng.bump_dynamic_epoch()
    st = sim.eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
d = sim.eng.pcg_layout_info(per_cta=True)
cta = d.pop("cta")
print(name, "it", st.pcg_iterations, d)
it = max(st.pcg_iterations, 1)
us = cta[:, :5] / it / 1000.0  # ns -> us per iteration
cols = ["far", "wait", "tiles", "Bspill", "Bupd"]
print("per-iteration us: " + " ".join(f"{c}: mean {us[:, k].mean():.1f} max {us[:, k].max():.1f} (cta {us[:, k].argmax()})"
                                      for k, c in enumerate(cols)))
tot = us[:, 0] + us[:, 1] + us[:, 2]
print(f"phase A work: mean {tot.mean():.1f} max {tot.max():.1f} (cta {tot.argmax()})")
tb = us[:, 3] + us[:, 4]
print(f"phase B work: mean {tb.mean():.1f} max {tb.max():.1f} (cta {tb.argmax()})")
order = np.argsort(-tot)[:8]
for b in order:
    print(f"  cta {b}: rows {cta[b,5]} far {cta[b,6]} spills {cta[b,7]} | " + " ".join(f"{c}={us[b,k]:.1f}" for k, c in enumerate(cols)))
order = np.argsort(-tb)[:5]
for b in order:
    print(f"  B cta {b}: rows {cta[b,5]} far {cta[b,6]} spills {cta[b,7]} | " + " ".join(f"{c}={us[b,k]:.1f}" for k, c in enumerate(cols)))
