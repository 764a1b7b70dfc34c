"""Run k frames of a scene on the B200 library and report Newton / PCG work per
frame (development aid for the bench's prepared state).
usage: python tools/rollout.py c5 25"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig, Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cfg = SimConfig.from_dict(configs.CONFIGS[name]())
t0 = time.perf_counter()
sim = Simulation(cfg)
print(f"build {time.perf_counter() - t0:.1f}s dofs {sim.eng.s} pairs {sim.pair_count()}", flush=True)
for f in range(frames):
    t0 = time.perf_counter()
    rep = sim.step()
    print(f"frame {f + 1}: newton {rep.iterations} pcg {rep.pcg_iterations} conv {rep.converged} "
          f"pairs {sim.pair_count()} {time.perf_counter() - t0:.2f}s", flush=True)
sim.begin_frame()
sim.refresh_dynamic_pairs()
eng = sim.eng
eng.set_profiling(True)
for k in range(6):
    eng.set_option("overlap", 0 if k >= 3 else 1)
    eng.set_option("eval_evd", 0 if k == 5 else 1)
    eng.bump_dynamic_epoch()
    st = eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
    ms, _, nevd = eng.stage_times(True)
    print(f"prepared step (overlap {int(k < 3)}, evd {int(k != 5)}): refresh {ms[0]:.3f} pcg {st.pcg_iterations} stages eval {ms[1]:.3f} gather {ms[2]:.3f} rows {ms[3]:.3f} "
          f"pcg {ms[4]:.3f} total {ms[6]:.3f} indefinite {nevd} jacobi-fallback {eng.evd_fallbacks()}", flush=True)
