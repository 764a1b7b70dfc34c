"""Quick device smoke timing of minimize_step on C1..C5 (development aid)."""
import sys
import time

import numpy as np

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import prepare  # noqa: E402

state = os.environ.get("STATE", "rollout")
names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
for name in names:
    t0 = time.perf_counter()
    sim = prepare(name, True, "gpu", state=state)
    cfg = sim.config
    t1 = time.perf_counter()
    n = sim.pair_count()
    t2 = time.perf_counter()
    eng = sim.eng
    eng.set_profiling(True)
    times = []
    for k in range(4):
        eng.bump_dynamic_epoch()
        a = time.perf_counter()
        st = eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
        times.append(time.perf_counter() - a)
    ms, launches, nevd = eng.stage_times(True)
    sp_ms, sp_b = eng.time_kernel(0, 50)
    as_ms, as_b = eng.time_kernel(1, 10)
    ev_ms, _ = eng.time_kernel(2, 10)
    print(f"{name}: s={eng.s} pairs={n} build={t1-t0:.2f}s pairs_t={t2-t1:.2f}s "
          f"step_ms={[round(1e3*t,2) for t in times]} pcg_it={st.pcg_iterations} conv={st.pcg_converged} "
          f"res={st.pcg_residual:.2e} stages(ms) refresh={ms[0]:.3f} eval={ms[1]:.3f} gather={ms[2]:.3f} "
          f"rows={ms[3]:.3f} pcg={ms[4]:.3f} total={ms[6]:.3f} launches={launches} evd={nevd} "
          f"pcg_phases(ms)={[round(v, 2) for v in ms[8:12]]} path={eng.pcg_path()} aux={[round(v, 3) for v in ms[12:16]]}", flush=True)
    print(f"   spmv {sp_ms*1e3:.1f}us {sp_b/sp_ms/1e6:.0f} GB/s | assembly {as_ms*1e3:.1f}us {as_b/as_ms/1e6:.0f} GB/s | "
          f"eval {ev_ms*1e3:.1f}us | dev bytes {eng.device_bytes()/1e9:.2f} GB", flush=True)
