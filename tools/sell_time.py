"""Times the 3x3 SpMV variants (upper-storage row gather vs the sliced-ELL
full copy, H lanes per row) and the whole minimize_step (development aid).
usage: YS_PCG_SELL=<H> python tools/sell_time.py c5"""
import os
import sys

from paper_2605_23088_b200 import configs
from paper_2605_23088_b200.scene import SimConfig, Simulation

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = SimConfig.from_dict(configs.CONFIGS[name]())
sim = Simulation(cfg, backend="gpu")
configs.jitter_targets(sim, 0.1 * (0.025 if name == "c1" else 0.01))
sim.begin_frame()
n = sim.refresh_dynamic_pairs()
eng = sim.eng
eng.set_profiling(True)
for k in range(3):
    eng.bump_dynamic_epoch()
    st = eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
ms, launches, nevd = eng.stage_times(True)
print(f"{name} YS_PCG_SELL={os.environ.get('YS_PCG_SELL')} pcg_it={st.pcg_iterations} res={st.pcg_residual:.6e} "
      f"total={ms[6]:.3f} pcg={ms[4]:.3f} per-it={1e3*ms[4]/max(st.pcg_iterations,1):.1f}us "
      f"phases={[round(1e3*v/max(st.pcg_iterations,1), 2) for v in ms[8:12]]}", flush=True)
VARIANTS = [(0, "row gather k_spmv33"), (40, "sell H=1"), (41, "sell H=2"), (42, "sell H=4"), (43, "sell H=8"),
            (46, "sell build H=4")]
only = os.environ.get("SELL_VARIANTS")
if only:
    keep = {int(v) for v in only.split(",")}
    VARIANTS = [v for v in VARIANTS if v[0] in keep]
for which, label in VARIANTS:
    t, b = eng.time_kernel(which, 50 if which < 44 else 5)
    print(f"  {label:22s} {t*1e3:8.1f} us  {b/t/1e6 if b else 0:7.0f} GB/s (upper-storage algorithmic bytes)", flush=True)
