"""One prepared Newton iteration of a config (profiling driver: run under ncu
with a kernel filter).  usage: python tools/one_step.py c5 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig, Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = SimConfig.from_dict(configs.CONFIGS[name]())
sim = Simulation(cfg)
configs.jitter_targets(sim, 0.1 * (0.025 if name == "c1" else 0.01))
sim.begin_frame()
sim.refresh_dynamic_pairs()
for _ in range(steps):
    sim.eng.bump_dynamic_epoch()
    st = sim.eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
print(name, "pcg_iterations", st.pcg_iterations, "path", sim.eng.pcg_path())
sim.eng.close()  # destroy the context: compute-sanitizer --leak-check sees every allocation freed
