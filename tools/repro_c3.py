from paper_2605_23088_b200 import configs
from paper_2605_23088_b200.scene import SimConfig, Simulation
cfg = SimConfig.from_dict(configs.c3())
s = Simulation(cfg, backend="gpu")
configs.jitter_targets(s, 0.002)
s.begin_frame()
print("pairs", s.refresh_dynamic_pairs(), flush=True)
s.eng.refresh_dynamic(); print("refreshed", flush=True)
s.eng.assemble(); print("assembled", flush=True)
st = s.eng.minimize_step(1e-4)
print(st.pcg_iterations, st.pcg_converged)
