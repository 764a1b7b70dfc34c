"""One prepared Newton iteration of a config (profiling driver: run under ncu
with a kernel filter).  usage: python tools/one_step.py c5 [steps] [rollout|jitter]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import prepare  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
state = sys.argv[3] if len(sys.argv) > 3 else "rollout"
sim = prepare(name, True, "gpu", state=state)
# ncu --profile-from-start off: the capture starts here, after the rollout
ctypes.CDLL("libcuda.so.1").cuProfilerStart()
for _ in range(steps):
    sim.eng.bump_dynamic_epoch()
    st = sim.eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
print(name, "pcg_iterations", st.pcg_iterations, "path", sim.eng.pcg_path())
sim.eng.close()  # destroy the context: compute-sanitizer --leak-check sees every allocation freed
