"""Builds a scene's prepared state and runs the hot kernels a few times
(target command for ncu captures; run ncu with --profile-from-start off: the
capture starts after the 25-frame rollout)."""
import ctypes
import sys

from bench import prepare

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
sim = prepare(name, True, "gpu")
eng = sim.eng
ctypes.CDLL("libcuda.so.1").cuProfilerStart()
st = eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
print("pcg iterations", st.pcg_iterations, flush=True)
for which in (3, 1, 2):  # SELL SpMV (4 lanes / row), assembly, eval
    print(which, eng.time_kernel(which, 3), flush=True)
