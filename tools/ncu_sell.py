"""ncu target: prepared C5 state, then one launch of the given time_kernel variants."""
import sys

from bench import prepare

name = sys.argv[1]
sim = prepare(name, True, "gpu")
eng = sim.eng
eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
for w in sys.argv[2:]:
    print(w, eng.time_kernel(int(w), 1), flush=True)
