"""Repeated SpMV launches on the prepared state (for ncu --cache-control none)."""
import sys

from bench import prepare

sim = prepare(sys.argv[1] if len(sys.argv) > 1 else "c5", True, "gpu")
eng = sim.eng
eng.minimize_step(1e-4, -1, want_dx=False)
for w in [int(a) for a in sys.argv[2:]]:
    eng.time_kernel(w, 4)
