"""Times the 3x3 SpMV diagnostic variants (ys_time_kernel which >= 10) on the
prepared C5 state; back-to-back launches, like the PCG loop."""
import sys

from bench import prepare

sim = prepare(sys.argv[1] if len(sys.argv) > 1 else "c5", True, "gpu")
eng = sim.eng
eng.minimize_step(1e-4, -1, want_dx=False)
names = {0: "production (static + dynamic)", 23: "u2 SW4 4CTA", 24: "u2 SW4 3CTA", 25: "u2 SW8 3CTA",
         26: "u2 SW2 3CTA", 27: "u2 SW4 2CTA", 18: "static only SW4 4CTA"}
for w, nm in names.items():
    ms, b = eng.time_kernel(w, 50)
    print(f"{nm:32s} {ms*1e3:7.1f} us  {b/ms/1e6:7.0f} GB/s(alg, both groups)", flush=True)
