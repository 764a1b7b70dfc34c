"""Prices the persistent PCG's grid barrier: ys_time_kernel(5) = 1000 counter
barriers, (6) = 1000 barriers + fixed-order partial reductions, at the PCG's grid."""
from bench import prepare

sim = prepare("c1", True, "gpu")
for w, nm in ((5, "counter barrier"), (6, "counter barrier + reduce_partials_all")):
    ms, _ = sim.eng.time_kernel(w, 5)
    print(f"{nm:32s} {ms * 1e3 / 1000:.3f} us each", flush=True)
