"""Times the contact-candidate refresh (ys_refresh_pairs) on a prepared scene."""
import sys
import time

from bench import prepare

sim = prepare(sys.argv[1] if len(sys.argv) > 1 else "c5", True, "gpu")
for k in range(4):
    t0 = time.perf_counter()
    n = sim.refresh_dynamic_pairs()
    print(f"refresh_pairs: {n} pairs in {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
