"""Assembly (gather + block rows) time at C5 for several static gather-order windows
(ys_set_option "gather_window": run-length sort inside windows of 2^w blocks)."""
import os, sys
sys.path.insert(0, os.getcwd())
from bench import prepare
sim = prepare("c5", True, "gpu")
eng = sim.eng
for w in (11, 12, 13, 14, 16):
    eng.set_option("gather_window", w)
    eng.time_kernel(1, 2)
    ms, b = eng.time_kernel(1, 20)
    print(f"window 2^{w}: assembly {ms*1e3:.1f} us {b/ms/1e6:.0f} GB/s", flush=True)
