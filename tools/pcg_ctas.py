"""PCG time per iteration vs CTAs per SM of the persistent solve (ys_set_option
"pcg_ctas") on a scene's rolled-out state.  usage: python tools/pcg_ctas.py c4 c5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import prepare  # noqa: E402

for name in sys.argv[1:] or ["c5"]:
    sim = prepare(name, True, "gpu")
    eng = sim.eng
    eng.set_profiling(True)
    for per in (3, 2, 1):
        eng.set_option("pcg_ctas", per)
        best = None
        for _ in range(3):
            eng.bump_dynamic_epoch()
            st = eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
            ms, _ = eng.stage_times()
            best = ms[4] if best is None else min(best, ms[4])
        print(f"{name} pcg_ctas={per}: PCG {best:.3f} ms / {st.pcg_iterations} it = "
              f"{1e3 * best / max(st.pcg_iterations, 1):.1f} us/it", flush=True)
