"""A/B of the side-stream priority (ys_set_option "eval_low_priority") on the
bench's rolled-out state: device time of minimize_step and its stages,
interleaved, median of 10.  usage: python tools/prio_ab.py [c5]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench import rollout  # noqa: E402
from p2p_time import clone  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    src = rollout(name, True)
    sims = {}
    for v in (1, 0):
        s = clone(src, name)
        s.eng.set_option("eval_low_priority", v)
        s.eng.set_profiling(True)
        sims[v] = s
    rows = {1: [], 0: []}
    for k in range(13):
        for v, s in sims.items():
            s.eng.bump_dynamic_epoch()
            st = s.eng.minimize_step(s.config.pcg_tol, -1, want_dx=False)
            ms, _ = s.eng.stage_times()
            if k >= 3:
                rows[v].append((ms[6], ms[0], ms[1] + ms[2], ms[4], st.pcg_iterations))
    for v in (1, 0):
        r = rows[v]
        med = [statistics.median(x[i] for x in r) for i in range(4)]
        print(f"{name} eval_low_priority={v}: step {med[0]:.3f} ms (refresh {med[1]:.3f}, after-refresh eval+gather "
              f"{med[2]:.3f}, pcg {med[3]:.3f}), iterations {r[0][4]}", flush=True)


if __name__ == "__main__":
    main()
