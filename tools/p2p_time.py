"""Peer-memory row-partitioned solve of C5 (or another scene) from the bench's
rolled-out state, N emulated ranks in one cooperative launch on cuda:0, against
the single-GPU step: iteration count, dx agreement, the solve kernel's device
time and per-iteration phase clocks (CTA 0 of rank 0: A = SpMV + pHp exchange,
B = update + r.r / r.z exchange, C = p update + rank barrier).
usage: python tools/p2p_time.py c5 2 4 8"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from bench import _read_pairs, rollout, scene_config  # noqa: E402


def clone(src, name):
    """A GPU Simulation in the state of `src` (targets, velocities, begin_frame, pairs)."""
    from backends import simulation
    from paper_2605_23088_b200.scene import SimConfig
    sim = simulation(SimConfig.from_dict(scene_config(name, True)), "gpu", refresh_pairs=False)
    for bs, bd in zip(src.bodies, sim.bodies):
        for t in bs.targets:
            sim.eng.set_target_values(t, src.eng.get_target_values(t))
        if bs.velocity is not None:
            bd.velocity = np.array(bs.velocity, copy=True)
    sim.begin_frame()
    if sim.contact_pairset >= 0:
        sim.eng.set_pairs(sim.contact_pairset, _read_pairs(src))
    return sim


def main():
    from paper_2605_23088_b200.engine import p2p_group, p2p_group_step
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
    src = rollout(name, True)
    tol = src.config.pcg_tol
    ref = clone(src, name)
    ref.eng.set_profiling(True)
    for _ in range(3):
        ref.eng.bump_dynamic_epoch()
        st_ref = ref.eng.minimize_step(tol)
    ms, _ = ref.eng.stage_times()
    print(f"{name} 1 GPU: {st_ref.pcg_iterations} iterations, PCG {ms[4]:.3f} ms "
          f"({1e3 * ms[4] / max(st_ref.pcg_iterations, 1):.1f} us/it), phases A/B/C "
          f"{[round(1e3 * v / max(st_ref.pcg_iterations, 1), 1) for v in (ms[8], ms[9] + ms[10], ms[11])]} us/it",
          flush=True)
    for n in worlds:
        sims = [clone(src, name) for _ in range(n)]
        engs = [s.eng for s in sims]
        p2p_group(engs)
        for e in engs:
            e.set_profiling(True)
        best = None
        for _ in range(4):
            for e in engs:
                e.bump_dynamic_epoch()
            steps = p2p_group_step(engs, tol)
            ms, _ = engs[0].stage_times()
            best = ms if best is None or ms[7] < best[7] else best
        it = steps[0].pcg_iterations
        dx = max(np.max(np.abs(st.dx - st_ref.dx)) for st in steps) / np.max(np.abs(st_ref.dx))
        same = all(np.array_equal(st.dx, steps[0].dx) for st in steps)
        info = [e.dist_info() for e in engs]
        ev = [i.get("eval_instances") for i in info]
        print(f"{name} {n} ranks (one launch, {n} x 1/{n} of the SMs): {it} iterations (1 GPU {st_ref.pcg_iterations}), "
              f"dx rel {dx:.2e}, ranks identical {same}; solve kernel {best[7]:.3f} ms = "
              f"{1e3 * best[7] / max(it, 1):.1f} us/it; rank-0 phases A/B/C "
              f"{[round(1e3 * v / max(it, 1), 1) for v in (best[8], best[9], best[11])]} us/it; "
              f"halo rows {[i['halo_rows'] for i in info]}; evaluated tets {ev}", flush=True)
        del sims, engs


if __name__ == "__main__":
    main()
