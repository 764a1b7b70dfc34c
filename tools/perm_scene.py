"""SpMV / PCG / Newton-iteration timing of C5 with a seeded random
vertex permutation of every soft block (as in the paper's SpMV runs) beside the
natural (lexicographic) order.  The permuted scene is the same C5 written as
the reference's "tet_mesh" bodies (vertices_file / elements_file) with vertex
ids shuffled by numpy's PCG64 seeded 1 (not the paper's mt19937_64 stream: the
point is an unordered mesh, not a particular permutation).  Both scenes are
rolled out 25 frames on the device and timed from that state.
usage: python tools/perm_scene.py [frames]"""
import copy
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def permuted_c5(cfg, seed=1):
    from paper_2605_23088_b200.scene import make_tet_block
    rng = np.random.default_rng(seed)
    d = tempfile.mkdtemp(prefix="yasps_perm_")
    out = copy.deepcopy(cfg)
    out["name"] = cfg["name"] + "_permuted"
    for b in out["bodies"]:
        if b.get("kind") != "tet_block":
            continue
        v, t = make_tet_block(b["nx"], b["ny"], b["nz"], b["spacing"], b["origin"])
        perm = rng.permutation(len(v))          # new id of old vertex k: inv[k]
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(v))
        vp = v[perm]
        tp = inv[np.asarray(t).reshape(-1)]
        vf, ef = os.path.join(d, b["name"] + ".v"), os.path.join(d, b["name"] + ".e")
        np.savetxt(vf, vp, fmt="%.17g")
        np.savetxt(ef, tp.reshape(-1, 4), fmt="%d")
        for k in ("nx", "ny", "nz", "spacing", "origin"):
            b.pop(k)
        b["kind"] = "tet_mesh"
        b["vertices_file"], b["elements_file"] = vf, ef
    return out


def run(cfg, frames):
    from backends import simulation
    from paper_2605_23088_b200.scene import SimConfig
    sim = simulation(SimConfig.from_dict(cfg), "gpu")
    t0 = time.perf_counter()
    for _ in range(frames):
        sim.step()
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    roll = time.perf_counter() - t0
    eng = sim.eng
    eng.set_profiling(True)
    steps = []
    for _ in range(6):
        eng.bump_dynamic_epoch()
        st = eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
        ms, _ = eng.stage_times()
        steps.append((ms[6], ms[4], st.pcg_iterations))
    sp_ms, sp_b = eng.time_kernel(3, 50)
    best = min(steps[2:])
    return roll, best, sp_ms, sp_b


def main():
    from paper_2605_23088_b200 import configs
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    base = configs.c5()
    for label, cfg in (("natural order", base), ("random vertex permutation", permuted_c5(base))):
        roll, (step_ms, pcg_ms, it), sp_ms, sp_b = run(cfg, frames)
        print(f"c5 {label}: rollout {roll:.1f} s; step {step_ms:.3f} ms, PCG {pcg_ms:.3f} ms / {it} it "
              f"= {1e3 * pcg_ms / max(it, 1):.1f} us/it; SpMV (sliced-ELL copy) {1e3 * sp_ms:.1f} us = "
              f"{sp_b / sp_ms / 1e6:.0f} GB/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
