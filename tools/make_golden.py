"""Writes tests/golden/*.npz: oracle outputs of one prepared Newton step on the
C1 (soft block on a fixed ground), C2 (8 soft blocks, uniform 3x3) and C3 (64 affine bodies +
soft slab, mixed shapes) scenes — structure checksums, the contact pair list
(reference loop order), PCG iteration count and history, the step dx, energy
and gradient.  The oracle is the CPU restatement of the reference (oracle/);
these fixtures pin it across rounds and let the GPU tests compare against
committed vectors.  usage: python tools/make_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
from backends import simulation  # noqa: E402

JITTER = {"c1": 0.0025, "c2": 0.001, "c3": 0.002}


def step_record(name: str, backend: str):
    cfg = SimConfig.from_dict(configs.CONFIGS[name]())
    sim = simulation(cfg, backend)
    configs.jitter_targets(sim, JITTER[name])
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    eng = sim.eng
    st = eng.minimize_step(cfg.pcg_tol)
    eng.assemble(True, True)
    return {
        "checksum_static": np.uint64(eng.hessian(0).checksum),
        "checksum_dynamic": np.uint64(eng.hessian(1).checksum),
        "pairs": eng.get_pairs(sim.contact_pairset).reshape(-1).astype(np.int32),
        "pcg_iterations": np.int64(st.pcg_iterations),
        "pcg_history": np.asarray(eng.pcg_history(), dtype=np.float64),
        "dx": np.asarray(st.dx, dtype=np.float64),
        "energy": np.float64(eng.total_energy()),
        "gradient": np.asarray(eng.gradient(), dtype=np.float64),
    }


if __name__ == "__main__":
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    for name in ("c1", "c2", "c3"):
        rec = step_record(name, "oracle")
        np.savez_compressed(os.path.join(out, f"{name}_step.npz"), **rec)
        print(name, {k: (v.shape if hasattr(v, "shape") and v.ndim else v) for k, v in rec.items()})
