"""Writes tests/golden/*.npz: one prepared Newton step of C1 (soft block on a
fixed ground), C2 (8 soft blocks, uniform 3x3) and C3 (64 affine bodies + soft
slab, mixed shapes), computed by THE REFERENCE ITSELF — the unmodified relsim
sources compiled against eigen-lite (oracle/ref_build.sh, driven by
oracle/ref_driver.cpp through tools/ref_step.py): structure checksums, the
contact pair list, PCG iteration count and history, the step dx, energy,
gradient and the DiagAccumulator blocks.  The oracle restatement and the B200
library are both tested against these fixtures (tests/test_golden.py), so the
parity chain ends at the reference, not at a restatement of it.
usage: python tools/make_golden.py [c1 c2 c3]   (needs /root/reference)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig  # noqa: E402
from backends import simulation  # noqa: E402

JITTER = {"c1": 0.0025, "c2": 0.001, "c3": 0.002}
FIELDS = ("checksum_static", "checksum_dynamic", "pairs", "pcg_iterations", "pcg_history", "dx", "energy",
          "gradient", "diag")


def step_record(name: str, backend: str):
    """The same prepared step on the oracle or the B200 library (the reference
    runs it through tools/ref_step.py)."""
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
        "diag": np.concatenate([b.ravel() for b in eng.diag_blocks()]),
    }


if __name__ == "__main__":
    from ref_step import reference_step
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    for name in sys.argv[1:] or ("c1", "c2", "c3"):
        rec = reference_step(configs.CONFIGS[name](), JITTER[name])
        rec = {k: rec[k] for k in FIELDS}
        rec["source"] = np.array("reference (relsim sources + eigen-lite, oracle/ref_build.sh)")
        np.savez_compressed(os.path.join(out, f"{name}_step.npz"), **rec)
        print(name, {k: (v.shape if hasattr(v, "shape") and v.ndim else v) for k, v in rec.items()})
