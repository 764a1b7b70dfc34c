"""TEST INFRASTRUCTURE: one prepared Newton step of a config through the
reference itself (oracle/_ref/ref_driver, the unmodified relsim sources compiled
against eigen-lite by oracle/ref_build.sh), as a record comparable with the
oracle's / the GPU's (tools/make_golden.py step_record).

The prepared state is the one make_golden uses: the config's scene, every free
soft-body vertex jittered by the seeded amplitude (applied through the oracle
engine, gathered and handed to the reference with Engine::scatter_targets),
begin_frame's x_tilde, a contact-pair refresh, one minimize_step, then an
assembly of the same state.
usage: python tools/ref_step.py c1 [jitter]"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def available() -> bool:
    return os.path.exists(DRIVER)


def prepared_x(cfg_dict: dict, jitter: float) -> np.ndarray:
    """The jittered DoF vector (targets in registration order), built on the oracle."""
    from backends import simulation
    sim = simulation(SimConfig.from_dict(cfg_dict), "oracle")
    configs.jitter_targets(sim, jitter)
    return sim.eng.gather_targets()


def _load(pre: str, name: str, dtype) -> np.ndarray:
    p = f"{pre}.{name}.bin"
    return np.fromfile(p, dtype=dtype) if os.path.exists(p) else np.zeros(0, dtype)


def reference_step(cfg_dict: dict, jitter: float, threads: int = 1, timeout: int = 3600) -> dict:
    with tempfile.TemporaryDirectory() as td:
        cfg_path = os.path.join(td, "scene.json")
        with open(cfg_path, "w") as f:
            json.dump(dict(cfg_dict, output_dir=os.path.join(td, "out")), f)
        x = prepared_x(cfg_dict, jitter)
        x_path = os.path.join(td, "x.bin")
        x.astype(np.float64).tofile(x_path)
        pre = os.path.join(td, "rec")
        r = subprocess.run([DRIVER, cfg_path, pre, "--x", x_path, "--threads", str(threads)], capture_output=True,
                           text=True, timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError(f"ref_driver failed ({r.returncode}): {r.stderr[-2000:]}")
        with open(pre + ".json") as f:
            meta = json.load(f)
        rec = {
            "checksum_static": np.uint64(int(meta["static_checksum"])),
            "checksum_dynamic": np.uint64(int(meta["dynamic_checksum"])),
            "pairs": _load(pre, "pairs", np.int64).astype(np.int32),
            "pcg_iterations": np.int64(meta["pcg_iterations"]),
            "pcg_residual": np.float64(meta["pcg_residual"]),
            "pcg_history": _load(pre, "pcg_history", np.float64),
            "dx": _load(pre, "dx", np.float64),
            "energy": np.float64(meta["energy"]),
            "gradient": _load(pre, "gradient", np.float64),
            "diag": _load(pre, "diag", np.float64),
        }
        for tag in ("static", "dynamic"):
            rec[f"{tag}_groups"] = _load(pre, f"{tag}_groups", np.int64).reshape(-1, 5)
            rec[f"{tag}_row"] = _load(pre, f"{tag}_row", np.int64)
            rec[f"{tag}_col"] = _load(pre, f"{tag}_col", np.int64)
            rec[f"{tag}_values"] = _load(pre, f"{tag}_values", np.float64)
        return rec


if __name__ == "__main__":
    import time
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    jit = float(sys.argv[2]) if len(sys.argv) > 2 else {"c1": 0.0025, "c2": 0.001, "c3": 0.002}.get(name, 0.001)
    t0 = time.time()
    rec = reference_step(configs.CONFIGS[name](), jit)
    print(name, f"{time.time() - t0:.1f}s", {k: (v.shape if hasattr(v, "shape") and v.ndim else v) for k, v in rec.items()})
