"""Pass B's projection paths (ys_terms.cuh psd_project9_tri / psd_project9,
ys_set_option "eval_evd"): the clamped-eigenpair path (default), the Jacobi
EVD (0) and the fallback kernel fed with every element (2) must give the same
assembled H within 1e-12 of each other and the oracle's within 1e-9, on C2
(SNH through F, 48k tets) and on the bending cloth of the parity suite."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from backends import simulation  # noqa: E402
from fixtures import rel  # noqa: E402
from paper_2605_23088_b200 import configs  # noqa: E402
from paper_2605_23088_b200.scene import SimConfig  # noqa: E402

pytestmark = pytest.mark.gpu


def _assembled(backend, name, mode=None, jitter=None):
    cfg = SimConfig.from_dict(configs.CONFIGS[name]())
    sim = simulation(cfg, backend)
    if mode is not None:
        sim.eng.set_option("eval_evd", mode)
    configs.jitter_targets(sim, jitter if jitter is not None else (0.002 if name == "c3" else 0.001))
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    sim.eng.refresh_dynamic()
    sim.eng.assemble(True, True)
    h = np.concatenate([sim.eng.hessian(w).values for w in (0, 1)])
    nevd = sim.eng.stage_times(True)[2] if backend == "gpu" else None
    fb = sim.eng.evd_fallbacks() if backend == "gpu" else None
    sim.eng.close()
    return h, nevd, fb


@pytest.mark.parametrize("name", ["c2", "c4_self"])
def test_projection_paths_agree(name):
    ho, _, _ = _assembled("oracle", name)
    ht, nt, ft = _assembled("gpu", name, 1)
    hj, _, _ = _assembled("gpu", name, 0)
    hf, nf, ff = _assembled("gpu", name, 2)
    assert nt > 0 and ft == 0 and ff == nf == nt  # every indefinite element through the fallback in mode 2
    assert rel(ht, hj) <= 1e-12 and rel(hf, hj) <= 1e-12
    for h in (ht, hj, hf):
        assert rel(h, ho) <= 1e-9


def test_projection_paths_under_strong_distortion():
    """C2 with a jitter of half the cell size: inverted and strongly sheared tets,
    up to nine negative eigenvalues (the positive-side path) and near-degenerate
    spectra (fallbacks allowed); every path within 1e-9 of the oracle."""
    ho, _, _ = _assembled("oracle", "c2", jitter=0.005)
    ht, nt, ft = _assembled("gpu", "c2", 1, jitter=0.005)
    hj, _, _ = _assembled("gpu", "c2", 0, jitter=0.005)
    assert nt > 0 and ft <= nt // 100
    assert rel(ht, hj) <= 1e-11
    assert rel(ht, ho) <= 1e-9 and rel(hj, ho) <= 1e-9
