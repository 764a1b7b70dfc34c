"""Committed golden vectors (tests/golden/, written by tools/make_golden.py
from THE REFERENCE ITSELF — relsim's unmodified sources compiled against
eigen-lite, oracle/ref_build.sh): one prepared Newton step of C1, C2 and C3.
The oracle restatement (CPU) and the B200 library (GPU) must both match them
with the parity bars of SURVEY §8(c): structure checksums and the contact pair
list bit-exact, identical PCG iteration counts, dx / gradient / diagonal blocks
within 1e-9 relative (max|diff| / max|ref|), energy within 1e-12."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from fixtures import rel  # noqa: E402
from make_golden import step_record  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}_step.npz")) as z:
        return {k: z[k] for k in z.files}


def check_against_reference(r, g):
    assert str(g["source"]).startswith("reference")
    assert int(g["checksum_static"]) == int(r["checksum_static"])
    assert int(g["checksum_dynamic"]) == int(r["checksum_dynamic"])
    assert np.array_equal(g["pairs"], r["pairs"])
    assert int(g["pcg_iterations"]) == int(r["pcg_iterations"])
    assert rel(r["dx"], g["dx"]) <= 1e-9
    assert rel(r["gradient"], g["gradient"]) <= 1e-9
    assert rel(r["diag"], g["diag"]) <= 1e-9
    assert rel(r["pcg_history"], g["pcg_history"]) <= 1e-6
    assert abs(float(r["energy"]) - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_oracle_matches_reference_golden(name):
    check_against_reference(step_record(name, "oracle"), load(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_gpu_matches_reference_golden(name):
    check_against_reference(step_record(name, "gpu"), load(name))
