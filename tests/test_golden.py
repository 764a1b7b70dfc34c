"""Committed golden vectors (tests/golden/, written by tools/make_golden.py
from the oracle): one prepared Newton step of C1, C2 and C3.  The oracle must
reproduce them exactly (it is deterministic: instance evaluation in parallel
is bit-identical to the serial loop); the B200 library must match them with
the parity bars of SURVEY §8(c) — structure checksums and the contact pair
list bit-exact, identical PCG iteration counts, dx / gradient within 1e-9."""
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


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_oracle_reproduces_golden(name):
    g, r = load(name), step_record(name, "oracle")
    assert int(g["checksum_static"]) == int(r["checksum_static"])
    assert int(g["checksum_dynamic"]) == int(r["checksum_dynamic"])
    assert np.array_equal(g["pairs"], r["pairs"])
    assert int(g["pcg_iterations"]) == int(r["pcg_iterations"])
    assert rel(r["dx"], g["dx"]) <= 1e-13
    assert rel(r["gradient"], g["gradient"]) <= 1e-13
    assert abs(float(r["energy"]) - float(g["energy"])) <= 1e-13 * abs(float(g["energy"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_gpu_matches_golden(name):
    g, r = load(name), step_record(name, "gpu")
    assert int(g["checksum_static"]) == int(r["checksum_static"])
    assert int(g["checksum_dynamic"]) == int(r["checksum_dynamic"])
    assert np.array_equal(g["pairs"], r["pairs"])
    assert int(g["pcg_iterations"]) == int(r["pcg_iterations"])
    assert rel(r["dx"], g["dx"]) <= 1e-9
    assert rel(r["gradient"], g["gradient"]) <= 1e-9
    assert rel(r["pcg_history"], g["pcg_history"]) <= 1e-6
    assert abs(float(r["energy"]) - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
