"""The oracle is pinned to the reference itself (SURVEY §8(c) option A): the
unmodified relsim sources, its CLI and its ten test suites compiled here
against eigen-lite / doctest-lite / CLI11-lite (oracle/ref_build.sh).  Needs
/root/reference (the build container); skipped where it is absent (the GPU box),
where tests/test_golden.py carries the reference's outputs as fixtures."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="the reference sources are not on this machine")

SUITES = ["test_scene", "test_expr", "test_eval", "test_diff", "test_index", "test_assembly", "test_solver",
          "test_energies", "test_sim", "test_acceptance"]


@pytest.fixture(scope="module")
def built():
    r = subprocess.run([os.path.join(ROOT, "oracle", "ref_build.sh"), "--tests"], capture_output=True, text=True,
                       timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    return OUT


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_shims(built, suite, tmp_path):
    """The reference's own doctest suite (tests/*.cpp) passes against its
    sources compiled with eigen-lite: the build is faithful."""
    r = subprocess.run([os.path.join(built, suite)], capture_output=True, text=True, timeout=900, cwd=tmp_path)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_oracle_matches_reference_live(built, name):
    """A prepared step through the reference's public API (oracle/ref_driver)
    against the oracle restatement on the same state: bit-exact structure,
    block coordinates and pairs, equal PCG iteration counts, values <= 1e-9."""
    from fixtures import rel
    from make_golden import JITTER, step_record
    from ref_step import reference_step

    from paper_2605_23088_b200 import configs
    r = reference_step(configs.CONFIGS[name](), JITTER[name])
    o = step_record(name, "oracle")
    assert int(r["checksum_static"]) == int(o["checksum_static"])
    assert int(r["checksum_dynamic"]) == int(o["checksum_dynamic"])
    assert np.array_equal(r["pairs"], o["pairs"])
    assert int(r["pcg_iterations"]) == int(o["pcg_iterations"])
    for k in ("dx", "gradient", "diag"):
        assert rel(o[k], r[k]) <= 1e-9, k
