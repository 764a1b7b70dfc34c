"""Driver-level known answers (test_sim.cpp, test_acceptance.cpp) through the
Newton driver on either backend: the oracle on CPU, the B200 library on the
GPU leg.  Scene JSONs of the reference (scenes/*.json) are embedded because
/root/reference is not present on the GPU box."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2605_23088_b200 import BlockSystem
from paper_2605_23088_b200.scene import SimConfig, Simulation
from backends import simulation  # noqa: E402

BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]

TWO_POINT = {  # test_sim.cpp:31-39
    "name": "two_points", "dt": 0.01, "frames": 3, "gravity": [0, 0, 0],
    "bodies": [{"name": "a", "kind": "free_points", "mass": 1.0, "points": [[0, 0, 0], [0.05, 0, 0]]},
               {"name": "b", "kind": "free_points", "mass": 1.0, "points": [[0.5, 0, 0], [0.55, 0, 0]]}],
    "contact": {"enabled": True, "dhat": 0.01, "kappa": 100.0, "bodies": ["a", "b"]}}

CONTACT_PAIR = {  # scenes/contact_pair.json
    "name": "contact_pair", "dt": 0.005, "frames": 50, "newton_tol": 0.01, "pcg_tol": 0.0001, "max_newton": 64,
    "gravity": [0.0, 0.0, 0.0], "seed": 1,
    "bodies": [
        {"name": "soft_cluster", "kind": "free_points", "mass": 0.8, "velocity": [1.2, 0.0, 0.0],
         "points": [[-0.12, 0.00, 0.00], [-0.18, 0.05, 0.02], [-0.18, -0.05, -0.02], [-0.24, 0.00, 0.04]]},
        {"name": "rigid_cluster", "kind": "affine_points", "mass": 1.2, "orthogonality_stiffness": 10000.0,
         "velocity": [-1.2, 0.0, 0.0],
         "points": [[0.12, 0.00, 0.00], [0.18, 0.06, 0.00], [0.18, -0.06, 0.02], [0.24, 0.00, -0.03]]}],
    "contact": {"enabled": True, "dhat": 0.01, "kappa": 100000000.0, "bodies": ["soft_cluster", "rigid_cluster"]}}

BLOCK_ON_CLOTH = {  # scenes/block_on_cloth.json
    "name": "block_on_cloth", "dt": 0.005, "frames": 50, "newton_tol": 0.01, "pcg_tol": 0.0001, "max_newton": 64,
    "gravity": [0.0, -9.8, 0.0], "seed": 1,
    "bodies": [
        {"name": "block", "kind": "tet_block", "nx": 3, "ny": 2, "nz": 3, "spacing": 0.05,
         "origin": [-0.075, 0.08, -0.075], "density": 800.0,
         "material": {"youngs_modulus": 20000.0, "poisson_ratio": 0.3}, "nh_via_deformation_gradient": True},
        {"name": "cloth", "kind": "cloth_grid", "nx": 15, "ny": 15, "spacing": 0.025, "origin": [-0.175, 0.0, -0.175],
         "fixed": True}],
    "contact": {"enabled": True, "dhat": 0.0009, "kappa": 1000000000.0, "bodies": ["block", "cloth"]}}


@pytest.mark.parametrize("backend", BACKENDS)
def test_proximity_refresh_kat(backend):
    # test_sim.cpp:102-137
    sim = simulation(SimConfig.from_dict(TWO_POINT), backend)
    a, b = sim.bodies
    sim.eng.set_target_values(a.targets[0], [0.0, 0.0, 0.0, 0.05, 0.0, 0.0])
    sim.eng.set_target_values(b.targets[0], [0.04, 0.0, 0.0, 0.09, 0.05, 0.0])
    n = sim.refresh_dynamic_pairs()
    pairs = {tuple(p) for p in sim.eng.get_pairs(sim.contact_pairset).tolist()}
    assert n == 3 and pairs == {(0, 2), (1, 2), (1, 3)}  # independent all-pairs count
    sim.eng.set_target_values(b.targets[0], [2, 0, 0, 3, 0, 0])
    assert sim.refresh_dynamic_pairs() == 0
    sim.eng.set_target_values(b.targets[0], [0.05 + 0.05, 0, 0, 3, 0, 0])
    assert sim.refresh_dynamic_pairs() == 1


@pytest.mark.parametrize("backend", BACKENDS)
def test_free_fall_one_step(backend):
    # test_sim.cpp:139-157: convex quadratic -> exact after one Newton step
    cfg = {"name": "quad", "dt": 0.01, "frames": 1, "gravity": [0, -9.8, 0],
           "bodies": [{"name": "a", "kind": "free_points", "mass": 2.0, "points": [[0, 0, 0], [1, 0, 0], [0, 1, 0]]}]}
    sim = simulation(SimConfig.from_dict(cfg), backend)
    rep = sim.step()
    assert rep.converged and rep.iterations <= 2 and rep.energy_nonincreasing
    sim.eng.assemble(True, False)
    assert np.linalg.norm(sim.eng.gradient()) < 1e-12
    y = sim.body_positions(sim.bodies[0])[0, 1]
    assert math.isclose(y, -9.8 * 0.01 * 0.01, rel_tol=1e-10)


@pytest.mark.parametrize("backend", BACKENDS)
def test_energy_nonincreasing_stiff_contact(backend):
    # test_sim.cpp:159-169 on scenes/contact_pair.json (free + affine bodies)
    sim = simulation(SimConfig.from_dict(CONTACT_PAIR), backend)
    for _ in range(20):
        rep = sim.step()
        assert rep.energy_nonincreasing and math.isfinite(rep.energy)


@pytest.mark.parametrize("backend", BACKENDS)
def test_deterministic_rerun(backend):
    # test_sim.cpp:171-195: byte-identical reruns
    runs = []
    for _ in range(2):
        sim = simulation(SimConfig.from_dict(CONTACT_PAIR), backend)
        for _ in range(8):
            sim.step()
        runs.append(np.concatenate([p.ravel() for p in sim.positions()]))
    assert np.array_equal(runs[0], runs[1])


@pytest.mark.parametrize("backend", BACKENDS)
def test_block_jacobi_beats_identity_on_block_on_cloth(backend):
    # test_acceptance.cpp:456-473: 25 frames to a contact-rich state, then
    # PCG with block Jacobi takes strictly fewer iterations than identity
    sim = simulation(SimConfig.from_dict(BLOCK_ON_CLOTH), backend)
    for _ in range(25):
        sim.step()
    eng = sim.eng
    eng.refresh_dynamic()
    eng.assemble()
    assert sim.pair_count() > 0
    # the assembled H_static + H_dynamic as one free-standing block system
    blocks = {}
    for which in (0, 1):
        for r, c, row, col, b in eng.hessian(which).blocks():
            blocks[(row, col)] = blocks.get((row, col), 0) + b
    coords = [(3, 3, row, col) for (row, col) in sorted(blocks)]
    sysm = BlockSystem(eng, eng.s, np.asarray(coords).ravel())
    v = np.zeros(sysm.n_values)
    for (row, col), b in blocks.items():
        off = sysm.value_offset(3, 3, row, col)
        v[off:off + 9] = b.ravel()
    sysm.set_values(v)
    g = eng.gradient()
    _, it_bj, _, c_bj = sysm.pcg(g, 3, 1e-8, 100000)
    _, it_id, _, c_id = sysm.pcg(g, 0, 1e-8, 100000)
    assert c_bj and c_id and it_bj < it_id
