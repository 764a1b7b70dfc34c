"""Edge cases of the hot path on both backends (oracle on CPU, the B200 library
on the GPU leg): empty dynamic sets, a single element, zero right-hand side,
stencil sets without candidates, and an energy-free pair set — results equal
across backends within the parity bars."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from backends import engine  # noqa: E402
from fixtures import ContactScene, rel, tet_scene  # noqa: E402
from paper_2605_23088_b200.engine import YS_POINTS_FREE  # noqa: E402

BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


def _single_tet(backend, perturb):
    e = engine(backend)
    t, t2v, rest = tet_scene(e, 1, seed=3, perturb=perturb)
    x = e.get_target_values(t)
    dom = e.add_points(YS_POINTS_FREE, 4, t)
    e.add_stable_neo_hookean(t, t2v.reshape(-1), rest, 2e4, 0.3, 1.0, True)
    e.add_inertia(dom, np.full(4, 10.0), x.reshape(-1))
    e.finalize()
    return e


@pytest.mark.parametrize("backend", BACKENDS)
def test_single_element_step_matches(backend):
    """One tet with inertia (a 4x4 block system): the step equals the oracle's,
    and a strongly deformed tet goes through the projection."""
    for perturb in (0.05, 0.4):
        eo, eb = _single_tet("oracle", perturb), _single_tet(backend, perturb)
        so, sb = eo.minimize_step(1e-10), eb.minimize_step(1e-10)
        assert sb.pcg_iterations == so.pcg_iterations
        assert rel(sb.dx, so.dx) <= 1e-9
        eb.assemble(True, True)
        eo.assemble(True, True)
        assert rel(eb.dense_hessian(), eo.dense_hessian()) <= 1e-9
        eo.close()
        eb.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_zero_gradient_returns_zero_step(backend):
    """Inertia at its anchor: the gradient is exactly zero and the PCG returns
    x = 0 without iterating (solver.cpp:156-159)."""
    e = engine(backend)
    x = np.random.default_rng(2).uniform(-1, 1, (7, 3))
    t = e.add_target(7, 3, x)
    dom = e.add_points(YS_POINTS_FREE, 7, t)
    e.add_inertia(dom, np.ones(7), x.reshape(-1))
    e.finalize()
    st = e.minimize_step(1e-6)
    assert st.pcg_converged and st.pcg_iterations == 0
    assert np.all(st.dx == 0.0)
    e.close()


def _two_clouds(backend, dhat):
    e = engine(backend)
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, (5, 3))
    b = rng.uniform(-1, 1, (4, 3)) + np.array([3.0, 0.0, 0.0])
    ta, tb = e.add_target(5, 3, a), e.add_target(4, 3, b)
    da, db = e.add_points(YS_POINTS_FREE, 5, ta), e.add_points(YS_POINTS_FREE, 4, tb)
    e.add_inertia(da, np.ones(5), (a + 0.01).reshape(-1))
    e.add_inertia(db, np.ones(4), (b - 0.01).reshape(-1))
    pp = e.add_pair_set(e.add_point_union([da, db]), True)
    e.add_point_point_barrier(pp, dhat, 1e3, 1.0)
    e.finalize()
    n = e.refresh_pairs(pp, dhat)
    return e, pp, n


@pytest.mark.parametrize("backend", BACKENDS)
def test_empty_dynamic_pair_set(backend):
    """A dynamic pair set with no candidate within dhat: an empty dynamic group;
    the step equals the oracle's (the inertia terms alone)."""
    eo, ppo, no = _two_clouds("oracle", 1e-2)
    eb, ppb, nb = _two_clouds(backend, 1e-2)
    assert no == nb == 0 and eb.pair_count(ppb) == 0
    so, sb = eo.minimize_step(1e-10), eb.minimize_step(1e-10)
    assert sb.pcg_converged and sb.pcg_iterations == so.pcg_iterations
    assert rel(sb.dx, so.dx) <= 1e-12
    eo.close()
    eb.close()


@pytest.mark.parametrize("backend", BACKENDS)
def test_stencil_set_without_candidates(backend):
    """Point-triangle and edge-edge sets whose primitives are far apart: zero
    stencils, zero barrier energy, a valid step."""
    e = engine(backend)
    pts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 5], [1, 0, 5], [0, 1, 5]], dtype=np.float64)
    t = e.add_target(6, 3, pts)
    dom = e.add_points(YS_POINTS_FREE, 6, t)
    e.add_inertia(dom, np.ones(6), pts.reshape(-1))
    uni = e.add_point_union([dom])
    pt = e.add_stencil_set(uni, 4, True)
    ee = e.add_stencil_set(uni, 4, True)
    e.add_point_triangle_barrier(pt, 1e-2, 1e3, 1.0)
    e.add_edge_edge_barrier(ee, 1e-2, 1e3, 1.0)
    e.finalize()
    e.set_stencil_primitives(pt, "pt", np.arange(6), np.array([0, 1, 2, 3, 4, 5]))
    e.set_stencil_primitives(ee, "ee", np.array([0, 1, 1, 2, 3, 4, 4, 5]))
    assert e.refresh_stencils(pt, 1e-2) == 0
    assert e.refresh_stencils(ee, 1e-2) == 0
    st = e.minimize_step(1e-8)
    assert st.pcg_converged
    assert abs(e.total_energy()) < 1e-12
    e.close()
