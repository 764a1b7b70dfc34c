"""Known-answer tests: the oracle (test infrastructure) pinned against the reference's
own known-answer tests, finite-difference checks of every energy kind, and
the reference's error wording.  Each test cites the reference test it
restates (/root/reference/proj/tests/...)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2605_23088_b200 import DeclError, NumericalError, ValidationError
from paper_2605_23088_b200.engine import (YS_POINTS_FIXED, YS_POINTS_FREE, YS_PROJECT_REDUCED, BlockSystem,
                                          Engine)
from fixtures import ContactScene, random_system, rel, tet_scene
from backends import engine  # noqa: E402


BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def mk(request):
    """Engine factory for the backend under test: the oracle on CPU, the B200
    library on the GPU leg (the same known answers pin both)."""
    return lambda: engine(request.param)


# ---------------------------------------------------------------- layout / slots (test_index.cpp)
def test_gradient_layout_boundaries(mk):
    # test_index.cpp:13-29: 3*5 + 9 + 3 DoFs, boundaries {0, 15, 24, 27}
    e = mk()
    cs = ContactScene(e, 5, 1, 3)
    e.finalize()
    assert e.total_dofs() == 27
    sizes = [n * rc for n, rc in e.targets]
    assert list(np.cumsum([0] + sizes)) == [0, 15, 24, 27]


def test_placement_index_rules(mk):
    # test_index.cpp:89-118: data slot instance 2 -> 7; JOIN (4, 1) -> [13, 4], cols [0, 3]
    e = mk()
    t = e.add_target(5, 3, np.full(15, 0.1))
    d = e.add_points(YS_POINTS_FREE, 5, t)
    e.add_inertia(d, np.ones(5), np.zeros(15))
    u = e.add_point_union([d])
    ps = e.add_pair_set(u, False)
    e.set_pairs(ps, [4, 1])
    e.add_repulsive(ps, 1.0)
    e.finalize()
    idx, ln, col = e.energy_slots(0)
    assert idx[2, 0] == 7 and ln[2, 0] == 3 and col[2, 0] == 0
    idx, ln, col = e.energy_slots(1)
    assert list(idx[0]) == [13, 4] and list(col[0]) == [0, 3]


def test_union_padding_kat(mk):
    # test_index.cpp:120-132: free(1)-abd(0) pair -> [4, 0, 10, 28], lens [3, ., 9, 3], cols 12, 21
    e = mk()
    cs = ContactScene(e, 3, 2, 4)
    e.add_repulsive(cs.pp, 1.0)
    cs.set_pairs([(cs.free_index(1), cs.abd_index(0))])
    e.finalize()
    idx, ln, col = e.energy_slots(0)
    assert list(idx[0]) == [4, 0, 10, 28]
    assert ln[0, 0] == 3 and ln[0, 2] == 9 and ln[0, 3] == 3
    assert col[0, 2] == 12 and col[0, 3] == 21
    info = e.energy_info(0)
    assert info["kappa"] == 4 and info["width"] == 24


# ---------------------------------------------------------------- structure (test_assembly.cpp)
def two_tets(e, seed=5):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, 18)
    t = e.add_target(6, 3, pos)
    rest = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1, 1, 0, 1, 0.5, 1.5], dtype=float)
    e.add_stable_neo_hookean(t, [0, 1, 2, 3, 2, 3, 4, 5], rest, 1e4, 0.3, 1.0)
    return t


def test_shared_vertices_dedup(mk):
    # test_assembly.cpp:63-81: 6 diagonal + 11 off-diagonal unique blocks
    e = mk()
    two_tets(e)
    e.finalize()
    h = e.static_hessian()
    diag = int(np.sum(h.row == h.col))
    assert diag == 6 and len(h.row) - diag == 11
    # sorted, duplicate-free within the shape group
    keys = list(zip(h.row, h.col))
    assert keys == sorted(set(keys))


def test_single_tet_ten_blocks(mk):
    # test_assembly.cpp:84-100
    e = mk()
    t = e.add_target(4, 3, [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1])
    e.add_stable_neo_hookean(t, [0, 1, 2, 3], [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], 1e4, 0.3, 1.0)
    e.finalize()
    assert len(e.static_hessian().row) == 10
    assert list(e.energy_compressed_sizes(0)) == [12]


def test_shape_groups_and_compressed_sizes(mk):
    # test_assembly.cpp:102-132
    e = mk()
    cs = ContactScene(e, 3, 2, 4)
    e.add_repulsive(cs.pp, 1.0)
    cs.set_pairs([(0, 1), (2, cs.abd_index(0)), (cs.abd_index(0), cs.abd_index(3))])
    e.finalize()
    g = e.dynamic_hessian().groups
    shapes = [(int(a), int(b)) for a, b in g[:, :2]]
    assert shapes == sorted(shapes)
    assert (3, 3) in shapes and (3, 9) in shapes and (9, 9) in shapes
    assert set(e.energy_compressed_sizes(0).tolist()) == {6, 15, 24}


def test_two_instances_accumulate(mk):
    # test_assembly.cpp:195-214: duplicated instance doubles every block
    vals = []
    for pairs in ([(0, 1)], [(0, 1), (0, 1)]):
        e = mk()
        t = e.add_target(2, 3, [0, 0, 0, 1, 1, 1])
        d = e.add_points(YS_POINTS_FREE, 2, t)
        u = e.add_point_union([d])
        ps = e.add_pair_set(u, False)
        e.set_pairs(ps, np.asarray(pairs).ravel())
        e.add_repulsive(ps, 1.0)
        e.finalize()
        e.assemble(False)
        vals.append(e.static_hessian().values)
    assert np.allclose(vals[1], 2.0 * vals[0], rtol=1e-14)


def test_checksum_idempotent_and_static_invariant(mk):
    # test_assembly.cpp:231-252 and test_index.cpp:226-273
    e = mk()
    cs = ContactScene(e, 4, 2, 5, seed=8)
    e.add_repulsive(cs.pp, 1.0)
    rng = np.random.default_rng(1)
    e.add_inertia(cs.d_free, np.ones(4), rng.uniform(-1, 1, 12))
    cs.set_pairs([(0, cs.abd_index(1))])
    e.finalize()
    c0 = e.static_hessian().checksum
    cs.set_pairs([(1, 2), (0, cs.abd_index(3))])
    e.refresh_dynamic()
    assert e.static_hessian().checksum == c0


# ---------------------------------------------------------------- energy KATs (test_energies.cpp)
def test_repulsive_value(mk):
    # test_energies.cpp:62-72: 1 / ||p0 - p1|| = 0.5 at distance 2
    e = mk()
    t = e.add_target(2, 3, [0, 0, 0, 2, 0, 0])
    d = e.add_points(YS_POINTS_FREE, 2, t)
    ps = e.add_pair_set(e.add_point_union([d]), True)
    e.set_pairs(ps, [0, 1])
    e.add_repulsive(ps, 1.0)
    e.finalize()
    assert math.isclose(e.total_energy(), 0.5, rel_tol=1e-14)


def test_barrier_zero_and_flat_at_dhat(mk):
    # test_energies.cpp:75-90
    dhat = 0.5
    e = mk()
    t = e.add_target(2, 3, [0, 0, 0, math.sqrt(dhat), 0, 0])
    d = e.add_points(YS_POINTS_FREE, 2, t)
    ps = e.add_pair_set(e.add_point_union([d]), True)
    e.set_pairs(ps, [0, 1])
    e.add_point_point_barrier(ps, dhat, 100.0, 1.0)
    e.finalize()
    assert abs(e.total_energy()) < 1e-14
    e.assemble(False)
    assert np.linalg.norm(e.gradient()) < 1e-12


def test_barrier_blows_up(mk):
    # test_energies.cpp:92-118
    dhat = 0.5
    e = mk()
    t = e.add_target(2, 3, np.zeros(6))
    d = e.add_points(YS_POINTS_FREE, 2, t)
    ps = e.add_pair_set(e.add_point_union([d]), True)
    e.set_pairs(ps, [0, 1])
    e.add_point_point_barrier(ps, dhat, 1.0, 1.0)
    e.finalize()

    def at(d2):
        e.scatter_targets([0, 0, 0, math.sqrt(d2), 0, 0])
        return e.total_energy()

    near, mid, nearer = at(dhat * 1e-6), at(dhat * 0.25), at(dhat * 1e-12)
    assert abs(at(dhat)) < 1e-12 and mid > 0 and near > mid and nearer > near
    e.scatter_targets(np.zeros(6))
    with pytest.raises(NumericalError, match="log of non-positive"):
        e.total_energy()


def test_snh_rest_value_and_gradient(mk):
    # test_energies.cpp:128-152: psi_rest = V (lambda/2 (3mu/4lambda)^2 - mu/2 log 4)
    E_, nu = 1e4, 0.3
    mu, lam = E_ / (2 * (1 + nu)), E_ * nu / ((1 + nu) * (1 - 2 * nu))
    e = mk()
    t, t2v, rest = tet_scene(e, 2, 5, 0.0)
    e.add_stable_neo_hookean(t, t2v, rest, E_, nu, 1.0)
    e.finalize()
    expect = 0.0
    for tet in t2v:
        fr = np.stack([rest[tet[c + 1]] - rest[tet[0]] for c in range(3)], axis=1)
        vol = abs(np.linalg.det(fr)) / 6.0
        a = 3 * mu / (4 * lam)
        expect += vol * (lam / 2 * a * a - mu / 2 * math.log(4.0))
    assert math.isclose(e.total_energy(), expect, rel_tol=1e-12)
    e.assemble(False)
    assert np.linalg.norm(e.gradient()) < 1e-8 * (1 + abs(expect))


def test_snh_via_f_equals_plain_unprojected(mk):
    # test_energies.cpp:154-183
    out = []
    for via in (False, True):
        e = mk()
        t, t2v, rest = tet_scene(e, 3, 31, 0.2)
        e.add_stable_neo_hookean(t, t2v, rest, 1.2e4, 0.33, 1.0, via)
        e.finalize()
        e.assemble(False)
        out.append((e.total_energy(), e.gradient(), e.dense_hessian()))
    assert math.isclose(out[0][0], out[1][0], rel_tol=1e-12)
    assert rel(out[1][1], out[0][1]) < 1e-10
    assert rel(out[1][2], out[0][2]) < 1e-10


def test_orthogonality_value(mk):
    # test_energies.cpp:185-219: ||4I - I||_F^2 / 2 = 13.5 at A = 2I; zero for a rotation
    e = mk()
    a = e.add_target(1, 9, 2.0 * np.eye(3))
    e.add_target(1, 3, np.zeros(3))
    e.add_affine_orthogonality(a, 1.0, 1.0)
    e.finalize()
    assert math.isclose(e.total_energy(), 13.5, rel_tol=1e-14)
    th = 0.83
    k = np.array([1, 2, -1]) / math.sqrt(6)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    R = np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K
    e.set_target_values(a, R)
    assert e.total_energy() <= 1e-12


# ---------------------------------------------------------------- finite differences (oracle.hpp:207-242)
def fd_check(e: Engine, h=1e-5):
    x0 = e.gather_targets()
    e.assemble(False)
    g = e.gradient()
    H = e.dense_hessian()
    gfd = np.zeros_like(x0)
    Hfd = np.zeros((len(x0), len(x0)))
    for j in range(len(x0)):
        xp, xm = x0.copy(), x0.copy()
        xp[j] += h
        xm[j] -= h
        e.scatter_targets(xp)
        ep = e.total_energy()
        e.assemble(False)
        gp = e.gradient()
        e.scatter_targets(xm)
        em = e.total_energy()
        e.assemble(False)
        gm = e.gradient()
        gfd[j] = (ep - em) / (2 * h)
        Hfd[:, j] = (gp - gm) / (2 * h)
    e.scatter_targets(x0)
    relf = lambda a, b: np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b)))  # sim.cpp:665-667
    return relf(g, gfd), relf(H, Hfd)


@pytest.mark.parametrize("kind", ["snh", "snh_f", "bending", "ortho", "pp_mixed", "repulsive", "inertia_abd"])
def test_fd_every_energy(mk, kind):
    e = mk()
    rng = np.random.default_rng(11)
    if kind in ("snh", "snh_f"):
        t, t2v, rest = tet_scene(e, 2, 21, 0.15)
        e.add_stable_neo_hookean(t, t2v, rest, 9.88e3, 0.35, 1.0, kind == "snh_f")
        tol = (1e-5, 2e-4)
    elif kind == "bending":
        rest = np.array([0, 0, 0, 1, 0, 0, 0.4, 1, 0.3, 0.6, -0.8, -0.5])
        t = e.add_target(4, 3, rest + 0.15 * rng.uniform(-1, 1, 12))
        e.add_bending(t, [0, 1, 2, 3], rest, 0.055, 1.0)
        tol = (1e-5, 5e-4)
    elif kind == "ortho":
        skew = np.eye(3)
        skew[0, 1], skew[2, 0] = 0.4, -0.2
        a = e.add_target(1, 9, skew)
        e.add_target(1, 3, np.zeros(3))
        e.add_affine_orthogonality(a, 1.0, 1.0)
        tol = (1e-5, 1e-4)
    elif kind in ("pp_mixed", "repulsive"):
        cs = ContactScene(e, 3, 2, 4, seed=11)
        if kind == "pp_mixed":
            e.add_point_point_barrier(cs.pp, 4.0, 10.0, 1.0)
        else:
            e.add_repulsive(cs.pp, 1.0)
        cs.set_pairs([(0, cs.abd_index(1)), (cs.abd_index(0), cs.abd_index(3))])
        tol = (1e-5, 1e-4)
    else:
        cs = ContactScene(e, 2, 2, 4, seed=6)
        e.add_inertia(cs.d_abd, [1.0, 2.0, 0.5, 1.5], rng.uniform(-1, 1, 12))
        tol = (1e-5, 1e-4)
    e.finalize()
    gr, hr = fd_check(e)
    assert gr < tol[0] and hr < tol[1], (gr, hr)


# ---------------------------------------------------------------- solver (test_solver.cpp)
def test_spmv_kats(mk):
    e = mk()
    bs = BlockSystem(e, 12, [(3, 3, 3 * i, 3 * i) for i in range(4)])
    bs.set_values(np.tile(np.eye(3).ravel(), 4))
    x = np.arange(1.0, 13.0)
    assert np.array_equal(bs.spmv(x), x)
    e2 = mk()
    b = np.arange(1.0, 10.0).reshape(3, 3)
    s2 = BlockSystem(e2, 6, [(3, 3, 0, 3)])
    s2.set_values(b.ravel())
    x = np.array([1, 1, 1, 2, 0, -1.0])
    y = s2.spmv(x)
    assert np.array_equal(y[:3], b @ x[3:]) and np.array_equal(y[3:], b.T @ x[:3])
    with pytest.raises(ValidationError):
        s2.spmv(np.zeros(3))


@pytest.mark.parametrize("nb,bs,seed", [(10, 3, 1), (25, 3, 2), (8, 9, 3)])
def test_spmv_matches_dense(mk, nb, bs, seed):
    s, coords, vals = random_system(nb, bs, 0.3, seed)
    e = mk()
    sysm = BlockSystem(e, s, np.asarray(coords).ravel())
    v = np.zeros(sysm.n_values)
    dense = np.zeros((s, s))
    for (r, c), blk in vals.items():
        off = sysm.value_offset(bs, bs, r, c)
        v[off:off + bs * bs] = blk.ravel()
        dense[r:r + bs, c:c + bs] += blk
        if r != c:
            dense[c:c + bs, r:r + bs] += blk.T
    sysm.set_values(v)
    x = np.random.default_rng(seed + 10).uniform(-1, 1, s)
    y = sysm.spmv(x)
    assert np.linalg.norm(y - dense @ x) <= 1e-12 * max(1.0, np.linalg.norm(dense @ x))
    g = np.random.default_rng(seed).uniform(-1, 1, s)
    xs, it, rr, conv = sysm.pcg(g, bs, 1e-8, s)
    assert conv and it <= s
    assert np.linalg.norm(xs - np.linalg.solve(dense, g)) <= 1e-6 * max(1.0, np.linalg.norm(xs))


def test_pcg_identity_one_iteration_and_zero_rhs(mk):
    e = mk()
    sysm = BlockSystem(e, 15, [(3, 3, 3 * i, 3 * i) for i in range(5)])
    sysm.set_values(np.tile(np.eye(3).ravel(), 5))
    g = np.linspace(-1, 3, 15)
    x, it, rr, conv = sysm.pcg(g, 3, 1e-10, 100)
    assert conv and it == 1 and np.linalg.norm(x - g) < 1e-10
    x, it, rr, conv = sysm.pcg(np.zeros(15), 3, 1e-8, 10)
    assert conv and it == 0 and np.linalg.norm(x) == 0.0


def test_errors_use_reference_wording(mk):
    e = mk()
    cs = ContactScene(e, 3, 2, 4)
    e.add_repulsive(cs.pp, 1.0)
    cs.set_pairs([(0, cs.abd_index(0))])
    e.finalize()
    e.assemble()
    cs.set_pairs([(1, cs.abd_index(1))])
    with pytest.raises(ValidationError, match="stale"):
        e.assemble()
    with pytest.raises(ValidationError, match="out of range"):
        cs.set_pairs([(0, 99)])
    with pytest.raises(DeclError, match="already built"):
        e.add_target(1, 3)
