"""GPU parity: the B200 library (through its C-ABI) against the CPU oracle on
identical scenes.  Bars (BASELINE.json north_star):
bit-exact slot tables, compressed sizes, shape groups, coordinates and
structure checksum; energy, gradient, Hessian blocks, diagonal blocks and PCG
solutions within 1e-9 relative (max|diff| / max|ref| per array); identical PCG
iteration counts."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2605_23088_b200 import NumericalError, ValidationError
from paper_2605_23088_b200.engine import (YS_POINTS_AFFINE, YS_POINTS_FIXED, YS_POINTS_FREE, YS_PROJECT_FULL,
                                          YS_PROJECT_REDUCED, BlockSystem, Engine)
from fixtures import ContactScene, random_system, rel, tet_scene
from backends import engine, simulation  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-9


def both(build):
    out = []
    for backend in ("gpu", "oracle"):
        eng = engine(backend)
        handles = build(eng)
        eng.finalize()
        out.append((eng, handles))
    return out


def assert_structures_equal(g: Engine, o: Engine):
    for which in (0, 1):
        hg, ho = g.hessian(which), o.hessian(which)
        assert np.array_equal(hg.groups, ho.groups), f"groups differ ({which})"
        assert np.array_equal(hg.row, ho.row) and np.array_equal(hg.col, ho.col), f"coords differ ({which})"
        assert hg.checksum == ho.checksum, f"checksum differs ({which})"


def assert_tables_equal(g: Engine, o: Engine):
    for e in range(len(g.energy_names)):
        ig, io = g.energy_info(e), o.energy_info(e)
        assert ig == io
        for a, b in zip(g.energy_slots(e), o.energy_slots(e)):
            assert np.array_equal(a, b), f"slot tables of energy {e} differ"
        assert np.array_equal(g.energy_compressed_sizes(e), o.energy_compressed_sizes(e))


def assert_values_close(g: Engine, o: Engine, tol=TOL):
    assert rel(g.gradient(), o.gradient()) <= tol
    for which in (0, 1):
        vg, vo = g.hessian(which).values, o.hessian(which).values
        assert vg.shape == vo.shape
        if vo.size:
            assert rel(vg, vo) <= tol, f"H values ({which}) rel {rel(vg, vo)}"
    dg, do = g.diag_blocks(), o.diag_blocks()
    assert rel(np.concatenate([b.ravel() for b in dg]), np.concatenate([b.ravel() for b in do])) <= tol


def full_check(g, o, project=True, tol=TOL):
    assert_tables_equal(g, o)
    assert_structures_equal(g, o)
    g.assemble(project)
    o.assemble(project)
    assert_values_close(g, o, tol)
    assert abs(g.total_energy() - o.total_energy()) <= 1e-12 * max(1.0, abs(o.total_energy()))


@pytest.mark.parametrize("energy", ["repulsive", "pp"])
@pytest.mark.parametrize("project", [True, False])
def test_contact_scene_mixed_pairs(energy, project):
    pairs = [(0, 3 + 1), (1, 2), (3 + 0, 3 + 3), (0, 3 + 1), (3 + 0, 3 + 1), (2, 3 + 2)]

    def build(eng):
        cs = ContactScene(eng, 3, 2, 4, seed=12)
        if energy == "repulsive":
            eng.add_repulsive(cs.pp, 1.0)
        else:
            eng.add_point_point_barrier(cs.pp, 6.0, 5.0, 1.0)
        cs.set_pairs(pairs)
        return cs

    (g, _), (o, _) = both(build)
    full_check(g, o, project)
    # compressed sizes {6, 12, 15, 24} incl. the same-body merge (test_assembly.cpp:120-161)
    assert set(g.energy_compressed_sizes(0).tolist()) == {6, 12, 15, 24}


def test_contact_scene_with_fixed_branch_and_resize():
    def build(eng):
        cs = ContactScene(eng, 4, 2, 5, seed=8, n_fixed=3)
        eng.add_point_point_barrier(cs.pp, 8.0, 3.0, 0.5)
        cs.set_pairs([(0, cs.fixed_index(1)), (cs.abd_index(2), cs.fixed_index(0)), (1, cs.abd_index(4))])
        return cs

    (g, cg), (o, co) = both(build)
    full_check(g, o)
    assert set(g.energy_compressed_sizes(0).tolist()) == {3, 12, 15}
    # resize_dynamic -> stale -> refresh (engine.cpp:41-60)
    for eng, cs in ((g, cg), (o, co)):
        cs.set_pairs([(2, cs.abd_index(0)), (cs.abd_index(1), cs.fixed_index(2))])
        with pytest.raises(ValidationError, match="stale"):
            eng.assemble()
        eng.refresh_dynamic()
    full_check(g, o)
    # resize to zero
    for eng, cs in ((g, cg), (o, co)):
        cs.set_pairs([])
        eng.refresh_dynamic()
    full_check(g, o)
    assert g.dynamic_hessian().values.size == 0


@pytest.mark.parametrize("via_f", [False, True])
@pytest.mark.parametrize("seed", [21, 22])
def test_stable_neo_hookean(via_f, seed):
    def build(eng):
        t, t2v, rest = tet_scene(eng, 6, seed, 0.15)
        eng.add_stable_neo_hookean(t, t2v, rest, 9.88e3, 0.35, 1.0, via_f)
        return t

    (g, _), (o, _) = both(build)
    for project in (False, True):
        full_check(g, o, project)


def test_bending_and_inertia_cloth():
    from paper_2605_23088_b200.scene import hinges, make_grid_cloth

    def build(eng):
        rng = np.random.default_rng(3)
        v, tris = make_grid_cloth(6, 5, 0.1)
        v = v + 0.03 * rng.uniform(-1, 1, v.shape)
        t = eng.add_target(len(v), 3, v)
        d = eng.add_points(0, len(v), t)
        eng.add_bending(t, hinges(tris).reshape(-1), v, 0.055, 0.7)
        eng.add_inertia(d, rng.uniform(0.5, 2.0, len(v)), v + 0.01)
        return t

    (g, _), (o, _) = both(build)
    full_check(g, o, True)
    full_check(g, o, False)


def test_affine_orthogonality_and_abd_inertia():
    def build(eng):
        cs = ContactScene(eng, 2, 3, 6, seed=6)
        eng.add_affine_orthogonality(cs.t_A, 1e4, 0.3)
        rng = np.random.default_rng(61)
        eng.add_inertia(cs.d_abd, rng.uniform(0.5, 2.0, 6), rng.uniform(-1, 1, (6, 3)))
        eng.add_inertia(cs.d_free, np.ones(2), np.zeros((2, 3)))
        return cs

    (g, _), (o, _) = both(build)
    full_check(g, o, True)
    full_check(g, o, False)


def test_minimize_step_matches_oracle():
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    cfg = SimConfig.from_dict(configs.c3())
    sims = [simulation(cfg, b) for b in ("gpu", "oracle")]
    for s in sims:
        configs.jitter_targets(s, 0.002)
        s.begin_frame()
        s.refresh_dynamic_pairs()
    assert sims[0].pair_count() == sims[1].pair_count() > 0
    g, o = sims[0].eng, sims[1].eng
    assert_structures_equal(g, o)
    sg = g.minimize_step(1e-4)
    so = o.minimize_step(1e-4)
    assert sg.pcg_iterations == so.pcg_iterations
    assert sg.pcg_converged == so.pcg_converged
    assert rel(sg.dx, so.dx) <= TOL
    assert rel(g.pcg_history(), o.pcg_history()) <= 1e-6


def test_minimize_step_uniform_scene_matches_oracle():
    """C2 (8 soft bodies, 31,944 DoFs, ~15k contact pairs): the uniform 3x3
    path — sliced-ELL copy of static + dynamic H, persistent PCG — against the
    oracle's serial spmv_add / pcg (solver.cpp:10-200)."""
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    cfg = SimConfig.from_dict(configs.c2())
    sims = [simulation(cfg, b) for b in ("gpu", "oracle")]
    for s in sims:
        configs.jitter_targets(s, 0.001)
        s.begin_frame()
        s.refresh_dynamic_pairs()
    assert sims[0].pair_count() == sims[1].pair_count() > 1000
    g, o = sims[0].eng, sims[1].eng
    assert_structures_equal(g, o)
    sg = g.minimize_step(1e-4)
    so = o.minimize_step(1e-4)
    assert sg.pcg_iterations == so.pcg_iterations
    assert sg.pcg_converged and so.pcg_converged
    assert rel(sg.dx, so.dx) <= TOL
    assert rel(g.pcg_history(), o.pcg_history()) <= 1e-6
    x = np.random.default_rng(5).uniform(-1, 1, g.s)
    assert rel(g.apply_hessian(x), o.apply_hessian(x)) <= 1e-12


def test_block_system_spmv_and_pcg():
    for nb, bs, seed in ((10, 3, 1), (25, 3, 2), (8, 9, 3), (30, 3, 11)):
        s, coords, vals = random_system(nb, bs, 0.3, seed)
        systems = []
        for backend in ("gpu", "oracle"):
            eng = engine(backend)
            bsys = BlockSystem(eng, s, np.asarray(coords).reshape(-1))
            v = np.zeros(bsys.n_values)
            for (r, c), b in vals.items():
                off = bsys.value_offset(bs, bs, r, c)
                v[off:off + bs * bs] = b.ravel()
            bsys.set_values(v)
            systems.append((eng, bsys))
        (eg, g), (eo, o) = systems
        assert g.checksum == o.checksum
        x = np.random.default_rng(seed).uniform(-1, 1, s)
        yg, yo = g.spmv(x), o.spmv(x)
        assert rel(yg, yo) <= 1e-12
        rhs = np.random.default_rng(seed + 3).uniform(-1, 1, s)
        for pre in (bs, 0):
            xg, itg, rg, cg = g.pcg(rhs, pre, 1e-8, s)
            xo, ito, ro, co = o.pcg(rhs, pre, 1e-8, s)
            assert itg == ito and cg == co
            assert rel(xg, xo) <= 1e-9


def test_numerical_errors_match_reference_wording():
    # singular / non-finite diagonal block names the DoF range (test_solver.cpp:176-194)
    s, coords, vals = random_system(2, 3, 0.0, 5)
    for backend in ("gpu", "oracle"):
        eng = engine(backend)
        bsys = BlockSystem(eng, s, np.asarray(coords).reshape(-1))
        v = np.zeros(bsys.n_values)
        v[0:9] = np.eye(3).ravel()
        v[9:18] = np.nan
        bsys.set_values(v)
        with pytest.raises(NumericalError, match=r"\[3, 6\)"):
            bsys.pcg(np.ones(s), 3, 1e-8, 10)
        # PCG divergence names the iteration
        v[9:18] = (-np.eye(3)).ravel()
        v[0:9] = (-np.eye(3)).ravel()
        bsys.set_values(v)
        with pytest.raises(NumericalError, match="iteration"):
            bsys.pcg(np.ones(s), 0, 1e-8, 10)


def test_refresh_pairs_bit_exact():
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    cfg = SimConfig.from_dict(configs.c3())
    sims = [simulation(cfg, b) for b in ("gpu", "oracle")]
    for s in sims:
        configs.jitter_targets(s, 0.004, seed=99)
    n = [s.refresh_dynamic_pairs() for s in sims]
    assert n[0] == n[1] > 0
    sims[0].eng.refresh_dynamic()
    sims[1].eng.refresh_dynamic()
    assert_tables_equal(sims[0].eng, sims[1].eng)
    assert_structures_equal(sims[0].eng, sims[1].eng)


def test_newton_frames_positions():
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    cfg = SimConfig.from_dict(configs.c1())
    sims = [simulation(cfg, b) for b in ("gpu", "oracle")]
    for frame in range(3):
        reps = [s.step() for s in sims]
        assert reps[0].iterations == reps[1].iterations
        assert reps[0].pcg_iterations == reps[1].pcg_iterations
        pg = np.concatenate([p.ravel() for p in sims[0].positions()])
        po = np.concatenate([p.ravel() for p in sims[1].positions()])
        assert rel(pg, po) <= TOL
        assert sims[0].pair_count() == sims[1].pair_count()


@pytest.mark.parametrize("dhat", [0.0, 0.01, 0.0625, 0.5])
def test_contact_candidates_grid_bit_exact(dhat):
    """The device grid candidates (ys_contact.cu) against the oracle's
    all-pairs loop (sim.cpp:456-484): identical pair list and order.  Dense
    clouds, coordinates on multiples of sqrt(dhat) (cell boundaries), pairs at
    exactly d2 == dhat (excluded), a fixed child (fixed-fixed skipped)."""
    rng = np.random.default_rng(5)
    h = np.sqrt(dhat) if dhat > 0 else 0.1

    def build(eng):
        n_free, n_bodies, n_abd, n_fix = 400, 3, 300, 200
        free = rng.uniform(-0.6, 0.6, (n_free, 3)) if eng.backend == "gpu" else build.free
        build.free = free
        free[:40] = np.round(free[:40] / h) * h  # on cell boundaries
        free[40] = free[41] + np.array([h, 0.0, 0.0])  # d2 == dhat exactly (not a pair)
        t_free = eng.add_target(n_free, 3, free)
        av = np.tile(np.eye(3).reshape(-1), (n_bodies, 1))
        t_A = eng.add_target(n_bodies, 9, av)
        t_t = eng.add_target(n_bodies, 3, np.zeros((n_bodies, 3)))
        rest = build.rest if hasattr(build, "rest") else rng.uniform(-0.5, 0.5, (n_abd, 3))
        build.rest = rest
        fix = build.fix if hasattr(build, "fix") else rng.uniform(-0.7, 0.7, (n_fix, 3))
        build.fix = fix
        d_free = eng.add_points(YS_POINTS_FREE, n_free, t_free)
        d_abd = eng.add_points(YS_POINTS_AFFINE, n_abd, t_A, t_t,
                               np.array([i * n_bodies // n_abd for i in range(n_abd)], dtype=np.int64), rest)
        d_fix = eng.add_points(YS_POINTS_FIXED, n_fix, rest=fix)
        d_fix2 = eng.add_points(YS_POINTS_FIXED, 50, rest=fix[:50] + 1e-3)
        uni = eng.add_point_union([d_free, d_abd, d_fix, d_fix2])
        pp = eng.add_pair_set(uni, True)
        eng.add_point_point_barrier(pp, max(dhat, 1e-3), 1.0, 1.0)
        return pp

    (g, pg), (o, po) = both(build)
    flags = [0, 0, 1, 1]
    ng, no = g.refresh_pairs(pg, dhat, flags), o.refresh_pairs(po, dhat, flags)
    assert ng == no
    assert np.array_equal(g.get_pairs(pg), o.get_pairs(po))
    if dhat >= 0.01:
        assert ng > 0


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_overlap_and_sequential_steps_are_bitwise_equal(name):
    """The static energies' evaluation on side streams (overlapping the dynamic
    rebuild, the default) must give exactly the sequential step
    (ys_set_option("overlap", 0))."""
    import hashlib

    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    outs = []
    for ov in (1, 0):
        cfg = SimConfig.from_dict(configs.CONFIGS[name]())
        sim = Simulation(cfg)
        sim.eng.set_option("overlap", ov)
        configs.jitter_targets(sim, 0.002 if name == "c3" else 0.001)
        sim.begin_frame()
        sim.refresh_dynamic_pairs()
        st = sim.eng.minimize_step(1e-4)
        outs.append((hashlib.sha256(np.ascontiguousarray(st.dx).tobytes()).hexdigest(), st.pcg_iterations))
    assert outs[0] == outs[1], outs


@pytest.mark.parametrize("name", ["c2"])
def test_row_gather_pcg_path(name):
    """The uniform-3x3 solve's second kernel (row gather from upper storage, the
    path taken when the sliced-ELL copy's plan does not fit shared memory),
    forced with ys_set_option("pcg_copy", 0): the oracle's iteration count and
    dx within 1e-9, and the path is reported."""
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig
    from backends import simulation

    def step(backend, copy=None):
        sim = simulation(SimConfig.from_dict(configs.CONFIGS[name]()), backend)
        if copy is not None:
            sim.eng.set_option("pcg_copy", copy)
        configs.jitter_targets(sim, 0.001)
        sim.begin_frame()
        sim.refresh_dynamic_pairs()
        st = sim.eng.minimize_step(1e-4)
        path = sim.eng.pcg_path() if backend == "gpu" else None
        sim.eng.close()
        return st, path

    so, _ = step("oracle")
    sg, pg = step("gpu", 0)
    assert pg == "row gather"
    assert sg.pcg_iterations == so.pcg_iterations
    assert np.max(np.abs(sg.dx - so.dx)) <= 1e-9 * np.max(np.abs(so.dx))


@pytest.mark.parametrize("opt,values,bitwise", [
    ("gather_window", [12, 4, 20], True),       # static gather order: every block's sum keeps its order
    ("eval_low_priority", [1, 0], True),        # side-stream priority: scheduling only
    ("pcg_ctas", [0, 2, 1], False),             # CTA count: the partial sums' grouping changes the rounding
])
def test_execution_options_keep_the_step(opt, values, bitwise):
    """Execution options never change results beyond rounding: the static
    gather order and the stream priority are bitwise neutral; the PCG's CTA
    count regroups the dot-product partials (same iteration count, dx within
    1e-10 at C2)."""
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    outs = []
    for v in values:
        sim = Simulation(SimConfig.from_dict(configs.c2()))
        sim.eng.set_option(opt, v)
        configs.jitter_targets(sim, 0.001)
        sim.begin_frame()
        sim.refresh_dynamic_pairs()
        st = sim.eng.minimize_step(1e-4)
        outs.append((st.dx, st.pcg_iterations))
    for dx, it in outs[1:]:
        assert it == outs[0][1]
        if bitwise:
            assert np.array_equal(dx, outs[0][0])
        else:
            assert np.max(np.abs(dx - outs[0][0])) <= 1e-10 * np.max(np.abs(outs[0][0]))
