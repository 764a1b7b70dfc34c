"""Point-triangle, edge-edge and point-edge barriers (SURVEY §8 rows A10 /
(f)3) — NOT IN THE REFERENCE (relsim's contact is point-point only,
proj/README.md:110-111), so their parity is unpinned by the reference: the
oracle restatement (oracle/yo_oracle.c: jets over IPC's distance types) is
checked by the reference's FD harness pattern (tests/support/oracle.hpp:207-242,
central differences, tolerances 1e-5 gradient / 1e-4 Hessian as SPEC.md:729)
and PSD checks, and the B200 kernels (ys_contact4.cuh) against the oracle.

Every distance type is exercised: point-plane / point-edge / point-point for
PT, line-line / point-edge / point-point for EE, point-line / point-point for
PE, with fixed points in the stencils (pads) and random configurations."""
from __future__ import annotations

import numpy as np
import pytest

from backends import engine
from fixtures import rel
from paper_2605_23088_b200.engine import YS_POINTS_FIXED, YS_POINTS_FREE

DHAT, KAPPA, W = 0.01, 1e3, 0.7
H = 0.05

# (kind, arity, free points, fixed points, stencils) — union order: free then fixed
TRI = [[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]
CASES = {
    "pt_face": ("pt", [[0.2, 0.2, H]] + TRI, [], [[0, 1, 2, 3]]),
    "pt_edge": ("pt", [[0.5, -0.04, H]] + TRI, [], [[0, 1, 2, 3]]),
    "pt_vertex": ("pt", [[-0.03, -0.04, H]] + TRI, [], [[0, 1, 2, 3]]),
    "pt_fixed_triangle": ("pt", [[0.25, 0.3, H]], TRI, [[0, 1, 2, 3]]),
    "ee_line_line": ("ee", [[0, 0, 0], [1, 0, 0], [0.5, -0.5, H], [0.45, 0.5, H]], [], [[0, 1, 2, 3]]),
    "ee_point_edge": ("ee", [[0, 0, 0], [1, 0, 0], [1.05, -0.5, H], [1.05, 0.5, H]], [], [[0, 1, 2, 3]]),
    "ee_point_point": ("ee", [[0, 0, 0], [1, 0, 0], [1.04, 0.03, H], [1.3, 1.0, H]], [], [[0, 1, 2, 3]]),
    "ee_fixed_edge": ("ee", [[0.5, -0.5, H], [0.55, 0.5, H]], [[0, 0, 0], [1, 0, 0]], [[2, 3, 0, 1]]),
    "pe_line": ("pe", [[0.5, 0.05, 0.01], [0, 0, 0], [1, 0, 0]], [], [[0, 1, 2]]),
    "pe_point": ("pe", [[-0.05, 0.02, 0.0], [0, 0, 0], [1, 0, 0]], [], [[0, 1, 2]]),
}


def build(backend, kind, free, fixed, stencils):
    eng = engine(backend)
    free = np.asarray(free, dtype=np.float64)
    t = eng.add_target(len(free), 3, free)
    doms = [eng.add_points(YS_POINTS_FREE, len(free), t)]
    if fixed:
        doms.append(eng.add_points(YS_POINTS_FIXED, len(fixed), rest=np.asarray(fixed, dtype=np.float64)))
    u = eng.add_point_union(doms)
    arity = 3 if kind == "pe" else 4
    st = eng.add_stencil_set(u, arity, True)
    add = {"pt": eng.add_point_triangle_barrier, "ee": eng.add_edge_edge_barrier, "pe": eng.add_point_edge_barrier}
    add[kind](st, DHAT, KAPPA, W)
    eng.finalize()
    eng.set_pairs(st, np.asarray(stencils, dtype=np.int64).reshape(-1))
    eng.refresh_dynamic()
    return eng, t


def energy_at(eng, t, x):
    eng.set_target_values(t, x)
    return eng.total_energy()


@pytest.mark.parametrize("case", sorted(CASES))
def test_oracle_fd_and_psd(case):
    kind, free, fixed, stencils = CASES[case]
    eng, t = build("oracle", kind, free, fixed, stencils)
    x0 = np.asarray(free, dtype=np.float64).reshape(-1)
    e0 = energy_at(eng, t, x0)
    assert e0 > 0.0
    eng.assemble(False, True)
    g = eng.gradient().copy()
    Hd = eng.dense_hessian()
    h = 1e-7
    gfd = np.zeros_like(x0)
    hfd = np.zeros((x0.size, x0.size))
    for k in range(x0.size):
        xp, xm = x0.copy(), x0.copy()
        xp[k] += h
        xm[k] -= h
        gfd[k] = (energy_at(eng, t, xp) - energy_at(eng, t, xm)) / (2 * h)
        eng.set_target_values(t, xp)
        eng.assemble(False, True)
        gp = eng.gradient().copy()
        eng.set_target_values(t, xm)
        eng.assemble(False, True)
        gm = eng.gradient().copy()
        hfd[:, k] = (gp - gm) / (2 * h)
    eng.set_target_values(t, x0)
    assert rel(g, gfd) <= 1e-5, (case, rel(g, gfd))
    assert rel(Hd, hfd) <= 1e-4, (case, rel(Hd, hfd))
    # FullProject: the assembled (projected) Hessian is PSD
    eng.assemble(True, True)
    Hp = eng.dense_hessian()
    assert np.min(np.linalg.eigvalsh(0.5 * (Hp + Hp.T))) >= -1e-12 * np.abs(Hp).max()


def test_oracle_rejects_wrong_arity_and_affine_unions():
    from paper_2605_23088_b200 import DeclError
    eng = engine("oracle")
    t = eng.add_target(4, 3, np.zeros((4, 3)))
    u = eng.add_point_union([eng.add_points(YS_POINTS_FREE, 4, t)])
    st3 = eng.add_stencil_set(u, 3, True)
    with pytest.raises(DeclError, match="arity 4"):
        eng.add_point_triangle_barrier(st3, DHAT, KAPPA)


def random_cases(rng, n):
    """Random stencils around a unit configuration (every distance type occurs)."""
    pts = rng.uniform(-0.08, 0.08, (n * 4, 3))
    base = np.array([[0.0, 0.0, 0.05], [0, 0, 0], [0.12, 0.0, 0.0], [0.0, 0.12, 0.0]])
    for s in range(n):
        pts[4 * s:4 * s + 4] += base * rng.uniform(0.5, 1.5)
    return pts


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_gpu_matches_oracle_cases(case):
    kind, free, fixed, stencils = CASES[case]
    out = []
    for b in ("gpu", "oracle"):
        eng, t = build(b, kind, free, fixed, stencils)
        e = eng.total_energy()
        eng.assemble(False, True)
        gu, hu = eng.gradient().copy(), eng.dense_hessian()
        eng.assemble(True, True)
        out.append((e, gu, hu, eng.gradient().copy(), eng.hessian(1).values.copy(), eng.hessian(1).checksum))
    (eg, gug, hug, gg, hg, cg), (eo, guo, huo, go, ho, co) = out
    assert cg == co
    assert abs(eg - eo) <= 1e-12 * abs(eo)
    assert rel(gug, guo) <= 1e-9 and rel(hug, huo) <= 1e-9
    assert rel(gg, go) <= 1e-9 and rel(hg, ho) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["pt", "ee", "pe"])
def test_gpu_matches_oracle_random(kind):
    rng = np.random.default_rng({"pt": 1, "ee": 2, "pe": 3}[kind])
    n = 400
    pts = random_cases(rng, n)
    arity = 3 if kind == "pe" else 4
    stencils = np.array([[4 * s + k for k in range(arity)] for s in range(n)])
    out = []
    for b in ("gpu", "oracle"):
        eng, t = build(b, kind, pts, [], stencils)
        e = eng.total_energy()
        eng.assemble(True, True)
        out.append((e, eng.gradient().copy(), eng.hessian(1).values.copy(), eng.hessian(1).checksum))
    (eg, gg, hg, cg), (eo, go, ho, co) = out
    assert cg == co
    assert abs(eg - eo) <= 1e-12 * abs(eo)
    assert rel(gg, go) <= 1e-9, rel(gg, go)
    assert rel(hg, ho) <= 1e-9, rel(hg, ho)


# ---------------------------------------------------------------------------
# Contact candidates (ys_refresh_stencils): two free cloth layers over a fixed
# one — PT (points x triangles), EE self-contact (edges x edges, incident pairs
# excluded), PE (points x edges) — GPU grid search == oracle all-pairs loop.

def cloth(n, spacing, origin, jitter, rng):
    y, x = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v = np.stack([origin[0] + x.ravel() * spacing, np.full(n * n, origin[1]), origin[2] + y.ravel() * spacing], 1)
    v = v + rng.uniform(-jitter, jitter, v.shape)
    tris, edges = [], set()
    for j in range(n - 1):
        for i in range(n - 1):
            a, b, c, d = j * n + i, j * n + i + 1, (j + 1) * n + i, (j + 1) * n + i + 1
            tris += [(a, b, c), (b, d, c)]
            for e in ((a, b), (a, c), (b, c), (b, d), (c, d)):
                edges.add(tuple(sorted(e)))
    return v, np.array(tris), np.array(sorted(edges))


def layered_scene(backend, kind, seed=5):
    rng = np.random.default_rng(seed)
    n, sp = 9, 0.02
    v0, t0, e0 = cloth(n, sp, (0.0, 0.0, 0.0), 0.002, rng)
    v1, t1, e1 = cloth(n, sp, (0.005, 0.012, 0.004), 0.004, rng)
    vf, tf, ef = cloth(n, sp, (0.0, -0.012, 0.0), 0.0, rng)
    free = np.concatenate([v0, v1])
    eng = engine(backend)
    t = eng.add_target(len(free), 3, free)
    u = eng.add_point_union([eng.add_points(YS_POINTS_FREE, len(free), t),
                             eng.add_points(YS_POINTS_FIXED, len(vf), rest=vf)])
    off1, offf = len(v0), len(free)
    tris = np.concatenate([t0, t1 + off1, tf + offf])
    edges = np.concatenate([e0, e1 + off1, ef + offf])
    pts = np.arange(len(free) + len(vf))
    arity = 3 if kind == "pe" else 4
    st = eng.add_stencil_set(u, arity, True)
    add = {"pt": eng.add_point_triangle_barrier, "ee": eng.add_edge_edge_barrier, "pe": eng.add_point_edge_barrier}
    add[kind](st, (0.012) ** 2, KAPPA, W)
    eng.finalize()
    if kind == "pt":
        eng.set_stencil_primitives(st, "pt", pts, tris.reshape(-1))
    elif kind == "ee":
        eng.set_stencil_primitives(st, "ee", edges.reshape(-1))
    else:
        eng.set_stencil_primitives(st, "pe", pts, edges.reshape(-1))
    return eng, st, tris, edges


@pytest.mark.parametrize("kind", ["pt", "ee", "pe"])
def test_oracle_candidates_exclude_incident_and_fixed(kind):
    eng, st, tris, edges = layered_scene("oracle", kind)
    n = eng.refresh_stencils(st, (0.012) ** 2)
    assert n > 0
    s = eng.get_pairs(st)
    assert len(s) == n
    for row in s[:2000]:
        assert len(set(row.tolist())) == len(row)  # no shared point
    nfree = 2 * 81
    assert np.all((s < nfree).any(axis=1))  # never all-fixed


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["pt", "ee", "pe"])
def test_gpu_candidates_match_oracle(kind):
    out = []
    for b in ("gpu", "oracle"):
        eng, st, _, _ = layered_scene(b, kind)
        n = eng.refresh_stencils(st, (0.012) ** 2)
        out.append((n, eng.get_pairs(st)))
        eng.refresh_dynamic()
        eng.assemble(True, True)
        out[-1] += (eng.gradient().copy(), eng.hessian(1).values.copy(), eng.total_energy())
    (ng, pg, gg, hg, eg), (no, po, go, ho, eo) = out
    assert ng == no and ng > 0
    assert np.array_equal(pg, po)
    assert rel(gg, go) <= 1e-9 and rel(hg, ho) <= 1e-9
    assert abs(eg - eo) <= 1e-12 * abs(eo)
