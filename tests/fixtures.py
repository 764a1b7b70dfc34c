"""Test scenes built through the C-ABI, mirroring the reference's fixtures
(tests/support/scenes.hpp:15-120, test_assembly.cpp:14-36,
test_energies.cpp:14-48).  Values come from numpy's seeded generator and are
fed identically to every backend (GPU library, oracle, reference build)."""
from __future__ import annotations

import numpy as np

from paper_2605_23088_b200.engine import (YS_POINTS_AFFINE, YS_POINTS_FIXED, YS_POINTS_FREE, YS_PROJECT_FULL,
                                          Engine)


class ContactScene:
    """Free vertices + affine-body vertices under one UNION with a dynamic
    point-point pair primitive (scenes.hpp:15-95)."""

    def __init__(self, eng: Engine, n_free: int, n_bodies: int, n_abd: int, seed: int = 42, n_fixed: int = 0):
        rng = np.random.default_rng(seed)
        self.eng = eng
        self.free_pos = rng.uniform(-1, 1, (n_free, 3))
        av = np.zeros((n_bodies, 9))
        for b in range(n_bodies):
            av[b, [0, 4, 8]] = 1.0
            for d in range(3):
                av[b, d * 3 + (d + 1) % 3] = 0.2 * rng.uniform(-1, 1)
        tv = rng.uniform(-1, 1, (n_bodies, 3))
        self.rest = rng.uniform(-1, 1, (n_abd, 3))
        self.v2b = np.array([(i * n_bodies) // n_abd for i in range(n_abd)], dtype=np.int64)
        self.t_free = eng.add_target(n_free, 3, self.free_pos)
        self.t_A = eng.add_target(n_bodies, 9, av)
        self.t_t = eng.add_target(n_bodies, 3, tv)
        self.d_free = eng.add_points(YS_POINTS_FREE, n_free, self.t_free)
        self.d_abd = eng.add_points(YS_POINTS_AFFINE, n_abd, self.t_A, self.t_t, self.v2b, self.rest)
        doms = [self.d_free, self.d_abd]
        self.n_free, self.n_abd = n_free, n_abd
        if n_fixed:
            self.fixed_pos = rng.uniform(-1, 1, (n_fixed, 3))
            self.d_fixed = eng.add_points(YS_POINTS_FIXED, n_fixed, rest=self.fixed_pos)
            doms.append(self.d_fixed)
        self.union = eng.add_point_union(doms)
        self.pp = eng.add_pair_set(self.union, True)

    def free_index(self, i):
        return i

    def abd_index(self, i):
        return self.n_free + i

    def fixed_index(self, i):
        return self.n_free + self.n_abd + i

    def set_pairs(self, pairs):
        self.eng.set_pairs(self.pp, np.asarray(pairs, dtype=np.int64).reshape(-1))


def tet_scene(eng: Engine, n_tets: int, seed: int, perturb: float):
    """Fan of tets around a shared face (test_energies.cpp:14-48 style) with
    varied vertex orders so oriented-block swaps are exercised."""
    rng = np.random.default_rng(seed)
    nv = n_tets + 3
    rest = np.zeros((nv, 3))
    rest[1] = [1, 0, 0]
    rest[2] = [0, 1, 0]
    for k in range(n_tets):
        rest[3 + k] = [0.3 * rng.uniform(-1, 1), 0.3 * rng.uniform(-1, 1), (1.0 if k % 2 == 0 else -1.0) * (0.8 + 0.1 * k)]
    orders = [(3, 0, 1, 2), (1, 3, 2, 0), (0, 1, 2, 3), (2, 0, 3, 1)]
    t2v = []
    for k in range(n_tets):
        ids = (0, 1, 2, 3 + k)
        # map the template index 3 to the apex vertex of this tet
        t2v.append([ids[o] if o < 3 else ids[3] for o in orders[k % 4]])
    t2v = np.asarray(t2v, dtype=np.int64)
    pos = rest + perturb * rng.uniform(-1, 1, rest.shape)
    t = eng.add_target(nv, 3, pos)
    return t, t2v, rest


def random_system(n_blocks: int, bs: int, density: float, seed: int):
    """Diagonally dominant random block SPD (test_solver.cpp:15-58)."""
    rng = np.random.default_rng(seed)
    coords, vals = [], {}
    for i in range(n_blocks):
        coords.append((bs, bs, i * bs, i * bs))
        for j in range(i + 1, n_blocks):
            if rng.uniform() < density:
                coords.append((bs, bs, i * bs, j * bs))
    diag = [np.zeros((bs, bs)) for _ in range(n_blocks)]
    for (_, _, r, c) in coords:
        if r == c:
            continue
        b = rng.uniform(-1, 1, (bs, bs))
        vals[(r, c)] = b
        diag[r // bs] += np.diag(np.abs(b).sum(axis=1))
        diag[c // bs] += np.diag(np.abs(b).sum(axis=0))
    for i in range(n_blocks):
        d = rng.uniform(-0.2, 0.2, (bs, bs))
        d = 0.5 * (d + d.T) + diag[i] + np.eye(bs) * (1.0 + rng.uniform())
        vals[(i * bs, i * bs)] = d
    return n_blocks * bs, coords, vals


def rel(a, b) -> float:
    """max|a-b| / max(|b|, tiny): the per-array metric of SURVEY §8(c)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0 and b.size == 0:
        return 0.0
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale)
