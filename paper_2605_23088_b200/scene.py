"""Scene construction and the Newton driver, mirroring relsim's Simulation.

`Simulation(config)` builds the same targets, point domains, energies and
contact union as Simulation::build_from_config (sim.cpp:212-451), in the same
registration order, then drives frames exactly like Simulation::step /
newton_solve (sim.cpp:488-581).  The engine underneath is the C-ABI
(`Engine`) of the B200 library (tests inject the oracle's library through
`library=`).
"""
from __future__ import annotations

import json
import math
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import (YS_POINTS_AFFINE, YS_POINTS_FIXED, YS_POINTS_FREE, Engine)


# ---------------------------------------------------------------------------
# Generators (sim.cpp:62-126)

def make_grid_cloth(nx: int, ny: int, spacing: float, origin=(0.0, 0.0, 0.0)):
    if nx < 2 or ny < 2:
        raise _lib.ValidationError("cloth grid needs at least 2x2 vertices")
    ys, xs = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    v = np.stack([origin[0] + xs * spacing, np.full(xs.shape, float(origin[1])), origin[2] + ys * spacing],
                 axis=-1).reshape(-1, 3)
    tris = []
    for y in range(ny - 1):
        for x in range(nx - 1):
            a, b, c, d = y * nx + x, y * nx + x + 1, (y + 1) * nx + x, (y + 1) * nx + x + 1
            tris += [a, b, c, b, d, c]
    return v.astype(np.float64), np.asarray(tris, dtype=np.int64)


def hinges(tris: np.ndarray) -> np.ndarray:
    """TriMesh::hinges (sim.cpp:83-99): interior edges in std::map key order."""
    t = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    edge_faces: dict[tuple[int, int], list[tuple[int, int]]] = {}
    for f, (a0, a1, a2) in enumerate(t):
        tri = (int(a0), int(a1), int(a2))
        for e in range(3):
            a, b, c = tri[e], tri[(e + 1) % 3], tri[(e + 2) % 3]
            edge_faces.setdefault((min(a, b), max(a, b)), []).append((f, c))
    out = [(e[0], e[1], fs[0][1], fs[1][1]) for e, fs in sorted(edge_faces.items()) if len(fs) == 2]
    return np.asarray(out, dtype=np.int64).reshape(-1, 4)


_KUHN = ((1, 0, 0), (1, 1, 0), (1, 1, 1)), ((1, 0, 0), (1, 0, 1), (1, 1, 1)), \
        ((0, 1, 0), (1, 1, 0), (1, 1, 1)), ((0, 1, 0), (0, 1, 1), (1, 1, 1)), \
        ((0, 0, 1), (1, 0, 1), (1, 1, 1)), ((0, 0, 1), (0, 1, 1), (1, 1, 1))


def make_tet_block(nx: int, ny: int, nz: int, spacing: float, origin=(0.0, 0.0, 0.0)):
    if nx < 1 or ny < 1 or nz < 1:
        raise _lib.ValidationError("tet block needs at least one cell")
    vx, vy, vz = nx + 1, ny + 1, nz + 1
    z, y, x = np.meshgrid(np.arange(vz), np.arange(vy), np.arange(vx), indexing="ij")
    v = np.stack([origin[0] + x * spacing, origin[1] + y * spacing, origin[2] + z * spacing],
                 axis=-1).reshape(-1, 3).astype(np.float64)
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cx, cy, cz = cx.reshape(-1), cy.reshape(-1), cz.reshape(-1)

    def vid(a, b, c):
        return (c * vy + b) * vx + a

    tets = np.empty((cx.size, 6, 4), dtype=np.int64)
    for k, perm in enumerate(_KUHN):
        tets[:, k, 0] = vid(cx, cy, cz)
        for l, o in enumerate(perm):
            tets[:, k, l + 1] = vid(cx + o[0], cy + o[1], cz + o[2])
    return v, tets.reshape(-1)


# ---------------------------------------------------------------------------
# Config (sim.cpp:19-57)

@dataclass
class SimConfig:
    name: str = "scene"
    dt: float = 1e-2
    frames: int = 10
    newton_tol: float = 1e-2
    pcg_tol: float = 1e-4
    max_newton: int = 64
    max_line_search: int = 32
    gravity: tuple = (0.0, -9.8, 0.0)
    output_dir: str = "out"
    seed: int = 0
    threads: int = 1
    contact_enabled: bool = False
    contact_dhat: float = 1e-2
    contact_kappa: float = 1e3
    contact_bodies: list = field(default_factory=list)
    # extension (not in the reference): point-triangle + edge-edge self-contact
    # among the triangle surfaces of these bodies, with its own dhat
    contact_surface: list = field(default_factory=list)
    contact_surface_dhat: float = 0.0
    contact_surface_kappa: float = 0.0
    bodies: list = field(default_factory=list)

    @staticmethod
    def from_dict(j: dict) -> "SimConfig":
        c = SimConfig()
        for k in ("name", "dt", "frames", "newton_tol", "pcg_tol", "max_newton", "max_line_search", "output_dir",
                  "seed", "threads"):
            if k in j:
                setattr(c, k, j[k])
        if "gravity" in j:
            g = list(c.gravity)
            for d in range(min(3, len(j["gravity"]))):
                g[d] = float(j["gravity"][d])
            c.gravity = tuple(g)
        if c.dt <= 0:
            raise _lib.ValidationError("dt must be positive")
        if c.newton_tol <= 0 or c.pcg_tol <= 0:
            raise _lib.ValidationError("tolerances must be positive")
        if "contact" in j:
            ct = j["contact"]
            c.contact_enabled = ct.get("enabled", True)
            c.contact_dhat = ct.get("dhat", c.contact_dhat)
            c.contact_kappa = ct.get("kappa", c.contact_kappa)
            c.contact_bodies = list(ct.get("bodies", []))
            c.contact_surface = list(ct.get("surface", []))
            c.contact_surface_dhat = float(ct.get("surface_dhat", c.contact_dhat))
            c.contact_surface_kappa = float(ct.get("surface_kappa", c.contact_kappa))
        if not isinstance(j.get("bodies"), list) or not j["bodies"]:
            raise _lib.ValidationError("config needs a non-empty 'bodies' array")
        c.bodies = j["bodies"]
        return c

    @staticmethod
    def load(path: str) -> "SimConfig":
        try:
            with open(path) as f:
                j = json.load(f)
        except OSError:
            raise _lib.ValidationError(f"cannot open config file '{path}'")
        except json.JSONDecodeError as e:
            raise _lib.ValidationError(f"config parse error in '{path}': {e}")
        return SimConfig.from_dict(j)


@dataclass
class Body:
    name: str
    kind: str
    fixed: bool = False
    domain: int = -1          # point domain (contact / output vertices)
    n: int = 0
    inertial: bool = False
    inertia_energy: int = -1
    velocity: np.ndarray | None = None
    prev_positions: np.ndarray | None = None
    targets: list = field(default_factory=list)


@dataclass
class NewtonReport:
    iterations: int = 0
    pcg_iterations: int = 0
    converged: bool = False
    last_step_norm: float = 0.0
    energy: float = 0.0
    energy_nonincreasing: bool = True
    diff_seconds: float = 0.0
    pcg_seconds: float = 0.0


def _vec3(j, fallback):
    out = list(fallback)
    for d in range(min(3, len(j or []))):
        out[d] = float(j[d])
    return out


class Simulation:
    def __init__(self, config: SimConfig, device: int = 0, refresh_pairs: bool = True, library=None):
        self.config = config
        self.eng = Engine(device, library)
        self.bodies: list[Body] = []
        self.dt2 = config.dt * config.dt
        self.contact_pairset = -1
        self.contact_children_fixed: list[int] = []
        self.surface_sets: list[int] = []  # PT / EE self-contact stencil sets (extension)
        self.energy_labels: list[str] = []
        self._build()
        self.eng.finalize()
        for b in self.bodies:
            if not b.fixed:
                b.prev_positions = self.body_positions(b).reshape(-1)
        if (self.contact_pairset >= 0 or self.surface_sets) and refresh_pairs:
            self.refresh_dynamic_pairs()

    # -------------------------------------------------------------- build
    def _build(self):
        eng, cfg = self.eng, self.config
        for bj in cfg.bodies:
            body = Body(name=bj.get("name", f"body{len(self.bodies)}"), kind=bj.get("kind", ""),
                        fixed=bool(bj.get("fixed", False)))
            kind = body.kind
            if kind in ("free_points", "affine_points"):
                pts = np.asarray([[float(p[d]) for d in range(3)] for p in bj["points"]], dtype=np.float64)
                n = len(pts)
                body.n = n
                if kind == "free_points":
                    if body.fixed:
                        body.domain = eng.add_points(YS_POINTS_FIXED, n, rest=pts)
                    else:
                        t = eng.add_target(n, 3, pts)
                        body.targets = [t]
                        body.domain = eng.add_points(YS_POINTS_FREE, n, t)
                else:
                    ta = eng.add_target(1, 9, np.eye(3).reshape(-1))
                    tb = eng.add_target(1, 3, np.zeros(3))
                    body.targets = [ta, tb]
                    body.domain = eng.add_points(YS_POINTS_AFFINE, n, ta, tb, np.zeros(n, dtype=np.int64), pts)
                    eng.add_affine_orthogonality(ta, float(bj.get("orthogonality_stiffness", 1e4)), self.dt2)
                if not body.fixed:
                    body.inertial = True
                    mass = np.full(n, float(bj.get("mass", 1.0)))
                    body.inertia_energy = eng.add_inertia(body.domain, mass, pts)
                    v0 = _vec3(bj.get("velocity"), (0.0, 0.0, 0.0))
                    body.velocity = np.tile(np.asarray(v0), n)
            elif kind in ("tet_block", "tet_mesh"):
                if kind == "tet_block":
                    v, tets = make_tet_block(int(bj.get("nx", 2)), int(bj.get("ny", 2)), int(bj.get("nz", 2)),
                                             float(bj.get("spacing", 0.1)), _vec3(bj.get("origin"), (0, 0, 0)))
                else:
                    v = np.loadtxt(bj["vertices_file"]).reshape(-1, 3)
                    tets = np.loadtxt(bj["elements_file"], dtype=np.int64).reshape(-1)
                n = len(v)
                body.n = n
                if body.fixed:
                    body.domain = eng.add_points(YS_POINTS_FIXED, n, rest=v)
                    self.bodies.append(body)
                    continue
                t = eng.add_target(n, 3, v)
                body.targets = [t]
                body.domain = eng.add_points(YS_POINTS_FREE, n, t)
                mat = bj.get("material", {})
                E = float(mat.get("youngs_modulus", 1e4))
                nu = float(mat.get("poisson_ratio", 0.3))
                eng.add_stable_neo_hookean(t, tets, v, E, nu, self.dt2,
                                           bool(bj.get("nh_via_deformation_gradient", False)))
                density = float(bj.get("density", 1000.0))
                tt = tets.reshape(-1, 4)
                d = v[tt[:, 1:]] - v[tt[:, :1]]  # (nt, 3 cols, 3 coords) -> fr(r, c) = d[c][r]
                det = np.linalg.det(np.transpose(d, (0, 2, 1)))
                share = density * np.abs(det) / 6.0 / 4.0
                lumped = np.zeros(n)
                for k in range(4):
                    np.add.at(lumped, tt[:, k], share)
                body.inertial = True
                body.inertia_energy = eng.add_inertia(body.domain, lumped, v)
                body.velocity = np.zeros(3 * n)
            elif kind in ("cloth_grid", "obj_cloth"):
                if kind == "cloth_grid":
                    v, tris = make_grid_cloth(int(bj.get("nx", 4)), int(bj.get("ny", 4)), float(bj.get("spacing", 0.1)),
                                              _vec3(bj.get("origin"), (0, 0, 0)))
                else:
                    v, tris = load_obj(bj["obj_file"])
                if "perturb" in bj:  # synthetic-scene extension: deterministic out-of-plane jitter
                    rng = np.random.default_rng(int(bj.get("seed", 1)))
                    v = v.copy()
                    v[:, 1] += float(bj["perturb"]) * rng.uniform(-1.0, 1.0, len(v))
                n = len(v)
                body.n = n
                if body.fixed:
                    body.domain = eng.add_points(YS_POINTS_FIXED, n, rest=v)
                    self.bodies.append(body)
                    continue
                t = eng.add_target(n, 3, v)
                body.targets = [t]
                body.domain = eng.add_points(YS_POINTS_FREE, n, t)
                body.tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
                hg = hinges(tris)
                if len(hg):
                    eng.add_bending(t, hg.reshape(-1), v, float(bj.get("bending_stiffness", 0.055)), self.dt2)
                density = float(bj.get("density", 0.3))
                tt = tris.reshape(-1, 3)
                a, b, c = v[tt[:, 0]], v[tt[:, 1]], v[tt[:, 2]]
                share = density * 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1) / 3.0
                lumped = np.zeros(n)
                for k in range(3):
                    np.add.at(lumped, tt[:, k], share)
                body.inertial = True
                body.inertia_energy = eng.add_inertia(body.domain, lumped, v)
                body.velocity = np.zeros(3 * n)
            elif kind == "mass_spring":
                raise _lib.DeclError("body kind 'mass_spring' (angular springs) has no B200 kernel")
            else:
                raise _lib.ValidationError(f"unknown body kind '{kind}'")
            self.bodies.append(body)

        if cfg.contact_enabled:
            children, fixed = [], []
            for name in cfg.contact_bodies:
                found = False
                for b in self.bodies:
                    if b.name != name:
                        continue
                    children.append(b.domain)
                    fixed.append(1 if b.fixed else 0)
                    found = True
                if not found:
                    raise _lib.ValidationError(f"contact body '{name}' is not declared")
            if len(children) < 2:
                raise _lib.ValidationError("contact needs at least two bodies")
            uni = eng.add_point_union(children)
            self.contact_pairset = eng.add_pair_set(uni, True)
            self.contact_children_fixed = fixed
            eng.add_point_point_barrier(self.contact_pairset, cfg.contact_dhat, cfg.contact_kappa, self.dt2)
        if cfg.contact_surface:
            self._build_surface_contact()

    def _build_surface_contact(self):
        """Extension (not in the reference): point-triangle and edge-edge
        self-contact among the triangle surfaces of `contact.surface` bodies
        (ys_contact4.cuh / ys_stencil.cu), the point-point barrier's b(d) on
        the squared distance, dhat = `contact.surface_dhat`, kappa =
        `contact.surface_kappa` (default: the point-point kappa)."""
        eng, cfg = self.eng, self.config
        doms, tris, off = [], [], 0
        for name in cfg.contact_surface:
            b = next((b for b in self.bodies if b.name == name), None)
            if b is None or getattr(b, "tris", None) is None:
                raise _lib.ValidationError(f"surface contact body '{name}' is not a free triangle surface")
            doms.append(b.domain)
            tris.append(b.tris + off)
            off += b.n
        tri = np.concatenate(tris)
        e = np.sort(np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [0, 2]]]), axis=1)
        edges = np.unique(e, axis=0)
        uni = eng.add_point_union(doms)
        pt = eng.add_stencil_set(uni, 4, True)
        ee = eng.add_stencil_set(uni, 4, True)
        eng.add_point_triangle_barrier(pt, cfg.contact_surface_dhat, cfg.contact_surface_kappa, self.dt2)
        eng.add_edge_edge_barrier(ee, cfg.contact_surface_dhat, cfg.contact_surface_kappa, self.dt2)
        self._surface_prims = (pt, np.arange(off), tri.reshape(-1), ee, edges.reshape(-1))
        self.surface_sets = [pt, ee]

    # -------------------------------------------------------------- driver
    def body_positions(self, b: Body) -> np.ndarray:
        return self.eng.get_points(b.domain, b.n)

    def refresh_dynamic_pairs(self) -> int:
        """Simulation::refresh_dynamic_pairs (sim.cpp:456-484), on the engine's device
        (plus the PT / EE self-contact stencils of the surface extension)."""
        n = 0
        if self.surface_sets:
            pt, pts, tri, ee, edges = self._surface_prims
            if not getattr(self, "_surface_prims_set", False):
                self.eng.set_stencil_primitives(pt, "pt", pts, tri)
                self.eng.set_stencil_primitives(ee, "ee", edges)
                self._surface_prims_set = True
            for st in self.surface_sets:
                self.eng.refresh_stencils(st, self.config.contact_surface_dhat)
        if self.contact_pairset < 0:
            return n
        return self.eng.refresh_pairs(self.contact_pairset, self.config.contact_dhat, self.contact_children_fixed)

    def pair_count(self) -> int:
        return self.eng.pair_count(self.contact_pairset) if self.contact_pairset >= 0 else 0

    def begin_frame(self):
        cfg = self.config
        g = np.asarray(cfg.gravity)
        for b in self.bodies:
            if not b.inertial:
                continue
            p = self.body_positions(b).reshape(-1)
            xt = p + cfg.dt * b.velocity
            xt = (xt.reshape(-1, 3) + cfg.dt * cfg.dt * g).reshape(-1)
            self.eng.set_inertia_anchor(b.inertia_energy, xt)
            b.prev_positions = p

    def end_frame(self):
        for b in self.bodies:
            if not b.inertial:
                continue
            p = self.body_positions(b).reshape(-1)
            b.velocity = (p - b.prev_positions) / self.config.dt
            b.prev_positions = p

    def _ip_energy(self) -> float:
        try:
            return self.eng.total_energy()
        except _lib.NumericalError:
            return math.inf

    def newton_solve(self) -> NewtonReport:
        """Simulation::newton_solve (sim.cpp:511-573), device resident: the line
        search moves X = X0 - alpha*dx on the device (ys_step_targets)."""
        cfg, eng = self.config, self.eng
        rep = NewtonReport()
        for it in range(cfg.max_newton):
            t0 = time.perf_counter()
            st = eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
            t1 = time.perf_counter()
            rep.diff_seconds += st.assemble_seconds
            rep.pcg_seconds += (t1 - t0) - st.assemble_seconds
            rep.pcg_iterations += st.pcg_iterations
            rep.iterations += 1
            e0 = self._ip_energy()
            alpha, accepted, e_new, step = 1.0, False, e0, 0.0
            for _ in range(cfg.max_line_search):
                step = eng.step_targets(alpha)
                e_new = self._ip_energy()
                if e_new <= e0:
                    accepted = True
                    break
                alpha *= 0.5
            if not accepted:
                eng.step_targets(0.0)
                raise _lib.NumericalError(f"line search failed after {cfg.max_line_search} halvings (newton "
                                          f"iteration {it}, energy {e0:.6f})")
            rep.energy = e_new
            rep.energy_nonincreasing = rep.energy_nonincreasing and e_new <= e0
            rep.last_step_norm = step
            if self.contact_pairset >= 0 or self.surface_sets:
                self.refresh_dynamic_pairs()
            if rep.last_step_norm / cfg.dt < cfg.newton_tol:
                rep.converged = True
                break
        return rep

    def step(self) -> NewtonReport:
        self.begin_frame()
        if self.contact_pairset >= 0 or self.surface_sets:
            self.refresh_dynamic_pairs()
        rep = self.newton_solve()
        self.end_frame()
        return rep

    def positions(self) -> list[np.ndarray]:
        return [self.body_positions(b) for b in self.bodies]

    # -------------------------------------------------------------- output formats
    def write_frame(self, os_, frame: int):
        """Simulation::write_frame (sim.cpp:583-597): every body's "position"
        output, 17 significant digits (printf %.17g)."""
        os_.write(f"frame {frame}\n")
        for b in self.bodies:
            p = self.body_positions(b).reshape(-1, 3)
            os_.write(f"body {b.name} position {len(p)} 3\n")
            if len(p):
                os_.write(("%.17g %.17g %.17g\n" * len(p)) % tuple(p.reshape(-1).tolist()))

    def run(self, log=None):
        """Simulation::run (sim.cpp:599-629): trajectory.txt and stats.csv under
        output_dir, then the timing summary on `log`."""
        log = log if log is not None else sys.stdout
        cfg = self.config
        try:
            os.makedirs(cfg.output_dir, exist_ok=True)
            traj = open(os.path.join(cfg.output_dir, "trajectory.txt"), "w")
            stats = open(os.path.join(cfg.output_dir, "stats.csv"), "w")
        except OSError:
            raise _lib.ValidationError("cannot write to output directory " + cfg.output_dir)
        with traj, stats:
            stats.write("frame,newton,pcg,energy,max_step,pairs,nonincreasing\n")
            diff_total = pcg_total = 0.0
            newton_total = pcg_iters_total = 0
            for f in range(1, cfg.frames + 1):
                rep = self.step()
                self.write_frame(traj, f)
                stats.write("%d,%d,%d,%.17g,%.17g,%d,%d\n" % (f, rep.iterations, rep.pcg_iterations, rep.energy,
                                                             rep.last_step_norm, self.pair_count(),
                                                             1 if rep.energy_nonincreasing else 0))
                diff_total += rep.diff_seconds
                pcg_total += rep.pcg_seconds
                newton_total += rep.iterations
                pcg_iters_total += rep.pcg_iterations
        log.write("frames %d\n" % cfg.frames
                  + "diff total (s) %g\n" % diff_total
                  + "diff average (ms) %g\n" % (1e3 * diff_total / newton_total if newton_total else 0.0)
                  + "cg total (s) %g\n" % pcg_total
                  + "cg average (ms) %g\n" % (1e3 * pcg_total / pcg_iters_total if pcg_iters_total else 0.0)
                  + "newton iterations %d\n" % newton_total
                  + "cg iterations %d\n" % pcg_iters_total)

    def export_matrix(self, frame: int = 0) -> str:
        """The `export-matrix` subcommand (sim.cpp:848-861): step `frame` frames,
        refresh + assemble(project=true), merged MatrixMarket text."""
        from .engine import merged_coordinate_text
        for _ in range(frame):
            self.step()
        self.eng.refresh_dynamic()
        self.eng.assemble(True)
        return merged_coordinate_text(self.eng)


def load_obj(path: str):
    v, f = [], []
    with open(path) as fh:
        for line in fh:
            parts = line.split()
            if not parts:
                continue
            if parts[0] == "v":
                v.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                face = [int(tok.split("/")[0]) - 1 for tok in parts[1:]]
                if len(face) != 3:
                    raise _lib.ValidationError("OBJ loader accepts triangles only")
                f += face
    return np.asarray(v, dtype=np.float64), np.asarray(f, dtype=np.int64)
