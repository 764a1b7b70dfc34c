"""Synthetic scenes C1-C5 of BASELINE.json, expressed in the reference's own
config schema (README.md:52-120, sim.cpp:19-57) so the identical dict drives
the B200 engine, the oracle and the reference build.

Materials follow scenes/block_on_cloth.json: dt 0.005, E 2e4, nu 0.3, density
800, dhat 9e-4 (squared distance), kappa 1e9, pcg_tol 1e-4, newton_tol 1e-2.
The reference has only point-point contact, so PT/EE terms of the paper's
scenes are realised as PP barriers between distinct bodies.

`prepared(cfg)` perturbs the free vertices of every soft body by a seeded
jitter so that a Newton iteration from the initial state has non-trivial
elastic forces; contact pairs exist from the start because the initial gaps
are below sqrt(dhat).
"""
from __future__ import annotations

import math
import os
import tempfile

import numpy as np

MATERIAL = {"youngs_modulus": 20000.0, "poisson_ratio": 0.3}
BASE = {"dt": 0.005, "newton_tol": 0.01, "pcg_tol": 0.0001, "max_newton": 64, "gravity": [0.0, -9.8, 0.0],
        "seed": 1}


def _tet(name, n, spacing, origin, via_f=True):
    return {"name": name, "kind": "tet_block", "nx": n[0], "ny": n[1], "nz": n[2], "spacing": spacing,
            "origin": list(origin), "density": 800.0, "material": dict(MATERIAL),
            "nh_via_deformation_gradient": via_f}


def _ground(name, nx, spacing, origin):
    return {"name": name, "kind": "cloth_grid", "nx": nx, "ny": nx, "spacing": spacing, "origin": list(origin),
            "fixed": True}


def c1(via_f: bool = True) -> dict:
    """Soft cube 6x5x6 cells (1,080 tets) over a fixed ground, PP barrier."""
    return dict(BASE, name="c1_soft_cube", frames=25, bodies=[
        _tet("block", (6, 5, 6), 0.025, (-0.075, 0.02, -0.075), via_f),
        _ground("ground", 15, 0.025, (-0.175, 0.0, -0.175))],
        contact={"enabled": True, "dhat": 0.0009, "kappa": 1e9, "bodies": ["block", "ground"]})


def c2(via_f: bool = True) -> dict:
    """Stack of 8 soft cubes, 10x10x10 cells each (48,000 tets), inter-body PP."""
    bodies, names = [], []
    gap, size = 0.02, 0.1
    for k in range(8):
        nm = f"cube{k}"
        bodies.append(_tet(nm, (10, 10, 10), 0.01, (-0.05, 0.02 + k * (size + gap), -0.05), via_f))
        names.append(nm)
    bodies.append(_ground("ground", 21, 0.01, (-0.1, 0.0, -0.1)))
    names.append("ground")
    return dict(BASE, name="c2_cube_stack", frames=25, bodies=bodies,
                contact={"enabled": True, "dhat": 0.0009, "kappa": 1e9, "bodies": names})


def c3() -> dict:
    """64 affine bodies (3x3x3 lattices) on a 4x4x4 grid over a 16x4x16 soft slab."""
    slab = _tet("slab", (16, 4, 16), 0.02, (-0.16, 0.02, -0.16), True)
    bodies, names = [slab], ["slab"]
    top = 0.02 + 4 * 0.02
    for gy in range(4):
        for gz in range(4):
            for gx in range(4):
                o = np.array([-0.16 + 0.02 + gx * 0.08, top + 0.025 + gy * 0.06, -0.16 + 0.02 + gz * 0.08])
                pts = [[float(o[0] + i * 0.02), float(o[1] + j * 0.02), float(o[2] + k * 0.02)]
                       for k in range(3) for j in range(3) for i in range(3)]
                nm = f"rb{gx}{gy}{gz}"
                bodies.append({"name": nm, "kind": "affine_points", "points": pts, "mass": 0.05,
                               "orthogonality_stiffness": 1e4})
                names.append(nm)
    bodies.append(_ground("ground", 17, 0.02, (-0.16, 0.0, -0.16)))
    names.append("ground")
    return dict(BASE, name="c3_mixed_abd_fem", frames=25, bodies=bodies,
                contact={"enabled": True, "dhat": 0.0009, "kappa": 1e9, "bodies": names})


def sphere_points(n: int, radius: float, center) -> list:
    """Fibonacci sphere."""
    pts = []
    ga = math.pi * (3.0 - math.sqrt(5.0))
    for i in range(n):
        y = 1.0 - 2.0 * (i + 0.5) / n
        r = math.sqrt(max(0.0, 1.0 - y * y))
        th = ga * i
        pts.append([center[0] + radius * r * math.cos(th), center[1] + radius * y, center[2] + radius * r * math.sin(th)])
    return pts


def write_cloth_obj(path: str, nx: int, spacing: float, origin, amplitude: float, seed: int = 1):
    """Grid cloth (make_grid_cloth layout) with a seeded out-of-plane jitter,
    written as OBJ so the reference's obj_cloth loader reads the same mesh."""
    rng = np.random.default_rng(seed)
    with open(path, "w") as f:
        for y in range(nx):
            for x in range(nx):
                f.write(f"v {origin[0] + x * spacing:.17g} {origin[1] + amplitude * rng.uniform(-1, 1):.17g} "
                        f"{origin[2] + y * spacing:.17g}\n")
        for y in range(nx - 1):
            for x in range(nx - 1):
                a, b, c, d = y * nx + x + 1, y * nx + x + 2, (y + 1) * nx + x + 1, (y + 1) * nx + x + 2
                f.write(f"f {a} {b} {c}\nf {b} {d} {c}\n")


def c4(nx: int = 317, cache_dir: str | None = None) -> dict:
    """Free cloth nx x nx (2(nx-1)^2 triangles, bending + inertia) draped over a
    fixed sphere of points; cloth-sphere PP contact (the reference has no EE)."""
    cache_dir = cache_dir or os.path.join(tempfile.gettempdir(), "yasps_b200_scenes")
    os.makedirs(cache_dir, exist_ok=True)
    spacing = 1.0 / (nx - 1)
    path = os.path.join(cache_dir, f"cloth_{nx}.obj")
    if not os.path.exists(path):
        write_cloth_obj(path + ".tmp", nx, spacing, (-0.5, 0.303, -0.5), 0.2 * spacing)
        os.replace(path + ".tmp", path)
    sphere = sphere_points(4000, 0.3, (0.0, 0.0, 0.0))
    dh = (1.5 * spacing) ** 2
    return dict(BASE, name="c4_cloth_sphere", frames=25, bodies=[
        {"name": "cloth", "kind": "obj_cloth", "obj_file": path, "density": 0.3, "bending_stiffness": 0.055},
        {"name": "sphere", "kind": "free_points", "points": sphere, "fixed": True}],
        contact={"enabled": True, "dhat": dh, "kappa": 1e9, "bodies": ["cloth", "sphere"]})


def c4_self(nx: int = 64, cache_dir: str | None = None) -> dict:
    """Extension (not in the reference): C4 at a smaller size with point-triangle
    and edge-edge self-contact on the cloth (dhat = (0.2 spacing)^2)."""
    cfg = c4(nx, cache_dir)
    spacing = 1.0 / (nx - 1)
    cfg["name"] = "c4_self_contact"
    cfg["contact"] = dict(cfg["contact"], surface=["cloth"], surface_dhat=(0.2 * spacing) ** 2)
    return cfg


def c5(n=(28, 28, 27), via_f: bool = True) -> dict:
    """Pile of 8 soft blocks (2x2x2), 1,016,064 tets at the default size."""
    bodies, names = [], []
    sp = 0.01
    gap = 0.02
    ext = [n[0] * sp, n[1] * sp, n[2] * sp]
    for k in range(8):
        i, j, l = k & 1, (k >> 1) & 1, (k >> 2) & 1
        o = (-ext[0] - gap / 2 + i * (ext[0] + gap), 0.02 + j * (ext[1] + gap), -ext[2] - gap / 2 + l * (ext[2] + gap))
        nm = f"ball{k}"
        bodies.append(_tet(nm, n, sp, o, via_f))
        names.append(nm)
    gn = int(round(2 * max(ext[0], ext[2]) / 0.02)) + 3
    bodies.append(_ground("ground", gn, 0.02, (-(gn - 1) * 0.01, 0.0, -(gn - 1) * 0.01)))
    names.append("ground")
    return dict(BASE, name="c5_pile", frames=25, bodies=bodies,
                contact={"enabled": True, "dhat": 0.0009, "kappa": 1e9, "bodies": names})


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "c4_self": c4_self}


def jitter_targets(sim, amplitude: float, seed: int = 7):
    """Seeded perturbation of every free (soft) vertex target: x += U(-a, a)."""
    rng = np.random.default_rng(seed)
    for b in sim.bodies:
        if b.fixed or b.kind not in ("tet_block", "tet_mesh", "cloth_grid", "obj_cloth"):
            continue
        t = b.targets[0]
        x = sim.eng.get_target_values(t)
        x = x + amplitude * rng.uniform(-1.0, 1.0, x.shape)
        sim.eng.set_target_values(t, x)
