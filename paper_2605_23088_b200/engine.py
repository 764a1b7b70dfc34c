"""Python mirror of relsim::Engine over the C-ABI (engine.hpp:27-80).

`Engine` drives one context of the B200 library (tests may inject another
implementation of the same C-ABI — see oracle/__init__.py; the product never
does).  Method names, argument meaning and raised
exception classes follow the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (YS_POINTS_AFFINE, YS_POINTS_FIXED, YS_POINTS_FREE, YS_PROJECT_FULL,  # noqa: F401
                   YS_PROJECT_REDUCED, StepStats, check)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _ip32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).reshape(-1)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64)).reshape(-1)


@dataclass
class Step:
    dx: np.ndarray | None
    pcg_iterations: int
    pcg_residual: float
    pcg_converged: bool
    regularized_blocks: int
    assemble_seconds: float
    solve_seconds: float


@dataclass
class HessianStructure:
    groups: np.ndarray  # n x 5 {rows, cols, coord_start, count, value_start}
    row: np.ndarray
    col: np.ndarray
    values: np.ndarray
    checksum: int
    total_dofs: int

    def to_dense(self) -> np.ndarray:
        """BlockSparseHessian::to_dense (assembly.cpp:91-104)."""
        s = self.total_dofs
        d = np.zeros((s, s))
        for rows, cols, cs, cnt, vs in self.groups:
            for k in range(cnt):
                r, c = self.row[cs + k], self.col[cs + k]
                b = self.values[vs + k * rows * cols: vs + (k + 1) * rows * cols].reshape(rows, cols)
                d[r:r + rows, c:c + cols] += b
                if r != c:
                    d[c:c + cols, r:r + rows] += b.T
        return d

    def blocks(self):
        """Yields (rows, cols, row, col, block) in storage order."""
        for rows, cols, cs, cnt, vs in self.groups:
            for k in range(cnt):
                yield (int(rows), int(cols), int(self.row[cs + k]), int(self.col[cs + k]),
                       self.values[vs + k * rows * cols: vs + (k + 1) * rows * cols].reshape(rows, cols))

    def coordinate_entries(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Scalar (row, col, value) entries, 0-based, in the storage order of
        BlockSparseHessian::to_coordinate_text (assembly.cpp:106-134): block by
        block, row-major inside a block, the strict lower part of diagonal
        blocks skipped."""
        rs, cs_, vs_ = [], [], []
        for rows, cols, cst, cnt, vst in self.groups:
            rows, cols, cnt = int(rows), int(cols), int(cnt)
            if cnt == 0:
                continue
            r0 = self.row[cst:cst + cnt].astype(np.int64)
            c0 = self.col[cst:cst + cnt].astype(np.int64)
            a, b = np.divmod(np.arange(rows * cols), cols)
            rr = r0[:, None] + a[None, :]
            cc = c0[:, None] + b[None, :]
            vv = self.values[vst:vst + cnt * rows * cols].reshape(cnt, rows * cols)
            keep = ~((r0 == c0)[:, None] & (a > b)[None, :])
            rs.append(rr[keep])
            cs_.append(cc[keep])
            vs_.append(vv[keep])
        if not rs:
            return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
        return np.concatenate(rs), np.concatenate(cs_), np.concatenate(vs_)

    def to_coordinate_text(self) -> str:
        """BlockSparseHessian::to_coordinate_text (assembly.cpp:106-134):
        MatrixMarket coordinate text of the stored upper triangle, values at
        17 significant digits."""
        r, c, v = self.coordinate_entries()
        return matrix_market_text(self.total_dofs, r, c, v)


def matrix_market_text(total_dofs: int, r: np.ndarray, c: np.ndarray, v: np.ndarray) -> str:
    """The header and entry lines both coordinate writers of the reference
    emit (`os.precision(17)` prints a double like printf's %.17g)."""
    head = ("%%MatrixMarket matrix coordinate real general\n% upper triangle of a symmetric matrix\n"
            f"{total_dofs} {total_dofs} {len(v)}\n")
    if len(v) == 0:
        return head
    flat = np.empty(3 * len(v), dtype=object)
    flat[0::3] = (r + 1).tolist()
    flat[1::3] = (c + 1).tolist()
    flat[2::3] = v.tolist()
    return head + ("%d %d %.17g\n" * len(v)) % tuple(flat)


def merged_coordinate_text(eng: "Engine") -> str:
    """merged_coordinate_text (sim.cpp:745-771), the `export-matrix` output: the
    static and dynamic upper entries merged in a std::map keyed by (row, col).
    Each map value starts at +0.0 and adds the static entry, then the dynamic
    one, so -0.0 prints as 0 exactly as in the reference."""
    parts = [eng.hessian(w).coordinate_entries() for w in (0, 1)]
    r = np.concatenate([p[0] for p in parts])
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    order = np.lexsort((c, r))  # stable: static before dynamic for equal keys
    r, c, v = r[order], c[order], v[order]
    first = np.ones(len(v), dtype=bool)
    first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    heads = np.flatnonzero(first)
    acc = 0.0 + v[heads]
    tail = np.flatnonzero(~first)  # blocks are unique per store: <= 1 dynamic entry per static key
    seg = np.searchsorted(heads, tail, side="right") - 1
    acc[seg] = acc[seg] + v[tail]
    return matrix_market_text(eng.total_dofs(), r[heads], c[heads], acc)


class Engine:
    def __init__(self, device: int = 0, library: _lib.Library | None = None):
        self.lib = library if library is not None else _lib.gpu_library()
        self.f = self.lib.fns
        h = C.c_void_p()
        st = self.f["create"](C.byref(h), device)
        if st != 0:
            raise _lib.CudaError(f"{self.lib.path.name}: context creation failed (status {st}); "
                                 "the B200 path needs an sm_100 device")
        self.ctx = h
        self.targets: list[tuple[int, int]] = []
        self.energy_names: list[str] = []
        self._arity: dict[int, int] = {}

    def close(self):
        if getattr(self, "ctx", None):
            self.f["destroy"](self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, status):
        check(self.lib, self.ctx, status)

    # ---------------- scene side ----------------
    def add_target(self, instances: int, rc: int, values=None) -> int:
        tid = C.c_int32()
        self._c(self.f["add_target"](self.ctx, int(instances), int(rc), C.byref(tid)))
        self.targets.append((int(instances), int(rc)))
        if values is not None:
            self.set_target_values(tid.value, values)
        return tid.value

    def set_target_values(self, tid: int, values):
        v = _f64(values)
        self._c(self.f["set_target_values"](self.ctx, tid, _dp(v)))

    def get_target_values(self, tid: int) -> np.ndarray:
        n, rc = self.targets[tid]
        out = np.zeros(n * rc)
        self._c(self.f["get_target_values"](self.ctx, tid, _dp(out)))
        return out

    def total_dofs(self) -> int:
        s = C.c_int64()
        self._c(self.f["total_dofs"](self.ctx, C.byref(s)))
        return s.value

    def add_points(self, kind: int, n: int, target_a: int = -1, target_b: int = -1, v2b=None,
                   rest=None) -> int:
        did = C.c_int32()
        vb = _i64(v2b if v2b is not None else np.zeros(0))
        rs = _f64(rest if rest is not None else np.zeros(0))
        self._c(self.f["add_points"](self.ctx, kind, int(n), target_a, target_b, _ip64(vb), _dp(rs),
                                     C.byref(did)))
        return did.value

    def get_points(self, domain: int, n: int) -> np.ndarray:
        out = np.zeros(3 * n)
        self._c(self.f["get_points"](self.ctx, domain, _dp(out)))
        return out.reshape(n, 3)

    def add_point_union(self, domains) -> int:
        d = np.ascontiguousarray(np.asarray(domains, dtype=np.int32))
        uid = C.c_int32()
        self._c(self.f["add_point_union"](self.ctx, len(d), _ip32(d), C.byref(uid)))
        return uid.value

    def add_pair_set(self, union_id: int, dynamic: bool = True) -> int:
        pid = C.c_int32()
        self._c(self.f["add_pair_set"](self.ctx, union_id, 1 if dynamic else 0, C.byref(pid)))
        self._arity[pid.value] = 2
        return pid.value

    def add_stencil_set(self, union_id: int, arity: int, dynamic: bool = True) -> int:
        """A stencil primitive of arity 2-4 into a union (contact stencils of the
        point-edge / point-triangle / edge-edge barriers; not in the reference)."""
        pid = C.c_int32()
        self._c(self.f["add_stencil_set"](self.ctx, union_id, int(arity), 1 if dynamic else 0, C.byref(pid)))
        self._arity[pid.value] = int(arity)
        return pid.value

    def set_stencil_primitives(self, stencils: int, kind: str, prims_a, prims_b=None):
        """Candidate primitives (union indices): kind "pt" (points, triangles),
        "ee" (edges; self-contact), "pe" (points, edges)."""
        k = {"pt": 1, "ee": 2, "pe": 3}[kind]
        a = _i64(prims_a)
        b = _i64(prims_b if prims_b is not None else [])
        na = len(a) // (2 if k == 2 else 1)
        nb = len(b) // (3 if k == 1 else 2)
        self._c(self.f["set_stencil_primitives"](self.ctx, stencils, k, na, _ip64(a), nb, _ip64(b)))

    def refresh_stencils(self, stencils: int, dhat: float) -> int:
        """Device contact candidates of a stencil set (resize_dynamic)."""
        n = C.c_int64()
        self._c(self.f["refresh_stencils"](self.ctx, stencils, float(dhat), C.byref(n)))
        return n.value

    def set_pairs(self, pairset: int, pairs):
        p = _i64(pairs)
        self._c(self.f["set_pairs"](self.ctx, pairset, len(p) // self._arity.get(pairset, 2), _ip64(p)))

    def pair_count(self, pairset: int) -> int:
        n = C.c_int64()
        self._c(self.f["pair_count"](self.ctx, pairset, C.byref(n)))
        return n.value

    def get_pairs(self, pairset: int) -> np.ndarray:
        n = self.pair_count(pairset)
        a = self._arity.get(pairset, 2)
        out = np.zeros(a * n, dtype=np.int64)
        if n:
            self._c(self.f["get_pairs"](self.ctx, pairset, _ip64(out)))
        return out.reshape(n, a)

    def refresh_pairs(self, pairset: int, dhat: float, child_is_fixed=None) -> int:
        n = C.c_int64()
        if child_is_fixed is None:
            fx = None
        else:
            a = np.ascontiguousarray(np.asarray(child_is_fixed, dtype=np.int32))
            fx = _ip32(a)
        self._c(self.f["refresh_pairs"](self.ctx, pairset, float(dhat), fx, C.byref(n)))
        return n.value

    def _eid(self, name: str, out: C.c_int32) -> int:
        self.energy_names.append(name)
        return out.value

    def add_stable_neo_hookean(self, pos_target: int, t2v, rest, youngs: float, poisson: float,
                               weight: float = 1.0, via_deformation_gradient: bool = False) -> int:
        t = _i64(t2v)
        r = _f64(rest)
        e = C.c_int32()
        self._c(self.f["add_stable_neo_hookean"](self.ctx, pos_target, len(t) // 4, _ip64(t), _dp(r),
                                                 float(youngs), float(poisson), float(weight),
                                                 1 if via_deformation_gradient else 0, C.byref(e)))
        return self._eid("stable_neo_hookean", e)

    def _contact(self, fn: str, name: str, stencils: int, dhat: float, kappa: float, weight: float) -> int:
        e = C.c_int32()
        self._c(self.f[fn](self.ctx, stencils, float(dhat), float(kappa), float(weight), C.byref(e)))
        return self._eid(name, e)

    def add_point_triangle_barrier(self, stencils: int, dhat: float, kappa: float, weight: float = 1.0) -> int:
        """Point-triangle barrier over an arity-4 stencil set (p, t0, t1, t2); not in the reference."""
        return self._contact("add_point_triangle_barrier", "point_triangle", stencils, dhat, kappa, weight)

    def add_edge_edge_barrier(self, stencils: int, dhat: float, kappa: float, weight: float = 1.0) -> int:
        """Edge-edge barrier over an arity-4 stencil set (a0, a1, b0, b1); not in the reference."""
        return self._contact("add_edge_edge_barrier", "edge_edge", stencils, dhat, kappa, weight)

    def add_point_edge_barrier(self, stencils: int, dhat: float, kappa: float, weight: float = 1.0) -> int:
        """Point-edge barrier over an arity-3 stencil set (p, e0, e1); not in the reference."""
        return self._contact("add_point_edge_barrier", "point_edge", stencils, dhat, kappa, weight)

    def add_point_point_barrier(self, pairset: int, dhat: float, kappa: float, weight: float = 1.0,
                                mode: int = YS_PROJECT_FULL) -> int:
        e = C.c_int32()
        self._c(self.f["add_point_point_barrier"](self.ctx, pairset, float(dhat), float(kappa), float(weight),
                                                  mode, C.byref(e)))
        return self._eid("point_point", e)

    def add_repulsive(self, pairset: int, weight: float = 1.0, mode: int = YS_PROJECT_FULL) -> int:
        e = C.c_int32()
        self._c(self.f["add_repulsive"](self.ctx, pairset, float(weight), mode, C.byref(e)))
        return self._eid("repulsive", e)

    def add_inertia(self, domain: int, mass, x_tilde) -> int:
        m = _f64(mass)
        x = _f64(x_tilde)
        e = C.c_int32()
        self._c(self.f["add_inertia"](self.ctx, domain, _dp(m), _dp(x), C.byref(e)))
        return self._eid("inertia", e)

    def set_inertia_anchor(self, energy: int, x_tilde):
        x = _f64(x_tilde)
        self._c(self.f["set_inertia_anchor"](self.ctx, energy, _dp(x)))

    def add_affine_orthogonality(self, amat_target: int, stiffness: float, weight: float = 1.0) -> int:
        e = C.c_int32()
        self._c(self.f["add_affine_orthogonality"](self.ctx, amat_target, float(stiffness), float(weight),
                                                   C.byref(e)))
        return self._eid("affine_orthogonality", e)

    def add_bending(self, pos_target: int, h2v, rest, stiffness: float, weight: float = 1.0) -> int:
        h = _i64(h2v)
        r = _f64(rest)
        e = C.c_int32()
        self._c(self.f["add_bending"](self.ctx, pos_target, len(h) // 4, _ip64(h), _dp(r), float(stiffness),
                                      float(weight), C.byref(e)))
        return self._eid("bending", e)

    # ---------------- engine side ----------------
    def finalize(self):
        self._c(self.f["finalize"](self.ctx))
        self.s = self.total_dofs()

    def refresh_dynamic(self):
        self._c(self.f["refresh_dynamic"](self.ctx))

    def dynamic_stale(self) -> bool:
        v = C.c_int32()
        self._c(self.f["dynamic_stale"](self.ctx, C.byref(v)))
        return bool(v.value)

    def assemble(self, project: bool = True, with_hessian: bool = True):
        self._c(self.f["assemble"](self.ctx, 1 if project else 0, 1 if with_hessian else 0))

    def gradient(self) -> np.ndarray:
        g = np.zeros(self.s)
        self._c(self.f["get_gradient"](self.ctx, _dp(g)))
        return g

    def total_energy(self) -> float:
        e = C.c_double()
        self._c(self.f["total_energy"](self.ctx, C.byref(e)))
        return e.value

    def energy_totals(self) -> np.ndarray:
        out = np.zeros(len(self.energy_names))
        self._c(self.f["energy_totals"](self.ctx, _dp(out)))
        return out

    def apply_hessian(self, x, y=None) -> np.ndarray:
        xv = _f64(x)
        yv = np.zeros(self.s) if y is None else _f64(y).copy()
        self._c(self.f["apply_hessian"](self.ctx, _dp(xv), _dp(yv)))
        return yv

    def minimize_step(self, tol: float = 1e-6, max_iter: int = -1, want_dx: bool = True) -> Step:
        st = StepStats()
        dx = np.zeros(self.s) if want_dx else None
        self._c(self.f["minimize_step"](self.ctx, float(tol), int(max_iter),
                                        _dp(dx) if want_dx else None, C.byref(st)))
        return Step(dx, st.pcg_iterations, st.pcg_residual, bool(st.pcg_converged), st.regularized_blocks,
                    st.assemble_seconds, st.solve_seconds)

    # ---------------- multi-GPU (row-partitioned PCG) ----------------
    def dist_init_nccl(self, rank: int, nranks: int, unique_id: bytes):
        """Solve with this rank's block rows, NCCL allgather on the engine's stream.
        unique_id: 128 bytes from dist_unique_id() on rank 0, broadcast by the caller."""
        if not self.lib.has("dist_init_nccl"):
            raise _lib.DeclError(f"{self.lib.path.name} has no NCCL transport")
        if len(unique_id) != 128:
            raise _lib.ValidationError("NCCL unique id must be 128 bytes")
        self._c(self.f["dist_init_nccl"](self.ctx, int(rank), int(nranks), bytes(unique_id)))

    def dist_init_host(self, rank: int, nranks: int, allgather):
        """Host transport: allgather(send (count,), recv (nranks, count)) fills recv
        rank-major from every rank's send (e.g. torch.distributed over gloo)."""
        def cb(_user, send, recv, count):
            try:
                s = np.ctypeslib.as_array(send, shape=(int(count),)) if count else np.zeros(0)
                r = np.ctypeslib.as_array(recv, shape=(int(nranks) * int(count),)) if count else np.zeros(0)
                allgather(s, r.reshape(int(nranks), int(count)))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status through the C-ABI
                import traceback
                traceback.print_exc()
                return 1
        self._dist_cb = _lib.ALLGATHER_FN(cb)  # keep the thunk alive
        self._c(self.f["dist_init_host"](self.ctx, int(rank), int(nranks), self._dist_cb, None))

    def dist_finalize(self):
        self._c(self.f["dist_finalize"](self.ctx))
        self._dist_cb = None

    # peer-memory transport: one persistent kernel per rank, NVLink P2P stores
    def dist_p2p_open(self, rank: int, nranks: int) -> bytes:
        """Allocate this rank's window; returns its 64-byte cudaIpcMemHandle."""
        if not self.lib.has("dist_p2p_open"):
            raise _lib.DeclError(f"{self.lib.path.name} has no peer-memory transport")
        buf = C.create_string_buffer(64)
        self._c(self.f["dist_p2p_open"](self.ctx, int(rank), int(nranks), buf))
        return buf.raw

    def dist_p2p_connect(self, handles: list[bytes]):
        """Map every peer's window (handles: one 64-byte handle per rank, rank order)."""
        table = b"".join(bytes(h) for h in handles)
        if any(len(h) != 64 for h in handles):
            raise _lib.ValidationError("cudaIpcMemHandle must be 64 bytes")
        self._c(self.f["dist_p2p_connect"](self.ctx, table))

    def dist_p2p_probe(self, read: bool) -> np.ndarray | None:
        """read=False: store rank+1 into every peer's probe slot; read=True: the slots peers wrote."""
        if not read:
            self._c(self.f["dist_p2p_probe"](self.ctx, None))
            return None
        seen = np.zeros(64, dtype=np.int64)
        self._c(self.f["dist_p2p_probe"](self.ctx, seen.ctypes.data_as(_lib._PI64)))
        return seen[:self.dist_info()["nranks"]]

    def dist_info(self) -> dict:
        rank, nranks = C.c_int32(), C.c_int32()
        bounds = np.zeros(65, dtype=np.int64)
        halo, exp = C.c_int64(), C.c_int64()
        self._c(self.f["dist_info"](self.ctx, C.byref(rank), C.byref(nranks), bounds.ctypes.data_as(_lib._PI64),
                                    C.byref(halo), C.byref(exp)))
        out = {"rank": rank.value, "nranks": nranks.value, "bounds": bounds[:nranks.value + 1].copy(),
               "halo_rows": halo.value, "export_rows": exp.value}
        if "dist_eval_counts" in self.f:
            ev, tot = C.c_int64(), C.c_int64()
            self._c(self.f["dist_eval_counts"](self.ctx, C.byref(ev), C.byref(tot)))
            out["eval_instances"], out["eval_total"] = ev.value, tot.value
        return out

    def split_per_target(self, flat: np.ndarray) -> list[np.ndarray]:
        out, off = [], 0
        for n, rc in self.targets:
            out.append(flat[off:off + n * rc])
            off += n * rc
        return out

    def pcg_history(self) -> np.ndarray:
        cnt = C.c_int64()
        cap = 1 << 20
        h = np.zeros(cap)
        self._c(self.f["pcg_history"](self.ctx, cap, _dp(h), C.byref(cnt)))
        return h[:min(cnt.value, cap)].copy()

    def gather_targets(self) -> np.ndarray:
        x = np.zeros(self.s)
        self._c(self.f["gather_targets"](self.ctx, _dp(x)))
        return x

    def scatter_targets(self, x):
        xv = _f64(x)
        if len(xv) != self.s:
            raise _lib.ValidationError("scatter_targets: length mismatch")
        self._c(self.f["scatter_targets"](self.ctx, _dp(xv)))

    def step_targets(self, alpha: float) -> float:
        m = C.c_double()
        self._c(self.f["step_targets"](self.ctx, float(alpha), C.byref(m)))
        return m.value

    # ---------------- introspection ----------------
    def hessian(self, which: int) -> HessianStructure:
        ng, nb, nv = C.c_int64(), C.c_int64(), C.c_int64()
        cs = C.c_uint64()
        self._c(self.f["hessian_info"](self.ctx, which, C.byref(ng), C.byref(nb), C.byref(nv), C.byref(cs)))
        groups = np.zeros(5 * ng.value, dtype=np.int64)
        row = np.zeros(nb.value, dtype=np.int64)
        col = np.zeros(nb.value, dtype=np.int64)
        vals = np.zeros(nv.value)
        if ng.value:
            self._c(self.f["hessian_groups"](self.ctx, which, _ip64(groups)))
        if nb.value:
            self._c(self.f["hessian_coords"](self.ctx, which, _ip64(row), _ip64(col)))
        if nv.value:
            self._c(self.f["hessian_values"](self.ctx, which, _dp(vals)))
        return HessianStructure(groups.reshape(-1, 5), row, col, vals, cs.value, self.s)

    def static_hessian(self) -> HessianStructure:
        return self.hessian(0)

    def dynamic_hessian(self) -> HessianStructure:
        return self.hessian(1)

    def dense_hessian(self) -> np.ndarray:
        """Engine::dense_hessian (engine.cpp:62)."""
        return self.static_hessian().to_dense() + self.dynamic_hessian().to_dense()

    def energy_info(self, e: int) -> dict:
        n, k, w, d = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        self._c(self.f["energy_info"](self.ctx, e, C.byref(n), C.byref(k), C.byref(w), C.byref(d)))
        return {"instances": n.value, "kappa": k.value, "width": w.value, "dynamic": bool(d.value)}

    def energy_slots(self, e: int):
        info = self.energy_info(e)
        cnt = info["instances"] * info["kappa"]
        idx = np.zeros(cnt, dtype=np.int64)
        ln = np.zeros(cnt, dtype=np.int32)
        col = np.zeros(cnt, dtype=np.int32)
        if cnt:
            self._c(self.f["energy_slots"](self.ctx, e, _ip64(idx), _ip32(ln), _ip32(col)))
        k = max(info["kappa"], 1)
        return idx.reshape(-1, k), ln.reshape(-1, k), col.reshape(-1, k)

    def energy_compressed_sizes(self, e: int) -> np.ndarray:
        n = self.energy_info(e)["instances"]
        m = np.zeros(n, dtype=np.int32)
        if n:
            self._c(self.f["energy_compressed_sizes"](self.ctx, e, _ip32(m)))
        return m

    def diag_blocks(self) -> list[np.ndarray]:
        total = sum(n * rc * rc for n, rc in self.targets)
        buf = np.zeros(total)
        self._c(self.f["diag_blocks"](self.ctx, _dp(buf)))
        out, off = [], 0
        for n, rc in self.targets:
            for _ in range(n):
                out.append(buf[off:off + rc * rc].reshape(rc, rc))
                off += rc * rc
        return out

    def device_bytes(self) -> int:
        b = C.c_int64()
        self._c(self.f["device_bytes"](self.ctx, C.byref(b)))
        return b.value

    def set_profiling(self, on: bool):
        if self.lib.has("set_profiling"):
            self._c(self.f["set_profiling"](self.ctx, 1 if on else 0))

    def bump_dynamic_epoch(self):
        self._c(self.f["bump_dynamic_epoch"](self.ctx))

    def stream_handle(self) -> int:
        h = C.c_void_p()
        self._c(self.f["stream"](self.ctx, C.byref(h)))
        return h.value or 0

    def set_option(self, name: str, value: int):
        """Execution options that do not change results (ys_set_option)."""
        self._c(self.f["set_option"](self.ctx, name.encode(), int(value)))

    def pcg_path(self) -> str:
        """Kernel path of the last uniform-3x3 solve."""
        ms = np.zeros(16)
        cnt = np.zeros(4, dtype=np.int64)
        self._c(self.f["stage_times"](self.ctx, _dp(ms), _ip64(cnt)))
        return {1: "sliced-ELL copy", 2: "row gather", 3: "peer-memory distributed"}.get(int(cnt[2]), "general")

    def time_kernel(self, which: int, reps: int = 20):
        ms, b = C.c_double(), C.c_double()
        self._c(self.f["time_kernel"](self.ctx, which, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def stage_times(self, with_counts: bool = False):
        ms = np.zeros(16)
        cnt = np.zeros(4, dtype=np.int64)
        self._c(self.f["stage_times"](self.ctx, _dp(ms), _ip64(cnt)))
        if with_counts:
            return ms, int(cnt[0]), int(cnt[1])
        return ms, int(cnt[0])

    def evd_fallbacks(self) -> int:
        """Indefinite elements of the last assembly projected by the Jacobi
        fallback instead of the clamped-eigenpair path."""
        ms = np.zeros(16)
        cnt = np.zeros(4, dtype=np.int64)
        self._c(self.f["stage_times"](self.ctx, _dp(ms), _ip64(cnt)))
        return int(cnt[3])


class BlockSystem:
    """Free-standing BlockSparseHessian + spmv_add + pcg (solver.hpp:13-48)."""

    def __init__(self, engine: Engine, total_dofs: int, coords):
        self.eng = engine
        self.s = int(total_dofs)
        c = _i64(coords)
        bid = C.c_int32()
        engine._c(engine.f["bsr_build"](engine.ctx, self.s, len(c) // 4, _ip64(c), C.byref(bid)))
        self.id = bid.value
        ng, nb, nv = C.c_int64(), C.c_int64(), C.c_int64()
        cs = C.c_uint64()
        engine._c(engine.f["bsr_info"](engine.ctx, self.id, C.byref(ng), C.byref(nb), C.byref(nv), C.byref(cs)))
        self.checksum = cs.value
        self.groups = np.zeros(5 * ng.value, dtype=np.int64)
        self.row = np.zeros(nb.value, dtype=np.int64)
        self.col = np.zeros(nb.value, dtype=np.int64)
        self.n_values = nv.value
        if ng.value:
            engine._c(engine.f["bsr_groups"](engine.ctx, self.id, _ip64(self.groups)))
            engine._c(engine.f["bsr_coords"](engine.ctx, self.id, _ip64(self.row), _ip64(self.col)))
        self.groups = self.groups.reshape(-1, 5)

    def value_offset(self, rows, cols, row, col) -> int:
        for r, c, cs, cnt, vs in self.groups:
            if r != rows or c != cols:
                continue
            lo, hi = cs, cs + cnt
            while lo < hi:
                mid = (lo + hi) // 2
                if (self.row[mid], self.col[mid]) < (row, col):
                    lo = mid + 1
                else:
                    hi = mid
            if lo < cs + cnt and self.row[lo] == row and self.col[lo] == col:
                return int(vs + (lo - cs) * r * c)
            break
        raise _lib.InternalError(f"block ({row},{col}) not present")

    def set_values(self, values):
        v = _f64(values)
        self.eng._c(self.eng.f["bsr_set_values"](self.eng.ctx, self.id, _dp(v)))

    def spmv(self, x, y=None) -> np.ndarray:
        xv = _f64(x)
        if len(xv) != self.s:
            raise _lib.ValidationError(f"spmv: vector length {len(xv)} != system size {self.s}")
        yv = np.zeros(self.s) if y is None else _f64(y).copy()
        self.eng._c(self.eng.f["bsr_spmv"](self.eng.ctx, self.id, _dp(xv), _dp(yv)))
        return yv

    def pcg(self, g, block_size: int, tol: float, max_iter: int):
        gv = _f64(g)
        x = np.zeros(self.s)
        it, rel, conv = C.c_int64(), C.c_double(), C.c_int32()
        self.eng._c(self.eng.f["bsr_pcg"](self.eng.ctx, self.id, int(block_size), _dp(gv), float(tol),
                                          int(max_iter), _dp(x), C.byref(it), C.byref(rel), C.byref(conv)))
        return x, it.value, rel.value, bool(conv.value)


def p2p_group(engines: list["Engine"]):
    """Make the engines (one process, one device, the same scene) the ranks of
    the peer-memory solve; step them with p2p_group_step (the one-GPU
    emulation of a multi-GPU job: one cooperative launch runs every rank)."""
    n = len(engines)
    arr = (C.c_void_p * n)(*[e.ctx for e in engines])
    check(engines[0].lib, engines[0].ctx, engines[0].f["dist_p2p_group"](arr, n))


def p2p_group_step(engines: list["Engine"], tol: float, max_iter: int = -1, want_dx: bool = True) -> list[Step]:
    n = len(engines)
    arr = (C.c_void_p * n)(*[e.ctx for e in engines])
    dxs = [np.zeros(e.s) for e in engines] if want_dx else None
    dxp = (_lib._PD * n)(*[_dp(d) for d in dxs]) if want_dx else None
    stats = (StepStats * n)()
    check(engines[0].lib, engines[0].ctx,
          engines[0].f["dist_p2p_group_step"](arr, n, float(tol), int(max_iter), dxp, stats))
    return [Step(dxs[k] if want_dx else None, stats[k].pcg_iterations, stats[k].pcg_residual,
                 bool(stats[k].pcg_converged), stats[k].regularized_blocks, stats[k].assemble_seconds,
                 stats[k].solve_seconds) for k in range(n)]
