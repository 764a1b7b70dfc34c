"""ctypes binding of the C-ABI declared in include/yasps_b200.h.

The product loads ``libyasps_b200.so`` (prefix ``ys_``) and raises if it is
missing — there is no CPU fallback.  ``Library`` binds any implementation of
the same ABI; the test infrastructure under oracle/ uses it for the CPU oracle
(``yo_``) and injects it into ``Engine`` — the product never loads it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libyasps_b200.so"


# --- error classes mirroring relsim (core.hpp:33-71) -----------------------
class Error(RuntimeError):
    pass


class UserError(Error):
    pass


class ValidationError(UserError):
    pass


class DeclError(UserError):
    pass


class NumericalError(Error):
    pass


class InternalError(Error):
    pass


class CudaError(Error):
    pass


_ERRORS = {1: ValidationError, 2: DeclError, 3: NumericalError, 4: InternalError, 5: CudaError}

YS_PROJECT_FULL = 0
YS_PROJECT_REDUCED = 1
YS_POINTS_FREE = 0
YS_POINTS_AFFINE = 1
YS_POINTS_FIXED = 2


class StepStats(C.Structure):
    _fields_ = [
        ("pcg_iterations", C.c_int64),
        ("pcg_residual", C.c_double),
        ("pcg_converged", C.c_int32),
        ("regularized_blocks", C.c_int32),
        ("assemble_seconds", C.c_double),
        ("solve_seconds", C.c_double),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_PI32 = C.POINTER(C.c_int32)
_PI64 = C.POINTER(C.c_int64)
_PU64 = C.POINTER(C.c_uint64)
_PD = C.POINTER(C.c_double)
# ys_allgather_fn: int (*)(void* user, const double* send, double* recv, int64_t count)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _PD, _PD, C.c_int64)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "create": [C.POINTER(_P), _I32],
    "destroy": [_P],
    "last_error": [_P],
    "last_error_class": [_P],
    "version": [],
    "add_target": [_P, _I64, _I32, _PI32],
    "set_target_values": [_P, _I32, _PD],
    "get_target_values": [_P, _I32, _PD],
    "total_dofs": [_P, _PI64],
    "add_points": [_P, _I32, _I64, _I32, _I32, _PI64, _PD, _PI32],
    "get_points": [_P, _I32, _PD],
    "add_point_union": [_P, _I32, _PI32, _PI32],
    "add_pair_set": [_P, _I32, _I32, _PI32],
    "add_stencil_set": [_P, _I32, _I32, _I32, _PI32],
    "set_pairs": [_P, _I32, _I64, _PI64],
    "pair_count": [_P, _I32, _PI64],
    "get_pairs": [_P, _I32, _PI64],
    "refresh_pairs": [_P, _I32, _D, _PI32, _PI64],
    "set_stencil_primitives": [_P, _I32, _I32, _I64, _PI64, _I64, _PI64],
    "refresh_stencils": [_P, _I32, _D, _PI64],
    "add_stable_neo_hookean": [_P, _I32, _I64, _PI64, _PD, _D, _D, _D, _I32, _PI32],
    "add_point_point_barrier": [_P, _I32, _D, _D, _D, _I32, _PI32],
    "add_repulsive": [_P, _I32, _D, _I32, _PI32],
    "add_point_triangle_barrier": [_P, _I32, _D, _D, _D, _PI32],
    "add_edge_edge_barrier": [_P, _I32, _D, _D, _D, _PI32],
    "add_point_edge_barrier": [_P, _I32, _D, _D, _D, _PI32],
    "add_inertia": [_P, _I32, _PD, _PD, _PI32],
    "set_inertia_anchor": [_P, _I32, _PD],
    "add_affine_orthogonality": [_P, _I32, _D, _D, _PI32],
    "add_bending": [_P, _I32, _I64, _PI64, _PD, _D, _D, _PI32],
    "finalize": [_P],
    "refresh_dynamic": [_P],
    "dynamic_stale": [_P, _PI32],
    "assemble": [_P, _I32, _I32],
    "get_gradient": [_P, _PD],
    "total_energy": [_P, _PD],
    "energy_totals": [_P, _PD],
    "apply_hessian": [_P, _PD, _PD],
    "minimize_step": [_P, _D, _I64, _PD, C.POINTER(StepStats)],
    "pcg_history": [_P, _I64, _PD, _PI64],
    "gather_targets": [_P, _PD],
    "scatter_targets": [_P, _PD],
    "step_targets": [_P, _D, _PD],
    "hessian_info": [_P, _I32, _PI64, _PI64, _PI64, _PU64],
    "hessian_groups": [_P, _I32, _PI64],
    "hessian_coords": [_P, _I32, _PI64, _PI64],
    "hessian_values": [_P, _I32, _PD],
    "energy_info": [_P, _I32, _PI64, _PI32, _PI32, _PI32],
    "energy_slots": [_P, _I32, _PI64, _PI32, _PI32],
    "energy_compressed_sizes": [_P, _I32, _PI32],
    "diag_blocks": [_P, _PD],
    "device_bytes": [_P, _PI64],
    "bsr_build": [_P, _I64, _I64, _PI64, _PI32],
    "bsr_info": [_P, _I32, _PI64, _PI64, _PI64, _PU64],
    "bsr_groups": [_P, _I32, _PI64],
    "bsr_coords": [_P, _I32, _PI64, _PI64],
    "bsr_set_values": [_P, _I32, _PD],
    "bsr_spmv": [_P, _I32, _PD, _PD],
    "bsr_pcg": [_P, _I32, _I32, _PD, _D, _I64, _PD, _PI64, _PD, _PI32],
    "set_profiling": [_P, _I32],
    "stage_times": [_P, _PD, _PI64],
    "bump_dynamic_epoch": [_P],
    "stream": [_P, C.POINTER(C.c_void_p)],
    "set_option": [_P, C.c_char_p, _I64],
    "time_kernel": [_P, _I32, _I32, _PD, _PD],
    "dist_unique_id": [C.c_char_p],
    "dist_init_nccl": [_P, _I32, _I32, C.c_char_p],
    "dist_init_host": [_P, _I32, _I32, ALLGATHER_FN, _P],
    "dist_finalize": [_P],
    "dist_info": [_P, _PI32, _PI32, _PI64, _PI64, _PI64],
    "dist_eval_counts": [_P, _PI64, _PI64],
    "dist_p2p_open": [_P, _I32, _I32, C.c_char_p],
    "dist_p2p_connect": [_P, C.c_char_p],
    "dist_p2p_probe": [_P, _PI64],
    "dist_p2p_group": [C.POINTER(_P), _I32],
    "dist_p2p_group_step": [C.POINTER(_P), _I32, _D, _I64, C.POINTER(_PD), C.POINTER(StepStats)],
}
_RESTYPES = {"destroy": None, "last_error": C.c_char_p, "version": C.c_char_p, "last_error_class": C.c_int}

# Functions the oracle does not implement (device-only instrumentation).
OPTIONAL = {"set_profiling", "stage_times", "device_bytes", "time_kernel", "stream", "set_option", "dist_unique_id",
            "dist_init_nccl", "dist_eval_counts", "dist_p2p_open", "dist_p2p_connect", "dist_p2p_probe",
            "dist_p2p_group", "dist_p2p_group_step"}


class Library:
    """A loaded C-ABI implementation (GPU library or oracle)."""

    def __init__(self, path: Path | str, prefix: str):
        path = Path(path)
        if not path.exists():
            raise FileNotFoundError(
                f"{path} is missing: build it first (python -m paper_2605_23088_b200.build); "
                "there is no fallback implementation")
        self.path = path
        self.prefix = prefix
        self.dll = C.CDLL(str(path))
        self.fns = {}
        for name, args in _SIGS.items():
            sym = prefix + name
            if not hasattr(self.dll, sym):
                if name in OPTIONAL:
                    continue
                raise AttributeError(f"{path.name} does not export {sym}")
            f = getattr(self.dll, sym)
            f.argtypes = args
            f.restype = _RESTYPES.get(name, C.c_int)
            self.fns[name] = f

    def has(self, name: str) -> bool:
        return name in self.fns

    def exported_symbols(self) -> list[str]:
        return [self.prefix + n for n in self.fns]


_LIBS: dict[str, Library] = {}


def gpu_library() -> Library:
    if "gpu" not in _LIBS:
        _LIBS["gpu"] = Library(LIB_PATH, "ys_")
    return _LIBS["gpu"]


def check(lib: Library, ctx, status: int):
    if status == 0:
        return
    msg = lib.fns["last_error"](ctx)
    msg = msg.decode() if msg else ""
    raise _ERRORS.get(status, Error)(msg)
