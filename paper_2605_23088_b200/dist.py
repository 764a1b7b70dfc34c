"""One process per GPU: wiring the engine's row-partitioned PCG to
torch.distributed.

`init_nccl(eng)` is the production path: rank 0 asks the library for an NCCL
unique id, the process group broadcasts it, and the library then runs its own
ncclAllGather on the engine's stream.  `init_host(eng)` routes the same
allgather through torch.distributed on host buffers — any backend, used by the
multi-process tests (gloo, several ranks sharing one device)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def unique_id(lib: _lib.Library | None = None) -> bytes:
    lib = lib or _lib.gpu_library()
    if not lib.has("dist_unique_id"):
        raise _lib.DeclError(f"{lib.path.name} has no NCCL transport")
    buf = C.create_string_buffer(128)
    st = lib.fns["dist_unique_id"](buf)
    if st != 0:
        raise _lib.CudaError("ncclGetUniqueId failed (is libnccl.so.2 loadable?)")
    return buf.raw


def init_nccl(eng, group=None):
    import torch
    import torch.distributed as dist
    rank, n = dist.get_rank(group), dist.get_world_size(group)
    uid = unique_id(eng.lib) if rank == 0 else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, 0, group=group)
    eng.dist_init_nccl(rank, n, bytes(t.cpu().numpy().tobytes()))


def torch_allgather(group=None):
    """allgather(send, recv) over torch.distributed on host tensors."""
    import torch
    import torch.distributed as dist

    def ag(send: np.ndarray, recv: np.ndarray):
        outs = [torch.from_numpy(recv[k]) for k in range(recv.shape[0])]
        dist.all_gather(outs, torch.from_numpy(np.ascontiguousarray(send)), group=group)
    return ag


def init_host(eng, group=None):
    import torch.distributed as dist
    eng.dist_init_host(dist.get_rank(group), dist.get_world_size(group), torch_allgather(group))


def init_p2p(eng, group=None) -> bool:
    """Peer-memory transport (production multi-GPU path on one NVSwitch node):
    every rank allocates its window, the 64-byte cudaIpcMemHandles are
    all-gathered over the process group, every rank maps its peers' windows.
    The solve then runs as one persistent kernel per rank exchanging through
    NVLink stores and device-side flags.  Returns True on every rank when every
    rank mapped every peer; otherwise every rank returns False with its windows
    released (collective decision: no rank is left waiting on another)."""
    import torch.distributed as dist
    rank, n = dist.get_rank(group), dist.get_world_size(group)
    handle = eng.dist_p2p_open(rank, n)
    handles = [None] * n
    dist.all_gather_object(handles, handle, group=group)
    why = ""
    try:
        eng.dist_p2p_connect(handles)
    except Exception as e:  # noqa: BLE001 - decided collectively below
        why = repr(e)
    oks = [None] * n
    dist.all_gather_object(oks, why, group=group)  # also the barrier: every window mapped before any store
    bad = [w for w in oks if w]
    if bad:
        eng.dist_finalize()
        import sys
        print(f"yasps_b200: peer-memory transport unavailable ({bad[0]})", file=sys.stderr)
        return False
    return True
