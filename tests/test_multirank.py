"""world_size-2 gloo test of bench.py's rank plumbing (CPU): identical scene
replicas on every rank and the max-over-ranks reduction the bench uses for
its timing.  The row-partitioned solve itself is tested in test_dist.py."""
from __future__ import annotations

import os
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig
    from backends import simulation
    sim = simulation(SimConfig.from_dict(configs.c1()), "oracle")
    configs.jitter_targets(sim, 0.0025)
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    st = sim.eng.minimize_step(1e-4)
    t = torch.tensor([float(st.pcg_iterations), float(abs(st.dx).max()), float(rank + 1)])
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    mn = t.clone()
    dist.all_reduce(mn, op=dist.ReduceOp.MIN)
    if rank == 0:
        out.put((mx.tolist(), mn.tolist()))
    dist.destroy_process_group()


def test_two_rank_replicas_agree():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    mx, mn = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert mx[0] == mn[0] and mx[1] == mn[1]  # identical replicas
    assert mx[2] == 2.0  # max over ranks
