"""Row-partitioned solve of a scene's rolled-out state with N ranks sharing
cuda:0 (host allgather over gloo) against the single-GPU solve (development
aid; tests/test_dist.py covers C1).  usage: python tools/dist_scene.py c5 2"""
import os
import sys
import time

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, name, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from bench import prepare
        from paper_2605_23088_b200 import dist as ysdist
        sim = prepare(name, True, "gpu")
        if world > 1:
            ysdist.init_host(sim.eng)
        t0 = time.perf_counter()
        st = sim.eng.minimize_step(sim.config.pcg_tol)
        out.put((rank, st.pcg_iterations, st.dx, sim.eng.dist_info(), time.perf_counter() - t0))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ctx = mp.get_context("spawn")
    res = {}
    for w in (1, world):
        q = ctx.Queue()
        port = 29800 + w
        ps = [ctx.Process(target=worker, args=(r, w, port, name, q)) for r in range(w)]
        for p in ps:
            p.start()
        res[w] = [q.get(timeout=1200) for _ in range(w)]
        for p in ps:
            p.join(timeout=120)
    ref = res[1][0]
    for rank, it, dx, info, dt in sorted(res[world], key=lambda r: r[0]):
        print(f"rank {rank}: iterations {it} (1 GPU {ref[1]}), dx rel {np.max(np.abs(dx - ref[2])) / np.max(np.abs(ref[2])):.2e}, "
              f"rows {info['bounds'][rank]}..{info['bounds'][rank + 1]}, halo {info['halo_rows']}, export {info['export_rows']}, "
              f"evaluated {info.get('eval_instances')} of {info.get('eval_total')}, step {dt * 1e3:.1f} ms (host transport)")
