#!/usr/bin/env python
"""Benchmark: ms per Newton iteration (eval + assembly + PCG) of the YASPS
hot path on B200 (BASELINE.json metric), with SpMV / assembly HBM GB/s
against the measured peak.

A step is one Engine::minimize_step (engine.cpp:75-101) — dynamic structure
rebuild, local evaluation, assembly, block-Jacobi build and PCG to pcg_tol —
on the prepared state of the selected scene (default C5, the 1M-tet pile).
Every step rebuilds the dynamic structure (the reference rebuilds it every
Newton iteration because each pair refresh bumps the dynamic epoch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

N > 1 (torchrun): the same scene on every rank, solved by the row-partitioned
multi-GPU PCG over NCCL ("strong": each rank evaluates the static stencil
instances touching its rows and solves its rows).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np


def simulation(cfg, backend: str = "gpu", **kw):
    """The product Simulation on the B200 library; backend "oracle" injects the
    CPU oracle (test infrastructure: the CPU baseline / reference arm only)."""
    from paper_2605_23088_b200.scene import Simulation
    lib = None
    if backend == "oracle":
        import oracle
        lib = oracle.library()
    return Simulation(cfg, library=lib, **kw)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per Newton iteration (eval+assembly+PCG); SpMV/assembly HBM GB/s vs peak"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c5")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--via-f", type=int, default=1)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--state", default="rollout", choices=["rollout", "jitter"])
    p.add_argument("--frames", type=int, default=None, help="rollout frames (default: the config's, 25 for C5)")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                   help="N>1: peer-memory persistent solve (default) or the NCCL-allgather loop")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def scene_config(name: str, via_f: bool):
    from paper_2605_23088_b200 import configs
    fn = configs.CONFIGS[name]
    try:
        return fn(via_f=via_f)
    except TypeError:
        return fn()


def jitter_amplitude(name: str) -> float:
    return 0.1 * (0.025 if name == "c1" else 0.02 if name == "c3" else 0.01)


def prepare(name: str, via_f: bool, backend: str, device: int = 0, state: str = "rollout", frames: int | None = None):
    """Scene + prepared state ("time from a prepared state").

    state "rollout" (default): the scene's first `frames` frames (config
    `frames`, 25 for C5 as in test_acceptance.cpp:460) simulated on the B200
    library — Newton + line search + contact refresh per iteration, bitwise
    deterministic — then begin_frame of the next frame and its contact pairs.
    The oracle side ("oracle") takes that state over (positions, velocities,
    then its own begin_frame) and refreshes its pairs with the reference's
    all-pairs loop: the O(n^2) refresh and ~8 s Newton iterations make a CPU
    rollout of C5 impractical (CPU baseline).
    state "jitter" (round 1): seeded jitter of the soft vertices at rest."""
    if state == "jitter":
        return _jitter_state(name, via_f, backend, device)
    gsim = rollout(name, via_f, device, frames)
    if backend == "gpu":
        return gsim
    return oracle_from(gsim, name, via_f)


def _jitter_state(name, via_f, backend, device):
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig
    cfg = SimConfig.from_dict(scene_config(name, via_f))
    sim = simulation(cfg, backend, device=device, refresh_pairs=False)
    configs.jitter_targets(sim, jitter_amplitude(name))
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    return sim


def rollout(name: str, via_f: bool, device: int = 0, frames: int | None = None):
    from paper_2605_23088_b200.scene import SimConfig
    cfg = SimConfig.from_dict(scene_config(name, via_f))
    sim = simulation(cfg, "gpu", device=device)
    sim.prepared_frames = cfg.frames if frames is None else frames
    sim.rollout_newton = 0
    for _ in range(sim.prepared_frames):
        sim.rollout_newton += sim.step().iterations
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    return sim


def oracle_from(src, name: str, via_f: bool, pairs=None):
    """An oracle Simulation in the state of `src` (a prepared GPU Simulation):
    target values and body velocities copied, begin_frame recomputed on the
    host (the same numpy arithmetic: identical x_tilde), contact pairs from the
    reference's all-pairs loop or, when given, the GPU's (bit-identical list,
    tests/test_gpu_large.py)."""
    from paper_2605_23088_b200.scene import SimConfig
    cfg = SimConfig.from_dict(scene_config(name, via_f))
    sim = simulation(cfg, "oracle", refresh_pairs=False)
    for bs, bd in zip(src.bodies, sim.bodies):
        for t in bs.targets:
            sim.eng.set_target_values(t, src.eng.get_target_values(t))
        if bs.velocity is not None:
            bd.velocity = np.array(bs.velocity, copy=True)
    sim.begin_frame()
    if sim.contact_pairset >= 0:
        if pairs is None:
            sim.refresh_dynamic_pairs()
        else:
            sim.eng.set_pairs(sim.contact_pairset, pairs)
    sim.prepared_frames = getattr(src, "prepared_frames", 0)
    return sim


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 7 for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def traffic_from_profiles(scene: str, key: str):
    """DRAM bytes (read + write) from the committed ncu capture (profiles/ncu_summary.json):
    "pcg_dram_bytes_per_iteration" of the persistent PCG kernel, "spmv_dram_bytes" per SpMV launch."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(scene, {}).get(key)
    except Exception:
        return None


def cpu_threads() -> int:
    """All host threads, as the reference configured with "threads" = nproc:
    instance evaluation (parallel_for, assembly.cpp:334-336) and the sharded
    spmv_add (solver.cpp:63-81); the scatter and the PCG vector updates stay
    serial, as in the reference."""
    n = int(os.environ.get("YO_THREADS") or os.cpu_count() or 1)
    os.environ["YO_THREADS"] = str(n)
    os.environ["YO_SPMV_THREADS"] = str(n)
    return n


def cpu_step(sim):
    """One Newton iteration of the oracle, timed on the host (perf_counter)."""
    eng = sim.eng
    eng.bump_dynamic_epoch()
    t0 = time.perf_counter()
    st = eng.minimize_step(sim.config.pcg_tol, -1, want_dx=False)
    return 1e3 * (time.perf_counter() - t0), st


def cpu_sample(gsim, name: str, via_f: bool):
    """Bounded CPU sample for the GPU arm: ONE full-scene Newton iteration of the
    same workload (the GPU arm's prepared state, its bit-identical pair list) on
    the oracle port, on all host threads (~10-20 s at C5)."""
    threads = cpu_threads()
    sim = oracle_from(gsim, name, via_f, _read_pairs(gsim) if gsim.contact_pairset >= 0 else None)
    ms, st = cpu_step(sim)
    return {"value": ms, "unit": "ms", "cores": threads, "kind": "port",
            "sample": (f"{name}: one full Newton iteration (minimize_step: dynamic rebuild, instance evaluation on "
                       f"{threads} threads, assembly, block-Jacobi, PCG with {threads}-shard spmv_add: "
                       f"{st.pcg_iterations} iterations) of the whole scene on the oracle port — the reference's "
                       f"algorithm restated in C, pinned to the reference built from its sources")}


def run_reference(args):
    """The reference arm: full-scene Newton iterations of the reference's
    algorithm on the host cores (the oracle port; the reference itself, built
    here against eigen-lite, is validated against it but its interpreted plans
    make a C5 step take tens of minutes), W untimed + K timed steps of the same
    workload as the GPU arm, from the same prepared state."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = cpu_threads()
    t0 = time.perf_counter()
    gsim = rollout(args.config, bool(args.via_f), 0, args.frames) if args.state == "rollout" else None
    prep_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    if gsim is not None:
        sim = oracle_from(gsim, args.config, bool(args.via_f))
        gsim.eng.close()
    else:
        sim = _jitter_state(args.config, bool(args.via_f), "oracle", 0)
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        cpu_step(sim)
    vals, iters = [], []
    for _ in range(args.steps):
        ms, st = cpu_step(sim)
        vals.append(ms)
        iters.append(st.pcg_iterations)
    v = float(statistics.mean(vals))
    cb = {"value": v, "unit": "ms", "cores": threads, "kind": "port",
          "sample": (f"{args.config}: the full scene, {args.warmup} untimed + {args.steps} timed Newton iterations "
                     f"(minimize_step) on {threads} host threads; PCG iterations {int(np.median(iters))}; "
                     f"setup (scene build + the reference's all-pairs contact refresh) {setup_s:.1f} s untimed; "
                     + (f"state: {args.frames if args.frames is not None else 'config'} frames rolled out on the B200 "
                        f"library ({prep_s:.1f} s untimed, deterministic) and taken over by the port"
                        if gsim is not None else "state: seeded jitter at rest"))}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args.config, args.state, sim), "scene": args.config, "dofs": int(sim.eng.s),
                       "contact_pairs": int(sim.pair_count()), "pcg_iterations": int(np.median(iters)),
                       "pcg_iterations_per_step": [int(i) for i in iters], "ms_per_step_min": min(vals),
                       "ms_per_step_max": max(vals), "nh_via_deformation_gradient": bool(args.via_f),
                       "parallelism": f"host threads {threads}"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload(name: str, state: str = "rollout", sim=None) -> str:
    if state == "jitter":
        where = "from a jittered rest state"
    else:
        where = f"from the prepared state after {getattr(sim, 'prepared_frames', '?')} simulated frames"
    return (f"{name}: one Newton iteration (dynamic rebuild + eval + assembly + block-Jacobi + PCG to pcg_tol) "
            + where)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch itself as N ranks (one
    process per GPU) through torch.distributed.run; the driver's own torchrun
    launch sets WORLD_SIZE and skips this."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world_env:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    from paper_2605_23088_b200 import _lib
    t_prep = time.perf_counter()
    sim = prepare(args.config, bool(args.via_f), "gpu", local, args.state, args.frames)
    t_prep = time.perf_counter() - t_prep
    eng = sim.eng
    if world > 1:
        from paper_2605_23088_b200 import dist as ysdist
        if args.transport == "p2p" and not ysdist.init_p2p(eng):
            args.transport = "nccl (peer memory unavailable on this node)"  # said on stderr by init_p2p
        if not args.transport.startswith("p2p"):
            ysdist.init_nccl(eng)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=torch.device("cuda", local))
    cfg = sim.config

    def step():
        eng.bump_dynamic_epoch()
        return eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)

    # ncu --profile-from-start off: the launch list starts here (after the
    # rollout that prepares the state); a no-op without a profiler
    try:
        import ctypes
        ctypes.CDLL("libcuda.so.1").cuProfilerStart()
    except OSError:
        pass
    for _ in range(max(3, args.warmup)):
        st = step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    eng.set_profiling(False)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    iters = []
    launches = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            st = step()
            iters.append(st.pcg_iterations)
        e1.record(stream)
        torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    # per-stage device times and launch count of one more step
    eng.set_profiling(True)
    st = step()
    stages, launches_per_step = eng.stage_times()
    eng.set_profiling(False)

    peak, peak_src = load_peaks()
    try:
        spmv_ms, spmv_bytes = eng.time_kernel(3, 50)  # the PCG's SpMV: sliced-ELL copy, 4 lanes per row
        spmv_kind = "k_spmv_sell<4> (sliced-ELL full copy of static + dynamic H), timed alone"
    except _lib.ValidationError:  # mixed block sizes (C3: affine bodies): the row-gather SpMV
        spmv_ms, spmv_bytes = eng.time_kernel(0, 50)
        spmv_kind = "k_spmv_gen (row gather from upper storage, per block-size class), timed alone"
    asm_ms, asm_bytes = eng.time_kernel(1, 10)
    eval_ms, _ = eng.time_kernel(2, 5)
    fp64_ms, fp64_flops = eng.time_kernel(4, 5)  # FP64 FMA peak probe (this box, this run)
    fp64_peak = fp64_flops / (fp64_ms * 1e-3) / 1e12
    eval_flops = traffic_from_profiles(args.config, "eval_flops_per_step")
    spmv_gbs = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    asm_gbs = asm_bytes / (asm_ms * 1e-3) / 1e9
    # The dominant kernel is the PCG (one persistent cooperative launch per
    # solve for uniform 3x3 systems).  Algorithmic bytes per iteration
    # (SURVEY §8(d)): the SpMV's 8 r c + 8 per upper block + 16 s, the
    # block-Jacobi apply's 72 B per 3x3 inverse + 16 s, 6 vector passes 48 s.
    nb = eng.s // 3
    pcg_iter_bytes = spmv_bytes + 72.0 * nb + 16.0 * eng.s + 48.0 * eng.s
    pcg_ms = stages[4]
    pcg_path = eng.pcg_path()
    pcg_gbs = pcg_iter_bytes * st.pcg_iterations / (pcg_ms * 1e-3) / 1e9

    # e2e through the C-ABI with pinned host buffers: positions + pair table in, dx out
    e2e = None
    if not args.no_e2e:
        x_host = torch.from_numpy(eng.gather_targets()).pin_memory()
        pairs = sim.eng.pair_count(sim.contact_pairset) if sim.contact_pairset >= 0 else 0
        dx_host = torch.empty(eng.s, dtype=torch.float64).pin_memory()
        import ctypes as C
        from paper_2605_23088_b200._lib import StepStats
        f = eng.f
        xp = C.cast(x_host.data_ptr(), C.POINTER(C.c_double))
        dp = C.cast(dx_host.data_ptr(), C.POINTER(C.c_double))
        pair_tab = None
        if pairs:
            # the current pair table, re-sent every step as the step's contact input
            pair_tab = np.asarray(_read_pairs(sim), dtype=np.int64)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            eng._c(f["scatter_targets"](eng.ctx, xp))
            if pair_tab is not None:
                eng.set_pairs(sim.contact_pairset, pair_tab)
            stt = StepStats()
            eng._c(f["minimize_step"](eng.ctx, float(cfg.pcg_tol), -1, dp, C.byref(stt)))
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(8 * eng.s + 16 * pairs),
               "d2h_bytes_per_step": int(8 * eng.s)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(sim, args.config, bool(args.via_f))
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": "ms", "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    stats_tets = sum(int(b.get("nx", 0)) * int(b.get("ny", 0)) * int(b.get("nz", 0)) * 6
                     for b in cfg.bodies if b.get("kind") == "tet_block")
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": ms_step, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(args.config, args.state, sim),
                   "scene": args.config, "tets": stats_tets, "dofs": int(eng.s),
                   "contact_pairs": int(sim.pair_count()), "pcg_iterations": int(np.median(iters)),
                   "nh_via_deformation_gradient": bool(args.via_f),
                   "prepared_frames": getattr(sim, "prepared_frames", 0),
                   "prepare_s": round(t_prep, 2),
                   "l2": "inputs larger than L2 (device working set %.2f GB >> 126 MB)" % (eng.device_bytes() / 1e9),
                   "parallelism": (f"rows{world}: owned-row evaluation + row-partitioned PCG ({args.transport})"
                                   if world > 1 else "single")},
        "roofline": {"kernel": ("k_pcg33_stream<SellPhaseA> (whole PCG solve over the sliced-ELL copy, one cooperative launch; avg_launch_ms = the solve stage: k_pcg_init + the persistent kernel; the copy's value fill runs before it, beside the preconditioner build)"
                                if pcg_path == "sliced-ELL copy" else
                                "k_pcg_gen_persistent (whole PCG solve, warp per block row of each block-size class, one cooperative launch)")
                     if world == 1 else
                     ("row-partitioned PCG: one persistent k_dpcg_p2p per rank, NVLink peer-memory exchanges"
                      if args.transport == "p2p" else
                      "row-partitioned PCG (k_dspmv_sell / k_dupdate per rank + NCCL allgather)"),
                     "bound": "hbm", "achieved": pcg_gbs, "peak": peak, "unit": "GB/s", "frac": pcg_gbs / peak,
                     "traffic": traffic_from_profiles(args.config, "pcg_dram_bytes_per_iteration"),
                     "algorithmic_bytes": pcg_iter_bytes,
                     "algorithmic_bytes_unit": "per PCG iteration", "iterations": int(st.pcg_iterations),
                     "avg_launch_ms": pcg_ms, "peak_source": peak_src,
                     "spmv": {"kernel": spmv_kind,
                              "achieved": spmv_gbs, "frac": spmv_gbs / peak, "algorithmic_bytes": spmv_bytes,
                              "traffic": traffic_from_profiles(args.config, "spmv_dram_bytes"),
                              "avg_launch_ms": spmv_ms}},
        "assembly_roofline": {"bound": "hbm", "achieved": asm_gbs, "peak": peak, "unit": "GB/s",
                              "frac": asm_gbs / peak, "algorithmic_bytes": asm_bytes, "avg_ms": asm_ms},
        "eval_ms": eval_ms,
        "eval_roofline": {"bound": "fp64", "kernel": "k_eval_* (pass A: gradient + H_D + Cholesky test; pass B: clamped-eigenpair projection of the indefinite 9x9 elements, Jacobi fallback; point terms)",
                          "achieved": (eval_flops / (eval_ms * 1e-3) / 1e12) if eval_flops else None,
                          "peak": fp64_peak, "unit": "TFLOP/s",
                          "frac": (eval_flops / (eval_ms * 1e-3) / 1e12 / fp64_peak) if eval_flops else None,
                          "flops_per_launch": eval_flops, "avg_launch_ms": eval_ms,
                          "flops_source": "ncu SASS counts 2 DFMA + DADD + DMUL of every k_eval* launch of one step (profiles/ncu_summary.json)",
                          "peak_source": "measured: k_dfma_probe (8 independent DFMA chains per thread, 8 CTAs of 256 per SM) timed in this run"},
        "stages_ms": {"refresh_dynamic": stages[0], "local_eval": stages[1], "assembly_gather": stages[2],
                      "gradient_diag_precond": stages[3], "pcg": stages[4], "total": stages[6]},
        "gpu_launches": int(launches_per_step * args.steps),
        "pcg_driver": "persistent cooperative kernel" if world == 1 else f"row-partitioned over {world} ranks",
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
        "library": _lib.gpu_library().fns["version"]().decode(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _read_pairs(sim):
    """Current pair table of the contact pair set (the e2e leg re-sends it)."""
    return sim.eng.get_pairs(sim.contact_pairset).reshape(-1)


if __name__ == "__main__":
    main()
