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
multi-GPU PCG over NCCL ("strong": evaluation and assembly replicated, the PCG
rows split across ranks).
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


def prepare(name: str, via_f: bool, backend: str, device: int = 0):
    """Scene + prepared state: seeded jitter of the soft vertices, x_tilde of
    frame 1 (begin_frame), contact pairs of that state."""
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig
    cfg = SimConfig.from_dict(scene_config(name, via_f))
    sim = simulation(cfg, backend, device=device, refresh_pairs=False)
    configs.jitter_targets(sim, jitter_amplitude(name))
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


def cpu_sample(name: str, via_f: bool, gpu_pcg_iterations: int, budget_s: float = 20.0):
    """Bounded CPU sample of the same workload on the host through the oracle
    port (the reference's algorithm restated in C; the reference itself cannot
    be built here): a single block of the scene (C5: one of the 8
    soft blocks) is assembled once, and the PCG's per-iteration cost is the
    difference of two solves capped at 2 and 42 iterations; both are scaled to
    the full scene and the GPU's PCG iteration count.  Like the reference's
    parallel_for, the oracle evaluates instances on all host threads
    (YO_THREADS caps them) and scatters / iterates serially."""
    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig
    backend, kind = "oracle", "port"
    full = scene_config(name, via_f)
    sub = dict(full)
    soft = [b for b in full["bodies"] if not b.get("fixed")]
    sub["bodies"] = [soft[0]] + [b for b in full["bodies"] if b.get("fixed")]
    sub["contact"] = dict(full["contact"], bodies=[soft[0]["name"]] + [b["name"] for b in full["bodies"] if b.get("fixed")])
    cfg = SimConfig.from_dict(sub)
    sim = simulation(cfg, backend, refresh_pairs=False)
    configs.jitter_targets(sim, jitter_amplitude(name))
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    eng = sim.eng
    threads = int(os.environ.get("YO_THREADS") or os.cpu_count() or 1)
    os.environ["YO_SPMV_THREADS"] = str(threads)  # the reference's threaded spmv_add (solver.cpp:63-81)
    eng.refresh_dynamic()
    t0 = time.perf_counter()
    eng.assemble(True, True)
    t_asm = time.perf_counter() - t0
    k1, k2 = 2, 42
    t0 = time.perf_counter()
    eng.minimize_step(1e-300, k1, want_dx=False)
    t_a = time.perf_counter() - t0
    t0 = time.perf_counter()
    eng.minimize_step(1e-300, k2, want_dx=False)
    t_b = time.perf_counter() - t0
    t_pcg_it = max(t_b - t_a, 0.0) / (k2 - k1)
    s_sub = eng.s
    scale = len(soft)
    ms = 1e3 * (t_asm * scale + t_pcg_it * scale * gpu_pcg_iterations)
    return {"value": ms, "unit": "ms", "cores": threads, "kind": kind,
            "sample": (f"{name} single soft body ({s_sub} DoFs, 1/{scale} of the scene): one assembly "
                       f"({t_asm:.2f}s, instance evaluation on {threads} threads) + PCG iterations (SpMV sharded over {threads} threads, "
                       f"{t_pcg_it*1e3:.2f} ms each, from solves capped at {k1} and {k2}), scaled x{scale} and to "
                       f"the GPU's {gpu_pcg_iterations} PCG iterations; oracle port library")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # a step = one bounded CPU sample; iteration counts from the oracle itself
    from paper_2605_23088_b200.scene import SimConfig  # noqa: F401
    vals = []
    pcg_it = int(os.environ.get("YASPS_REF_PCG_ITERS", "417"))
    for k in range(args.warmup + args.steps):
        cb = cpu_sample(args.config, bool(args.via_f), pcg_it)
        if k >= args.warmup:
            vals.append(cb["value"])
    v = float(statistics.median(vals))
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: one Newton iteration (bounded CPU sample, scaled)",
                       "scene": args.config},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
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
    sim = prepare(args.config, bool(args.via_f), "gpu", local)
    eng = sim.eng
    if world > 1:
        from paper_2605_23088_b200 import dist as ysdist
        ysdist.init_nccl(eng)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=torch.device("cuda", local))
    cfg = sim.config

    def step():
        eng.bump_dynamic_epoch()
        return eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)

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
    spmv_ms, spmv_bytes = eng.time_kernel(3, 50)  # the PCG's SpMV: sliced-ELL copy, 4 lanes per row
    asm_ms, asm_bytes = eng.time_kernel(1, 10)
    eval_ms, _ = eng.time_kernel(2, 5)
    spmv_gbs = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    asm_gbs = asm_bytes / (asm_ms * 1e-3) / 1e9
    # The dominant kernel is the PCG (one persistent cooperative launch per
    # solve for uniform 3x3 systems).  Algorithmic bytes per iteration
    # (SURVEY §8(d)): the SpMV's 8 r c + 8 per upper block + 16 s, the
    # block-Jacobi apply's 72 B per 3x3 inverse + 16 s, 6 vector passes 48 s.
    nb = eng.s // 3
    pcg_iter_bytes = spmv_bytes + 72.0 * nb + 16.0 * eng.s + 48.0 * eng.s
    pcg_ms = stages[4]
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
            cpu = cpu_sample(args.config, bool(args.via_f), int(np.median(iters)))
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
        "config": {"workload": f"{args.config}: one Newton iteration (dynamic rebuild + eval + assembly + "
                               f"block-Jacobi + PCG to pcg_tol) from a jittered rest state",
                   "scene": args.config, "tets": stats_tets, "dofs": int(eng.s),
                   "contact_pairs": int(sim.pair_count()), "pcg_iterations": int(np.median(iters)),
                   "nh_via_deformation_gradient": bool(args.via_f),
                   "l2": "inputs larger than L2 (device working set %.2f GB >> 126 MB)" % (eng.device_bytes() / 1e9),
                   "parallelism": f"pcg-rows{world} (eval/assembly replicated)" if world > 1 else "single"},
        "roofline": {"kernel": "k_pcg33_stream<SellPhaseA> (whole PCG solve over the sliced-ELL copy, one cooperative launch; the repack is included in avg_launch_ms)" if world == 1 else
                     "row-partitioned PCG (k_dspmv33 / k_dupdate per rank + NCCL allgather)",
                     "bound": "hbm", "achieved": pcg_gbs, "peak": peak, "unit": "GB/s", "frac": pcg_gbs / peak,
                     "traffic": traffic_from_profiles(args.config, "pcg_dram_bytes_per_iteration"),
                     "algorithmic_bytes": pcg_iter_bytes,
                     "algorithmic_bytes_unit": "per PCG iteration", "iterations": int(st.pcg_iterations),
                     "avg_launch_ms": pcg_ms, "peak_source": peak_src,
                     "spmv": {"kernel": "k_spmv_sell<4> (sliced-ELL full copy of static + dynamic H), timed alone",
                              "achieved": spmv_gbs, "frac": spmv_gbs / peak, "algorithmic_bytes": spmv_bytes,
                              "traffic": traffic_from_profiles(args.config, "spmv_dram_bytes"),
                              "avg_launch_ms": spmv_ms}},
        "assembly_roofline": {"bound": "hbm", "achieved": asm_gbs, "peak": peak, "unit": "GB/s",
                              "frac": asm_gbs / peak, "algorithmic_bytes": asm_bytes, "avg_ms": asm_ms},
        "eval_ms": eval_ms,
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
