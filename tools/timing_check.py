import subprocess, time, sys
import torch
from bench import prepare, ClockSampler
sim = prepare("c5", True, "gpu")
eng = sim.eng
stream = torch.cuda.ExternalStream(eng.stream_handle())
def step():
    eng.bump_dynamic_epoch()
    return eng.minimize_step(1e-4, -1, want_dx=False)
for _ in range(3): step()
def timed(k, sampler):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    if sampler:
        cs = ClockSampler(0); cs.__enter__()
    t0 = time.perf_counter(); e0.record(stream)
    for _ in range(k): st = step()
    e1.record(stream); torch.cuda.synchronize(); t1 = time.perf_counter()
    if sampler: cs.__exit__(); print("clocks", cs.summary())
    return e0.elapsed_time(e1)/k, (t1-t0)*1e3/k, st.pcg_iterations
for rep in range(2):
    print("no sampler", timed(5, False), flush=True)
    print("sampler   ", timed(5, True), flush=True)
