"""Checks the sliced-ELL SpMV variants (YS_APPLY_VARIANT routes
ys_apply_hessian through one) against the production row gather on the same
random x, in subprocesses (development aid)."""
import os
import subprocess
import sys

if len(sys.argv) > 2:  # child
    import numpy as np

    from paper_2605_23088_b200 import configs
    from paper_2605_23088_b200.scene import SimConfig, Simulation

    name, out = sys.argv[1], sys.argv[2]
    cfg = SimConfig.from_dict(configs.CONFIGS[name]())
    sim = Simulation(cfg, backend="gpu")
    configs.jitter_targets(sim, 0.1 * (0.025 if name == "c1" else 0.01))
    sim.begin_frame()
    sim.refresh_dynamic_pairs()
    eng = sim.eng
    eng.bump_dynamic_epoch()
    eng.minimize_step(cfg.pcg_tol, -1, want_dx=False)
    x = np.random.default_rng(1).standard_normal(eng.s)
    np.save(out, eng.apply_hessian(x))
    sys.exit(0)

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
import numpy as np  # noqa: E402

ys = {}
for v in [0, 40, 41, 42, 43]:
    env = dict(os.environ, YS_APPLY_VARIANT=str(v))
    f = f"/tmp/sellchk_{v}.npy"
    subprocess.run([sys.executable, __file__, name, f], env=env, check=True)
    ys[v] = np.load(f)
for v, y in ys.items():
    err = float(np.max(np.abs(y - ys[0])) / np.max(np.abs(ys[0])))
    print(f"{name} variant {v}: max rel diff vs row gather {err:.3e}", flush=True)
