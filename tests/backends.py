"""Test-side backend selection: the product's Engine / Simulation drive the
B200 library; the parity tests inject the oracle (or the reference build) as
another implementation of the same C-ABI (oracle/__init__.py)."""
from __future__ import annotations

import oracle
from paper_2605_23088_b200.engine import Engine
from paper_2605_23088_b200.scene import Simulation


def engine(backend: str = "gpu", device: int = 0) -> Engine:
    eng = Engine(device, oracle.for_backend(backend))
    eng.backend = backend
    return eng


def simulation(cfg, backend: str = "gpu", **kw) -> Simulation:
    sim = Simulation(cfg, library=oracle.for_backend(backend), **kw)
    sim.eng.backend = backend
    return sim
