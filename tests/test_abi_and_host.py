"""CPU tests of the boundary and the host logic: the C-ABI libraries load and
export every function include/yasps_b200.h declares; scene generators match
the reference's sizes; config errors use the reference's wording."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_23088_b200 import ValidationError, configs
import oracle
from backends import engine
from paper_2605_23088_b200._lib import LIB_PATH, ROOT, gpu_library
from paper_2605_23088_b200.scene import SimConfig, hinges, make_grid_cloth, make_tet_block

HEADER = ROOT / "include" / "yasps_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(?:int|void|const char\*)\s+(ys_\w+)\s*\(", text)))


def test_header_declares_the_engine_surface():
    names = declared()
    for n in ("ys_create", "ys_finalize", "ys_assemble", "ys_minimize_step", "ys_apply_hessian",
              "ys_total_energy", "ys_refresh_dynamic", "ys_hessian_values", "ys_bsr_pcg"):
        assert n in names
    assert len(names) >= 55


def test_b200_library_exports_every_declared_symbol():
    assert LIB_PATH.exists(), "libyasps_b200.so not built"
    dll = ctypes.CDLL(str(LIB_PATH))  # loads without a GPU (static cudart)
    missing = [n for n in declared() if not hasattr(dll, n)]
    assert not missing, missing
    assert b"sm_100a" in gpu_library().fns["version"]()


def test_oracle_exports_the_same_abi():
    lib = oracle.library()
    dll = lib.dll
    # device instrumentation and the NCCL / peer-memory transports have no CPU counterpart
    optional = {"ys_set_profiling", "ys_stage_times", "ys_device_bytes", "ys_time_kernel", "ys_dist_unique_id",
                "ys_dist_init_nccl", "ys_dist_p2p_open", "ys_dist_p2p_connect", "ys_dist_p2p_probe",
                "ys_dist_p2p_group", "ys_dist_p2p_group_step"}
    missing = [n for n in declared() if n not in optional and not hasattr(dll, "yo_" + n[3:])]
    assert not missing, missing


def test_no_device_means_loud_failure():
    import ctypes as C
    cu = None
    try:
        cu = C.CDLL("libcuda.so.1")
    except OSError:
        pass
    if cu is not None and cu.cuInit(0) == 0:
        n = C.c_int(0)
        if cu.cuDeviceGetCount(C.byref(n)) == 0 and n.value > 0:
            pytest.skip("a device is present")
    from paper_2605_23088_b200 import CudaError, Engine
    with pytest.raises(CudaError):
        engine("gpu")


def test_tet_block_sizes_match_survey():
    v, t = make_tet_block(6, 5, 6, 0.025)
    assert len(v) == 294 and len(t) // 4 == 1080
    v, t = make_tet_block(28, 28, 27, 0.01)
    assert len(v) == 23548 and len(t) // 4 == 127008  # x 8 blocks = 188,384 / 1,016,064
    # Kuhn tets all have positive volume
    tt = t.reshape(-1, 4)[:500]
    d = v[tt[:, 1:]] - v[tt[:, :1]]
    assert np.all(np.abs(np.linalg.det(d)) > 0)


def test_cloth_and_hinges_match_survey():
    v, tris = make_grid_cloth(317, 317, 1.0 / 316)
    assert len(v) == 100489 and len(tris) // 3 == 199712
    assert len(hinges(tris)) == 298936


def test_hinges_kat_small():
    v, tris = make_grid_cloth(2, 2, 1.0)
    h = hinges(tris)
    # one interior edge (1, 2) shared by faces (0, 1, 2) and (1, 3, 2)
    assert h.tolist() == [[1, 2, 0, 3]]


def test_config_errors():
    with pytest.raises(ValidationError, match="non-empty 'bodies'"):
        SimConfig.from_dict({"dt": 0.01})
    with pytest.raises(ValidationError, match="dt must be positive"):
        SimConfig.from_dict({"dt": -1, "bodies": [{}]})
    with pytest.raises(ValidationError, match="cannot open config file"):
        SimConfig.load("/nonexistent.json")


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_scene_configs_parse(name):
    cfg = SimConfig.from_dict(configs.CONFIGS[name]())
    assert cfg.contact_enabled and len(cfg.bodies) >= 2


@pytest.mark.gpu
def test_cpp_facade_on_device():
    """C++ host through include/yasps_b200.hpp (tools/cpp_smoke.cpp)."""
    import subprocess
    exe = ROOT / "tools" / "cpp_smoke"
    assert exe.exists(), "built by paper_2605_23088_b200/build.py"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp facade ok" in r.stdout
