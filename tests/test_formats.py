"""Wire / disk formats of SURVEY §8(f)4: MatrixMarket export
(assembly.cpp:106-134, sim.cpp:745-771) and trajectory.txt / stats.csv
(sim.cpp:583-629).  The writing rules are pinned by handwritten known answers;
the GPU leg checks that an exported GPU matrix is diffable against the oracle:
coordinate columns byte-identical, values within 1e-9."""
from __future__ import annotations

import io

import numpy as np
import pytest

from paper_2605_23088_b200.engine import HessianStructure, matrix_market_text, merged_coordinate_text
from paper_2605_23088_b200.scene import SimConfig, Simulation
from backends import simulation  # noqa: E402

from test_driver import BLOCK_ON_CLOTH, CONTACT_PAIR


def _structure(blocks, total):
    """A HessianStructure from [(rows, cols, row, col, values)], one group per shape."""
    shapes = sorted({(b[0], b[1]) for b in blocks})
    groups, row, col, vals = [], [], [], []
    for rows, cols in shapes:
        mine = [b for b in blocks if (b[0], b[1]) == (rows, cols)]
        groups.append([rows, cols, len(row), len(mine), len(vals)])
        for b in mine:
            row.append(b[2])
            col.append(b[3])
            vals.extend(np.asarray(b[4], dtype=float).ravel().tolist())
    return HessianStructure(np.asarray(groups, dtype=np.int64), np.asarray(row), np.asarray(col),
                            np.asarray(vals), 0, total)


def test_coordinate_text_kat():
    # a diagonal 2x2 block (lower entry skipped) and an off-diagonal 2x1 block
    h = _structure([(2, 2, 0, 0, [[4.0, 1.5], [1.5, 0.1]]), (2, 1, 0, 2, [[-0.0], [1e-5]])], 3)
    assert h.to_coordinate_text() == (
        "%%MatrixMarket matrix coordinate real general\n"
        "% upper triangle of a symmetric matrix\n"
        "3 3 5\n"
        "1 3 -0\n"
        "2 3 1.0000000000000001e-05\n"
        "1 1 4\n"
        "1 2 1.5\n"
        "2 2 0.10000000000000001\n")


def test_matrix_market_empty():
    assert matrix_market_text(4, np.zeros(0, int), np.zeros(0, int), np.zeros(0)) == (
        "%%MatrixMarket matrix coordinate real general\n% upper triangle of a symmetric matrix\n4 4 0\n")


class _FakeEngine:
    def __init__(self, s, d, total):
        self._h = [s, d]
        self._t = total

    def hessian(self, w):
        return self._h[w]

    def total_dofs(self):
        return self._t


def test_merged_text_sums_in_map_order():
    # static then dynamic per key; a lone -0.0 becomes +0 (std::map value starts at 0.0)
    s = _structure([(1, 1, 0, 0, [[0.1]]), (1, 1, 1, 1, [[-0.0]]), (1, 1, 0, 2, [[2.0]])], 3)
    d = _structure([(1, 1, 0, 0, [[0.2]]), (1, 1, 0, 1, [[-3.0]])], 3)
    txt = merged_coordinate_text(_FakeEngine(s, d, 3))
    assert txt.splitlines()[2:] == ["3 3 4", "1 1 %.17g" % (0.0 + 0.1 + 0.2), "1 2 -3", "1 3 2", "2 2 0"]


def test_run_writes_trajectory_and_stats(tmp_path):
    cfg = dict(CONTACT_PAIR, frames=3, output_dir=str(tmp_path / "out"))
    sim = simulation(SimConfig.from_dict(cfg), "oracle")
    log = io.StringIO()
    sim.run(log)
    traj = (tmp_path / "out" / "trajectory.txt").read_text().splitlines()
    stats = (tmp_path / "out" / "stats.csv").read_text().splitlines()
    assert stats[0] == "frame,newton,pcg,energy,max_step,pairs,nonincreasing" and len(stats) == 4
    for f, line in enumerate(stats[1:], 1):
        cols = line.split(",")
        assert int(cols[0]) == f and int(cols[1]) >= 1 and cols[6] in ("0", "1")
        assert float(cols[3]) == float("%.17g" % float(cols[3]))
    # frame headers, then per body "body <name> position <n> 3" and n rows of 3 values
    assert traj[0] == "frame 1"
    assert traj[1] == "body soft_cluster position 4 3"
    assert len(traj[2].split()) == 3
    assert traj.count("frame 3") == 1 and len(traj) == 3 * (1 + 2 * (1 + 4))
    last = np.array([[float(x) for x in ln.split()] for ln in traj[-4:]])
    assert np.array_equal(last, sim.body_positions(sim.bodies[1]))
    out = log.getvalue().splitlines()
    assert out[0] == "frames 3" and out[-1].startswith("cg iterations ")


@pytest.mark.gpu
def test_export_matrix_gpu_matches_oracle():
    texts = []
    for backend in ("oracle", "gpu"):
        sim = simulation(SimConfig.from_dict(BLOCK_ON_CLOTH), backend)
        texts.append(sim.export_matrix(frame=5).splitlines())
    a, b = texts
    assert a[:3] == b[:3]
    ca = [ln.rsplit(" ", 1) for ln in a[3:]]
    cb = [ln.rsplit(" ", 1) for ln in b[3:]]
    assert [x[0] for x in ca] == [x[0] for x in cb]  # coordinates: byte-identical
    va = np.array([float(x[1]) for x in ca])
    vb = np.array([float(x[1]) for x in cb])
    assert np.max(np.abs(va - vb)) <= 1e-9 * np.max(np.abs(va))
