"""The `md`-style CLI on the GPU engine: the reference's
run configs drive the B200 path with the reference's output formats; the
observables it prints match the reference engine (oracle/_ref) run on the
same generated system."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

BULK = """seed = 42
system.generator = lattice
system.n = 4000
system.rho = 0.8442
system.temperature = 0.6
interaction.epsilon = 1.0
interaction.sigma = 1.0
interaction.r_cut = 2.5
interaction.energy_shifted = true
interaction.r_skin = 0.3
engine.dt = 0.005
engine.steps = 100
engine.n_sub = auto
engine.worker_threads = 4
engine.thermostat.gamma = 1.0
engine.thermostat.temperature = 0.6
output.timing_path = bulk_timings.csv
output.timing_mode = per_step
output.trajectory_path = traj.xyz
output.trajectory_stride = 50
output.observable_stride = 20
"""

VERIFY = """seed = 1
system.generator = random
system.n = 500
system.rho = 0.8442
system.temperature = 0.72
system.min_distance = 0.8
interaction.r_cut = 2.5
interaction.r_skin = 0.3
engine.dt = 0.005
engine.steps = 0
engine.n_sub = 8
"""


def md(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2109_10876_b200.cli", *args],
                          cwd=cwd or ROOT, capture_output=True, text=True, timeout=600)


def test_run_matches_the_reference_engine(tmp_path, ref):
    cfg = tmp_path / "bulk.cfg"
    cfg.write_text(BULK)
    r = md("run", "--config", str(cfg), "--out", str(tmp_path / "out"))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "step,kinetic,potential,temperature"
    rows = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])
    assert rows[:, 0].tolist() == [0, 20, 40, 60, 80, 100]
    # the same system through the reference engine
    b, i, p, v = ref.gen_lattice(4000, 0.8442, 0.6, 42)
    e = ref.RefEngine(b, i, p, v, r_skin=0.3, dt=0.005, thermostat=(1.0, 0.6, 42))
    want = [e.observe()]
    for _ in range(5):
        e.run(20)
        want.append(e.observe())
    for row, w in zip(rows, want):
        assert row[1] == pytest.approx(w["kinetic"], rel=1e-9)
        assert row[2] == pytest.approx(w["potential"], rel=1e-9)
        assert row[3] == pytest.approx(w["temperature"], rel=1e-9)
    # completion line, timing file, trajectory
    assert "completed 100 steps in" in r.stderr and "list rebuilds, 0 steals" in r.stderr
    timing = (tmp_path / "out" / "bulk_timings.csv").read_text().splitlines()
    assert timing[0] == "step_range,section,seconds"
    assert len(timing) == 1 + 100 * 5 + 5 + 1 and timing[-1].startswith("0-100,Elapsed,")
    xyz = (tmp_path / "out" / "traj.xyz").read_text().splitlines()
    assert len(xyz) == 3 * (4000 + 2) and xyz[0] == "4000"
    assert xyz[1].startswith("step=0 box=") and xyz[4002 + 1].startswith("step=50 box=")


def test_verify_against_the_all_pairs_evaluation(tmp_path):
    cfg = tmp_path / "verify.cfg"
    cfg.write_text(VERIFY)
    r = md("verify", "--config", str(cfg))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "pair sets equal" in r.stdout and "N = 500, n_sub = 8" in r.stdout
    assert "max |dF| =" in r.stdout


def test_brute_force_matches_the_reference_oracle(ref):
    """The GPU all-pairs evaluation behind verify against oracle.hpp's."""
    f = E.gen_random(400, 0.8442, 0.8, 0.72, 3)
    forces, pe, pairs = E.brute_force(f, E.Interactions(), 2.8)
    want_f, want_pe = ref.oracle_forces(f.box, f.id, f.pos)
    assert np.abs(forces - want_f).max() <= 1e-10
    assert pe == pytest.approx(want_pe, rel=1e-12)
    np.testing.assert_array_equal(pairs, ref.oracle_pairs(f.box, f.id, f.pos, 2.8))


def test_physics_errors_exit_2(tmp_path):
    cfg = tmp_path / "hot.cfg"
    cfg.write_text(BULK.replace("engine.thermostat.temperature = 0.6",
                                "engine.thermostat.temperature = 1e308")
                   .replace("engine.steps = 100", "engine.steps = 5"))
    r = md("run", "--config", str(cfg), "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "physics error" in r.stderr and "non-finite" in r.stderr


def test_kg_melt_and_fcc_configs_run(tmp_path):
    kg = tmp_path / "kg.cfg"
    kg.write_text("seed = 3\nsystem.generator = kg_melt\nsystem.chains = 20\n"
                  "system.chain_length = 50\nsystem.rho = 0.85\n"
                  f"interaction.r_cut = {2 ** (1 / 6)!r}\ninteraction.r_skin = 0.4\n"
                  "engine.dt = 0.01\nengine.steps = 100\noutput.observable_stride = 50\n")
    r = md("run", "--config", str(kg), "--out", str(tmp_path / "o1"))
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.strip().splitlines()) == 1 + 3
    fcc = tmp_path / "fcc.cfg"
    fcc.write_text("seed = 12345\nsystem.generator = fcc\nsystem.cells = 8\nsystem.rho = 0.8442\n"
                   "system.temperature = 1.0\nengine.steps = 50\noutput.observable_stride = 25\n")
    r = md("autotune", "--config", str(fcc), "--out", str(tmp_path / "o2"))
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "o2" / "autotune.csv").read_text().startswith("n_sub,seconds,selected\n1,")
