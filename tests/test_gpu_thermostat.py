"""Langevin thermostat on the device.

thermostat_and_half_kick (engine.hpp:209-239) adds
-gamma m v + sqrt(2 m gamma T / dt) n, n = counter_normal3(seed, kThermostat,
step, id) (random.hpp:69-81, potentials.hpp:192-197), before the closing
half-kick; the initial evaluation uses step-0 noise (engine.hpp:244-278).
The GPU restates the counter hash exactly; log/cos/sin are CUDA's (<= 2 ulp
vs glibc), so trajectories are compared against the reference's golden runs
to 1e-9 rather than bitwise."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import assert_forces_close, assert_rel, load

pytestmark = pytest.mark.gpu

SYSTEMS = ["langevin_jit6", "langevin_fcc8"]


def bath(g):
    gamma, temp, seed = g["thermostat"]
    return E.LangevinParams(gamma=float(gamma), temperature=float(temp), seed=int(seed))


def engine(g, **cfg):
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    return E.Engine(flat, E.Interactions(), float(g["r_skin"]),
                    E.EngineConfig(dt=float(g["dt"]), thermostat=bath(g), **cfg))


@pytest.mark.parametrize("name", SYSTEMS)
def test_initial_forces_include_step0_noise(name):
    g = load(name)
    eng = engine(g)
    np.testing.assert_array_equal(eng.pairs(), g["pairs"])
    _, f = eng.forces()
    assert_forces_close(f, g["forces"])


@pytest.mark.parametrize("name", SYSTEMS)
@pytest.mark.parametrize("graphs", [True, False])
def test_trajectory_vs_golden(name, graphs):
    g = load(name)
    eng = engine(g, graphs=graphs)
    steps = int(g["steps"])
    every = max(1, steps // len(g["trace"]))
    for row in g["trace"]:
        eng.run(every)
        o = eng.observe()
        assert o.step == int(row[0])
        assert_rel(o.kinetic, row[1], 1e-9, f"KE at step {o.step}")
        assert_rel(o.potential, row[2], 1e-9, f"PE at step {o.step}")
    flat = eng.flatten()
    assert np.abs(flat.pos - g["final_pos"]).max() < 1e-9
    assert np.abs(flat.vel - g["final_vel"]).max() < 1e-9
    assert eng.rebuild_count() == int(g["rebuilds"])


def test_graph_and_eager_are_bitwise_identical():
    g = load("langevin_fcc8")
    outs = []
    for timers in (True, False):
        eng = engine(g, graphs=not timers)
        eng.run(37)
        outs.append(eng.flatten())
    np.testing.assert_array_equal(outs[0].pos, outs[1].pos)
    np.testing.assert_array_equal(outs[0].vel, outs[1].vel)


def test_decomposed_run_vs_golden():
    g = load("langevin_fcc8")
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    for R in (2, 4):
        eng = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                               E.EngineConfig(dt=float(g["dt"]), thermostat=bath(g)),
                               comm=InProcessComm(R))
        eng.run(int(g["steps"]))
        ids, pos, vel, _ = eng.local_state()
        assert np.abs(pos - g["final_pos"]).max() < 1e-9
        assert np.abs(vel - g["final_vel"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])
        eng.close()


def test_thermostat_pulls_a_cold_system_to_its_set_point():
    """test_engine.cpp:262-281: cold jittered lattice, bath T = 0.8, 400 steps,
    then the mean temperature over 100 steps is 0.8 +- 0.16."""
    g = load("langevin_jit6")
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], np.zeros_like(g["pos"]))
    eng = E.Engine(flat, E.Interactions(), 0.3,
                   E.EngineConfig(dt=0.005, thermostat=E.LangevinParams(1.0, 0.8, 7)))
    eng.run(400)
    temps = []
    for _ in range(100):
        eng.step()
        temps.append(eng.observe().temperature)
    assert abs(np.mean(temps) - 0.8) <= 0.16


def test_non_finite_noise_is_caught_with_the_step():
    """test_engine.cpp:369-382: T = 1e308 overflows the noise amplitude."""
    g = load("langevin_jit6")
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    with pytest.raises(E.PhysicsError, match=r"non-finite.*\(at step"):
        eng = E.Engine(flat, E.Interactions(), 0.3,
                       E.EngineConfig(dt=0.005, thermostat=E.LangevinParams(1.0, 1e308, 1)))
        eng.run(3)


def test_rollback_keeps_the_langevin_force():
    """A list overflow mid-run rolls back to the chunk checkpoint; with a bath
    the stored force (which carries the last Langevin kick) is restored, so the
    result matches the run that never overflowed."""
    g = load("langevin_fcc8")
    a = engine(g)
    a.run(80)
    b = engine(g, nbr_capacity=8)
    b.run(80)
    fa, fb = a.flatten(), b.flatten()
    assert np.abs(fa.pos - fb.pos).max() < 1e-9
    assert np.abs(fa.vel - fb.vel).max() < 1e-9
