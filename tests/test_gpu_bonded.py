"""FENE bonds on the device (the Kremer-Grest path).

compute_bonded_forces (bonded.hpp:167-199) is fused into the force kernel:
each particle adds the FENE force of its own bonds (the bond vector always
taken from the anchor a, so both ends see exactly opposite forces), both ends
book the energy, halved with the pair sums. Parity against the reference's golden runs of a KG melt
(WCA + FENE 30/1.5, skin 0.4) and of FENE chains in the LJ fluid: pair sets
bit-exact, forces 1e-10, PE/virial 1e-12 (fsum of the reference's terms),
200-step trajectories."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import E_RTOL, assert_forces_close, assert_rel, load

pytestmark = pytest.mark.gpu

SYSTEMS = ["kg_lattice10", "fene_lj8"]


def inter_of(g):
    lj = E.LjParams()
    if "lj" in g:
        eps, sig, rc, sh = g["lj"]
        lj = E.LjParams(float(eps), float(sig), float(rc), bool(sh))
    k, rmax = g["fene"]
    return E.Interactions(lj=lj, fene=E.FeneParams(float(k), float(rmax)))


def flat_of(g):
    return E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"], bonds=g["bonds"])


def engine(g, **cfg):
    return E.Engine(flat_of(g), inter_of(g), float(g["r_skin"]),
                    E.EngineConfig(dt=float(g["dt"]), **cfg))


@pytest.mark.parametrize("name", SYSTEMS)
@pytest.mark.parametrize("variant", [0, 1])
def test_initial_state_vs_golden(name, variant):
    g = load(name)
    eng = engine(g, variant=variant)
    np.testing.assert_array_equal(eng.pairs(), g["pairs"])
    ids, f = eng.forces()
    assert_forces_close(f, g["forces"])
    o = eng.observe()
    assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE (LJ + FENE)")
    assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial (LJ + FENE)")
    assert_rel(o.kinetic, float(g["ke_ref"]), 1e-13, "KE")


@pytest.mark.parametrize("name", SYSTEMS)
@pytest.mark.parametrize("graphs,build", [(True, 0), (False, 0), (True, 3), (True, 5)])
def test_trajectory_vs_golden(name, graphs, build):
    g = load(name)
    eng = engine(g, graphs=graphs, build=build)
    steps = int(g["steps"])
    every = max(1, steps // len(g["trace"]))
    for row in g["trace"]:
        eng.run(every)
        o = eng.observe()
        assert o.step == int(row[0])
        assert_rel(o.kinetic + o.potential, row[1] + row[2], 1e-10, f"E at step {o.step}")
    flat = eng.flatten()
    assert np.abs(flat.pos - g["final_pos"]).max() < 1e-9
    assert np.abs(flat.vel - g["final_vel"]).max() < 1e-9
    assert eng.rebuild_count() == int(g["rebuilds"])


@pytest.mark.parametrize("R", [2, 3])
def test_decomposed_trajectory_vs_golden(R):
    g = load("kg_lattice10")
    eng = DecomposedEngine(flat_of(g), inter_of(g), float(g["r_skin"]),
                           E.EngineConfig(dt=float(g["dt"])), comm=InProcessComm(R))
    try:
        np.testing.assert_array_equal(eng.local_pairs(), g["pairs"])
        o = eng.observe()
        assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
        eng.run(int(g["steps"]))
        ids, pos, vel, _ = eng.local_state()
        assert np.abs(pos - g["final_pos"]).max() < 1e-9
        assert np.abs(vel - g["final_vel"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])
    finally:
        eng.close()


def _dimer(r0, dr):
    f = E.FlatConfig(np.full(3, 10.0), np.array([0, 1]),
                     np.array([[5.0 - 0.5 * (r0 + dr), 5.0, 5.0],
                               [5.0 + 0.5 * (r0 + dr), 5.0, 5.0]]), None,
                     bonds=np.array([[0, 1]]))
    return f


def test_bond_overstretch_is_a_physics_error():
    """bonded.hpp:184-191: r >= r_max raises with both ids."""
    f = _dimer(1.55, 0.0)
    with pytest.raises(E.PhysicsError, match="fene bond overstretched between ids 0 and 1"):
        E.Engine(f, E.Interactions(fene=E.FeneParams(30.0, 1.5)), 0.4)


def test_dimer_oscillates_at_the_curvature_frequency():
    """test_engine.cpp:100-163: a bonded LJ dimer (LJ rc 2.5 + FENE 30/1.5)
    oscillates with period 2 pi / sqrt(U''(r0) / mu) within 1 %."""
    eps4, eps24 = 4.0, 24.0
    s6c = (1.0 / 6.25) ** 3
    shift = eps4 * (s6c * s6c - s6c)

    def u(r):
        i6 = (1.0 / (r * r)) ** 3
        lj = eps4 * (i6 * i6 - i6) - shift
        return lj - 0.5 * 30.0 * 2.25 * math.log(1.0 - r * r / 2.25)

    lo, hi = 0.9, 1.1
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        h = 1e-6
        slope = (u(mid + h) - u(mid - h)) / (2 * h)
        lo, hi = (mid, hi) if slope < 0.0 else (lo, mid)
    r0 = 0.5 * (lo + hi)
    h = 1e-4
    curv = (u(r0 + h) - 2.0 * u(r0) + u(r0 - h)) / (h * h)
    period = 2.0 * math.pi / math.sqrt(curv / 0.5)
    dt = 0.0005
    eng = E.Engine(_dimer(r0, 0.01), E.Interactions(fene=E.FeneParams(30.0, 1.5)), 0.4,
                   E.EngineConfig(dt=dt))
    crossings, prev = [], 0.01
    for s in range(1, 6001):
        eng.step()
        p = eng.flatten().pos
        d = p[0] - p[1]
        d -= 10.0 * np.round(d / 10.0)
        x = float(np.sqrt((d * d).sum())) - r0
        if prev < 0.0 <= x:
            crossings.append((s - 1 + prev / (prev - x)) * dt)
            if len(crossings) >= 5:
                break
        prev = x
    assert len(crossings) >= 3
    measured = (crossings[-1] - crossings[0]) / (len(crossings) - 1)
    assert measured == pytest.approx(period, rel=0.01)


def test_partner_out_of_reach_in_a_slab_decomposition():
    """test_domain.cpp:246-266 analog: a bond spanning two slabs that are not
    neighbours cannot be resolved: PhysicsError "out of reach"."""
    f = E.FlatConfig(np.full(3, 15.0), np.array([0, 1]),
                     np.array([[7.5, 7.5, 1.5], [7.5, 7.5, 7.5]]), None,
                     bonds=np.array([[0, 1]]))
    with pytest.raises(E.PhysicsError, match="out of reach"):
        DecomposedEngine(f, E.Interactions(fene=E.FeneParams(30.0, 1.5)), 0.5,
                         comm=InProcessComm(5))


def test_kg_melt_warmup_then_nve():
    """BASELINE configs[2] shape at small N: generated random-walk melt,
    force-capped Langevin warm-up, then KG NVE at dt 0.01 stays bounded."""
    f = E.gen_chains(40, 50, 0.85, 0.97, seed=3)
    warm = E.kg_warmup(f, steps_per_cap=100, equilibrate_steps=1500)
    eng = E.Engine(warm, E.kg_interactions(), 0.4, E.EngineConfig(dt=0.01))
    o0 = eng.observe()
    e0 = o0.kinetic + o0.potential
    eng.run(500)
    o = eng.observe()
    assert abs(o.kinetic + o.potential - e0) / abs(e0) < 5e-3
    assert 0.3 < o.temperature < 3.0


def test_bond_table_degree_limit_and_order():
    """The device-built bond table: a particle with more than kMaxBonds (8)
    bonds is a ConfigError naming the smallest such id; duplicate bonds keep
    both entries (forces and energies count the bond twice, as the reference's
    bond list does)."""
    box = np.full(3, 12.0)
    rng = np.random.default_rng(5)
    pos = rng.random((40, 3)) * 12.0
    ids = np.arange(100, 140, dtype=np.int64)
    star = np.array([[105, 110 + k] for k in range(9)], dtype=np.int64)
    flat = E.FlatConfig(box, ids, pos, None, bonds=star)
    inter = E.Interactions(fene=E.FeneParams(30.0, 1.5))
    with pytest.raises(E.ConfigError, match="particle id 105 has 9 bonds"):
        E.Engine(flat, inter, 0.4, E.EngineConfig(dt=0.001))
