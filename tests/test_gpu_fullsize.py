"""Parity at BASELINE.json's full sizes through size-independent properties.

* 1,048,576 jittered FCC (SURVEY §8c known answer, computed in long double
  from the reference's terms): PE and virial to 1e-12; cells, forces and
  the pair-set checksum against the reference engine itself (oracle/_ref).
* 16,384,000 perfect FCC (configs[4]): every particle sees exactly the five
  FCC shells inside r_v = 2.8 (78 full-list entries, 54 within r_cut) and the
  lattice energy per particle is the 32K known answer, -6.3328119926;
  100 NVE steps conserve energy like the reference at 32K.
* 4,000,000-bead Kremer-Grest melt (configs[2]) and the 2,097,152-particle
  liquid-vapour slab (configs[3]): the reference's decomposition invariance
  (the system as 4 native slabs against the single context: forces 1e-10,
  PE / virial 1e-12, equal rebuild steps), Newton's third law as a checksum
  (sum of forces = 0 to 1e-12 of the sum of |F|), bonds inside the FENE well.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from tests._util import assert_forces_close, assert_rel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

K_PLACEMENT = 3


def jittered_fcc64():
    f = E.gen_fcc(64, 0.8442, 1.0, 12345)
    u = np.array([E.counter_uniform3(777, K_PLACEMENT, 0, int(i)) for i in f.id])
    f.pos = f.pos + 0.15 * (2.0 * u - 1.0)
    return f


def test_1m_jittered_fcc_against_known_answers_and_the_reference(ref):
    f = jittered_fcc64()
    eng = E.Engine(f, E.Interactions(), 0.3)
    o = eng.observe()
    assert_rel(o.potential, -4654949.83609085, 1e-12, "PE (SURVEY §8c, long double)")
    assert_rel(o.virial, 11116436.7829377, 1e-12, "virial (SURVEY §8c, long double)")
    r = ref.RefEngine(f.box, f.id, f.pos, f.vel, r_skin=0.3, n_sub=8, workers=8)
    _, rc = r.cell_of()
    _, gc = eng.cell_of()
    np.testing.assert_array_equal(gc, rc)
    _, rf = r.forces()
    _, gf = eng.forces()
    assert_forces_close(gf, rf)
    rp = r.pairs()
    gp = eng.pairs()
    assert len(gp) == len(rp)
    # checksum of checksums instead of a 650 MB comparison in one go
    for a, b in zip(np.array_split(gp, 16), np.array_split(rp, 16)):
        np.testing.assert_array_equal(a, b)


def test_16m_perfect_fcc_shells_energy_and_drift():
    f = E.gen_fcc(160, 0.8442, 1.0, 12345)
    n = f.size()
    assert n == 16_384_000
    eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(section_timers=False))
    st = eng.list_stats()
    assert st["entries"] == 78 * n and st["in_cut"] == 54 * n and st["max_count"] == 78
    assert tuple(st["dims"]) == (95, 95, 95)
    o0 = eng.observe()
    assert o0.potential / n == pytest.approx(-6.3328119926, abs=5e-10)
    e0 = o0.kinetic + o0.potential
    rows = eng.run_observed(100, stride=10)
    worst = max(abs(r[1] + r[2] - e0) / abs(e0) for r in rows)
    assert worst < 2e-4  # the reference's 32K run: 1.154e-4 over 1000 steps


def _newton3_residual(f: np.ndarray) -> float:
    return float(np.abs(f.sum(axis=0)).max() / np.abs(f).sum())


def _slabs_match_single_context(flat, inter, r_skin, cfg, R, balance, steps):
    """The reference's decomposition invariance (test_engine.cpp:242-260,
    acceptance.cpp:121-150) at a BASELINE size: the system as R native slabs
    against the single context — pair count, forces 1e-10, PE / virial 1e-12,
    and the same rebuild steps and energies after `steps` steps."""
    from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
    one = E.Engine(flat, inter, r_skin, cfg)
    dec = DecomposedEngine(flat, inter, r_skin, cfg, comm=InProcessComm(R), native=True,
                           balance=balance)
    try:
        ids1, f1 = one.forces()
        ids2, _, _, f2 = dec.local_state()
        np.testing.assert_array_equal(ids2, ids1)
        assert_forces_close(f2, f1)
        assert _newton3_residual(f1) < 1e-12 and _newton3_residual(f2) < 1e-12
        o1, o2 = one.observe(), dec.observe()
        assert_rel(o2.potential, o1.potential, 1e-12, "PE")
        assert_rel(o2.virial, o1.virial, 1e-12, "virial")
        st = one.list_stats()
        assert sum(s["n_own"] for s in dec.slab_sizes().values()) == st["n"]
        one.run(steps)
        dec.run(steps)
        assert dec.rebuild_count() == one.rebuild_count() > 0
        o1, o2 = one.observe(), dec.observe()
        assert_rel(o2.potential, o1.potential, 1e-10, "PE after the run")
        assert_rel(o2.kinetic, o1.kinetic, 1e-10, "KE after the run")
        return one.flatten()
    finally:
        one.close()
        dec.close()


def test_4m_kremer_grest_melt_decomposition_invariance_and_bonds():
    """configs[2]: 20,000 chains of 200 beads after the force-capped warm-up."""
    flat = E.kg_warmup(E.gen_chains(20000, 200, 0.85, 0.97, seed=12345))
    assert flat.size() == 4_000_000 and flat.bonds.shape == (20000 * 199, 2)
    cfg = E.EngineConfig(dt=0.01, section_timers=False)
    end = _slabs_match_single_context(flat, E.kg_interactions(), 0.4, cfg, 4, "static", 20)
    # every bond still inside the FENE well (ids are dense: row = id)
    order = np.argsort(end.id)
    pos = end.pos[order]
    d = pos[end.bonds[:, 0]] - pos[end.bonds[:, 1]]
    d -= end.box * np.round(d / end.box)
    r = np.sqrt((d * d).sum(axis=1))
    assert 0.7 < r.min() and r.max() < 1.5


def test_2m_liquid_vapour_slab_decomposition_invariance_with_count_cuts():
    """configs[3]: 2,097,152 particles, a liquid slab in a 3x elongated box."""
    flat = E.gen_fcc_slab(81, 0.8442, 0.7, 12345, n=2097152)
    assert flat.size() == 2_097_152
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    _slabs_match_single_context(flat, E.Interactions(), 0.3, cfg, 4, "count", 30)
