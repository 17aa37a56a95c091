"""Parity at BASELINE.json's full sizes through size-independent properties.

* 1,048,576 jittered FCC (SURVEY §8c known answer, computed in long double
  from the reference's terms): PE and virial to 1e-12; cells, forces and
  the pair-set checksum against the reference engine itself (oracle/_ref).
* 16,384,000 perfect FCC (configs[4]): every particle sees exactly the five
  FCC shells inside r_v = 2.8 (78 full-list entries, 54 within r_cut) and the
  lattice energy per particle is the 32K known answer, -6.3328119926;
  100 NVE steps conserve energy like the reference at 32K.
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
