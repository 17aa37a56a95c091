"""The reference's acceptance criteria that the other GPU files do not already
restate, run on the CUDA path (acceptance.cpp; criterion 1, 2, 3 and 9 live
in test_gpu_parity.py, 6 in test_oracle_golden.py):

  4   Langevin thermostat holds the benchmark temperature (acceptance.cpp:186-211)
  5   mean half-list neighbour counts, equilibrated and random (213-230)
  10  finite-difference gradients of the pair and bond terms (350-381), here
      through the device's energies and forces, plus the dimer virial r.F
      (the reference has no virial: pinned to the force it must equal)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E

pytestmark = pytest.mark.gpu


def _half_neighbours(flat: E.FlatConfig) -> float:
    """mean_half_neighbors(oracle_pair_set(flat, 2.8)) from the device list."""
    eng = E.Engine(E.FlatConfig(flat.box, flat.id, flat.pos, None), E.Interactions(), 0.3,
                   E.EngineConfig(section_timers=False))
    try:
        return eng.pairs().shape[0] / flat.size()
    finally:
        eng.close()


def test_criteria_4_and_5_langevin_temperature_and_neighbour_statistics(ref):
    n = 4000
    flat = E.gen_lattice(n, 0.8442, 0.6, 17)
    cfg = E.EngineConfig(dt=0.005, section_timers=False,
                         thermostat=E.LangevinParams(1.0, 0.6, 17))
    eng = E.Engine(flat, E.Interactions(), 0.3, cfg)
    try:
        rows = eng.run_observed(5000, stride=1)
        assert rows.shape[0] == 5000 and rows[-1, 0] == 5000
        temps = 2.0 * rows[2500:, 1] / (3.0 * n)   # domain_kinetic(...).temperature()
        np.testing.assert_allclose(temps, rows[2500:, 3], rtol=1e-14)
        mean = float(temps.mean())
        assert abs(mean - 0.6) / 0.6 <= 0.05, f"<T> over the last half = {mean:.4f} vs 0.6"
        eq = eng.flatten()
    finally:
        eng.close()
    eq_mean = _half_neighbours(eq)
    assert abs(eq_mean - 41.2) / 41.2 <= 0.15, f"equilibrated half-list neighbours {eq_mean:.3f}"
    rnd = []
    for seed in range(1, 11):
        box, ids, pos, vel = ref.gen_random(500, 0.8442, 0.8, 0.72, seed)
        rnd.append(_half_neighbours(E.FlatConfig(box, ids, pos, vel)))
    rnd_mean = float(np.mean(rnd))
    assert abs(rnd_mean - 38.8) / 38.8 <= 0.05, f"random half-list neighbours {rnd_mean:.3f}"


def _dimer(r: float, axis: np.ndarray, inter: E.Interactions, bonded: bool,
           r_skin: float = 0.3):
    """(PE, W, force on particle 1 along the axis) of a dimer at separation r,
    placed across the periodic boundary of a 9.0 box."""
    box = np.full(3, 9.0)
    p0 = np.array([8.7, 0.2, 4.5])
    pos = np.stack([p0, p0 + r * axis])   # unwrapped input: wrapped at create
    bonds = np.array([[0, 1]]) if bonded else None
    eng = E.Engine(E.FlatConfig(box, np.array([0, 1]), pos, None, bonds=bonds), inter, r_skin,
                   E.EngineConfig(section_timers=False))
    try:
        pe, w = eng.compute_forces()
        _, f = eng.forces()
        np.testing.assert_allclose(f[0], -f[1], rtol=0, atol=0)   # Newton 3, bitwise
        return pe, w, float(f[1] @ axis)
    finally:
        eng.close()


def _unit(rng) -> np.ndarray:
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


def test_criterion_10_lj_gradient_and_dimer_virial_on_the_device():
    rng = np.random.default_rng(99)
    worst = 0.0
    for _ in range(40):
        r = 0.85 + 1.45 * rng.random()
        inter = E.Interactions(lj=E.LjParams(0.5 + rng.random(), 1.0, 2.5, True))
        axis = _unit(rng)
        h = 6e-6 * r
        up, _, _ = _dimer(r + h, axis, inter, False)
        dn, _, _ = _dimer(r - h, axis, inter, False)
        pe, w, f = _dimer(r, axis, inter, False)
        fd = -(up - dn) / (2.0 * h)
        worst = max(worst, abs(fd - f) / max(abs(f), 1.0))
        assert abs(w - r * f) <= 1e-13 * max(abs(r * f), 1.0)
    assert worst <= 1e-8, f"worst relative LJ gradient error {worst:.2e}"


def test_criterion_10_fene_gradient_on_the_device():
    """The bonded dimer feels FENE plus the (WCA-range) pair term, like a
    Kremer-Grest bond (r_skin 0.4 as in configs[2]: r_max <= r_cut + r_skin,
    domain.hpp's bond-reach rule); the gradient of their sum is checked at the
    reference's FENE tolerance."""
    rng = np.random.default_rng(199)
    worst = 0.0
    for _ in range(40):
        r = 0.8 + 0.55 * rng.random()
        inter = E.Interactions(lj=E.LjParams(1.0, 1.0, 2.0 ** (1.0 / 6.0), True),
                               fene=E.FeneParams(15.0 + 30.0 * rng.random(), 1.5))
        axis = _unit(rng)
        h = 6e-6 * r
        up, _, _ = _dimer(r + h, axis, inter, True, 0.4)
        dn, _, _ = _dimer(r - h, axis, inter, True, 0.4)
        _, w, f = _dimer(r, axis, inter, True, 0.4)
        fd = -(up - dn) / (2.0 * h)
        worst = max(worst, abs(fd - f) / max(abs(f), 1.0))
        assert abs(w - r * f) <= 1e-12 * max(abs(r * f), 1.0)
    assert worst <= 1e-6, f"worst relative FENE gradient error {worst:.2e}"
