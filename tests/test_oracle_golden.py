"""Pins the C restatement (oracle/taskmd_oracle.c) against the golden vectors
produced by the reference itself (oracle/make_golden.py) and against the
reference's own known-answer tests (test_potentials.cpp, test_grid.cpp,
acceptance.cpp). CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import port
from tests._util import (E_RTOL, SYSTEMS, assert_forces_close, assert_rel, load,
                         load_json)


# -- LJ (test_potentials.cpp:33-89) --------------------------------------------

def test_lj_table_bit_exact():
    g = load("lj_scalar")
    for r2, sh, e, ff in g["table"]:
        pe, pff = port.lj_eval(r2, shifted=bool(sh))
        assert pe == e and pff == ff, r2
    np.testing.assert_array_equal(port.lj_prepare(shifted=True), g["prep_shifted"])
    np.testing.assert_array_equal(port.lj_prepare(shifted=False), g["prep_unshifted"])


def test_lj_textbook_anchors():
    rmin = 2.0 ** (1.0 / 6.0)
    e, ff = port.lj_eval(rmin * rmin, shifted=False)
    assert abs(e + 1.0) <= 1e-12 and abs(ff) <= 1e-12
    assert port.lj_eval(1.0, shifted=False)[0] == 0.0
    e, _ = port.lj_eval(2.5 * 2.5 * (1.0 - 1e-14), shifted=False)
    assert abs(e + 0.016316891) <= 5e-10


def test_lj_zero_at_and_beyond_cutoff():
    for r2 in (6.25, 9.0):
        assert port.lj_eval(r2) == (0.0, 0.0)


def test_lj_shift_continuity_and_fd_gradient():
    q = port.lj_prepare(shifted=True)
    e_raw, _ = port.lj_eval(6.25 * (1 - 1e-13), shifted=False)
    assert abs(q[4] - e_raw) <= 1e-11
    assert abs(port.lj_eval(6.25 * (1 - 1e-13))[0]) < 1e-11
    rng = np.random.default_rng(11)
    for r in rng.uniform(0.8, 2.5, 100):
        if r * r >= 6.25:
            continue
        h = 1e-4 * r
        E = lambda x: port.lj_eval(x * x, shifted=False)[0]  # noqa: E731
        d = (8 * (E(r + h) - E(r - h)) - (E(r + 2 * h) - E(r - 2 * h))) / (12 * h)
        ff = port.lj_eval(r * r, shifted=False)[1]
        assert abs(ff - (-d / r)) <= 1e-8 * max(abs(ff), abs(d / r)) + 1e-9


# -- grid + binning (test_grid.cpp:8-95, acceptance criterion 6) ------------------

def test_cell_grids_match_reference():
    for g in load_json("grids.json"):
        dims, cl = port.cell_grid(np.array(g["box"]), g["r_cut"], g["r_skin"])
        assert dims.tolist() == g["dims"]
        assert cl.tolist() == g["cell_len"]
    dims, _ = port.cell_grid(np.array([67.7177] * 3), 2.5, 0.3)
    assert dims.tolist() == [24, 24, 24]


def test_wrap_and_cell_bit_exact():
    b = load("binning")
    dims, cl = port.cell_grid(b["box"], float(b["r_cut"]), float(b["r_skin"]))
    for p, w, c in zip(b["pos"], b["wrapped"], b["cell"]):
        wp = np.array([port.wrap1(p[k], b["box"][k]) for k in range(3)])
        assert np.array_equal(wp, w), p
        assert port.cell_of(wp, dims, cl) == c


def test_upper_face_clamp():
    dims, cl = port.cell_grid(np.array([12.0] * 3), 2.5, 0.5)
    c = port.cell_of(np.array([12.0 - 1e-13, 0.0, 6.0]), dims, cl)
    assert c == 3 + 4 * (0 + 4 * 2)


# -- counter RNG + thermal velocities (random.hpp, generators.hpp:19-39) ----------

def test_rng_bit_exact():
    g = load("rng")
    for k, n3, u3 in zip(g["keys"], g["normal3"], g["uniform3"]):
        k = [int(x) for x in k]
        assert np.array_equal(port.counter_normal3(*k), n3)
        assert np.array_equal(port.counter_uniform3(*k), u3)
    np.testing.assert_array_equal(port.thermal_velocities(g["tv_ids"], 1.0, 12345), g["tv"])


# -- systems -------------------------------------------------------------------------

@pytest.mark.parametrize("name", SYSTEMS)
def test_system_initial_state(name):
    g = load(name)
    s = port.PortSystem(g["box"], g["ids"], g["pos"], g["vel"], r_skin=float(g["r_skin"]),
                        dt=float(g["dt"]))
    np.testing.assert_array_equal(s.pairs(), g["pairs"])
    _, cell = s.cell_of()
    np.testing.assert_array_equal(cell, g["cell"])
    _, f = s.forces()
    assert_forces_close(f, g["forces"], rtol=1e-12)
    o = s.observe()
    assert_rel(o["potential"], float(g["pe_fsum"]), 1e-14, "PE vs fsum")
    assert_rel(o["virial"], float(g["w_fsum"]), 1e-13, "virial vs fsum")
    # the reference's running sum is itself only ~1e-12 good
    assert_rel(o["potential"], float(g["pe_ref"]), 1e-11, "PE vs reference running sum")


@pytest.mark.parametrize("name", [n for n in SYSTEMS if "fcc8" in n or n in ("aniso", "thin",
                                                                             "jit6_s41_T08")])
def test_system_trajectory(name):
    g = load(name)
    if "steps" not in g:
        pytest.skip("no trajectory in fixture")
    s = port.PortSystem(g["box"], g["ids"], g["pos"], g["vel"], r_skin=float(g["r_skin"]),
                        dt=float(g["dt"]))
    steps = int(g["steps"])
    every = steps // len(g["trace"])
    for row in g["trace"]:
        s.run(every)
        o = s.observe()
        assert o["step"] == int(row[0])
        e, e_ref = o["kinetic"] + o["potential"], row[1] + row[2]
        assert_rel(e, e_ref, 1e-10, f"energy at step {o['step']}")
    _, p, v = s.flatten()
    assert np.abs(p - g["final_pos"]).max() < 1e-9
    assert np.abs(v - g["final_vel"]).max() < 1e-9
    assert s.rebuild_count() == int(g["rebuilds"])


@pytest.mark.parametrize("name", ["jit6_s101", "random500_s1", "random500_s2", "random500_s3"])
def test_reference_engine_vs_brute_force(name):
    """acceptance criterion 1 on the fixtures: engine forces vs oracle_forces_energy
    (1e-10 abs) and listed pairs vs oracle_pair_set (exact)."""
    g = load(name)
    assert np.abs(g["forces"] - g["oracle_forces"][np.argsort(g["ids"])]).max() <= 1e-10
    np.testing.assert_array_equal(g["pairs"], g["oracle_pairs"])


def test_fcc_generator_and_known_answers():
    box, ids, pos = port.gen_fcc(20, 0.8442)
    s = load_json("fcc20_summary.json")
    assert box[0] == s["L"]
    vel = port.thermal_velocities(ids, 1.0, 12345)
    sysm = port.PortSystem(box, ids, pos, vel)
    pr = sysm.pairs()
    assert len(pr) == s["pairs"] == 39 * 32000
    assert int(((pr[:, 0] * 1000003 + pr[:, 1]) % 2147483647).sum()) == s["pair_checksum"]
    o = sysm.observe()
    assert_rel(o["potential"], s["pe_fsum"], E_RTOL, "32K FCC PE")
    assert_rel(o["virial"], s["w_fsum"], E_RTOL, "32K FCC virial")
    # perfect FCC: U/N = -6.3328119926 (positions only)
    e0 = (o["kinetic"] + o["potential"]) / 32000
    assert abs(o["potential"] / 32000 - (-6.3328119926)) < 5e-10
    assert abs(e0 - (-4.843462539)) < 1e-9
