"""PairIndexList on the device (neighbor_list.hpp:193-268): the explicit pair
list and its Newton-3 traversal agree with the sorted (full-list) layout —
the reference's test_neighbor.cpp:202-259 ("explicit pair indices agree with
the sorted layout": same pairs; forces to 1e-12, energy to 1e-12 relative)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import ref
from paper_2109_10876_b200 import engine as E
from tests._util import assert_rel, load

pytestmark = pytest.mark.gpu


def _sorted_rows(p):
    p = np.sort(p, axis=1)
    return p[np.lexsort((p[:, 1], p[:, 0]))]


@pytest.mark.parametrize("name", ["jit6_s101", "fcc8_jit", "aniso", "thin", "random500_s2"])
def test_pair_list_equals_the_sorted_layout(name):
    g = load(name)
    eng = E.Engine(E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"]), E.Interactions(),
                   float(g["r_skin"]), E.EngineConfig(dt=float(g["dt"])))
    try:
        m = eng.build_pair_index_list()
        pl = eng.pair_index_list()
        assert pl.shape == (m, 2)
        np.testing.assert_array_equal(_sorted_rows(pl), eng.pairs())
        np.testing.assert_array_equal(_sorted_rows(pl), g["pairs"])  # the reference's set
        pe1, w1 = eng.compute_forces()
        _, f1 = eng.forces()
        pe2, w2 = eng.compute_forces_pairs()
        ids, f2 = eng.forces()
        assert_rel(pe2, pe1, 1e-12, "PE")
        assert_rel(w2, w1, 1e-12, "virial")
        assert np.abs(f2 - f1).max() <= 1e-12 * max(1.0, np.abs(f1).max())
        assert_rel(pe2, float(g["pe_fsum"]), 1e-12, "PE vs reference")
    finally:
        eng.close()


def test_pair_list_vs_reference_engine_after_a_run():
    """50 NVE steps of a jittered lattice, then both traversals against the
    reference engine's pair set and forces at the same state."""
    g = load("fcc8_jit")
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    eng = E.Engine(flat, E.Interactions(), 0.3, E.EngineConfig(dt=0.005))
    try:
        eng.run(50)
        mid = eng.flatten()
        r = ref.RefEngine(mid.box, mid.id, mid.pos, mid.vel, r_skin=0.3, dt=0.005)
        eng2 = E.Engine(mid, E.Interactions(), 0.3, E.EngineConfig(dt=0.005))
        eng2.build_pair_index_list()
        np.testing.assert_array_equal(_sorted_rows(eng2.pair_index_list()), r.pairs())
        eng2.compute_forces_pairs()
        ids, f = eng2.forces()
        ids_r, f_r = r.forces()
        np.testing.assert_array_equal(ids, ids_r)
        assert np.abs(f - f_r).max() <= 1e-10 * np.abs(f_r).max()
        r.close()
        eng2.close()
    finally:
        eng.close()


def test_pair_list_goes_stale_after_a_resort():
    f = E.gen_fcc(6, 0.8442, 1.0, 5)
    eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005))
    try:
        eng.build_pair_index_list()
        eng.run(2)  # no rebuild yet: slots unchanged, the list still holds
        assert eng.rebuild_count() == 0
        eng.compute_forces_pairs()
        eng.run(200)
        assert eng.rebuild_count() > 0
        with pytest.raises(E.StateError, match="stale"):
            eng.compute_forces_pairs()
        with pytest.raises(E.StateError):
            E.Engine(f, E.Interactions(), 0.3).compute_forces_pairs()  # never built
    finally:
        eng.close()


def test_pair_traversal_timing_hook():
    f = E.gen_fcc(10, 0.8442, 1.0, 5)
    eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005))
    try:
        m = eng.build_pair_index_list()
        assert m == len(eng.pairs())
        assert eng.time_pair_traversal(3) > 0.0
        assert eng.time_force_kernel(3) > 0.0
    finally:
        eng.close()
