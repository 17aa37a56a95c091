"""The native C++ slab loop (tmd_slab_nccl.cuh) with R > 1 ranks on one GPU.

The loop the multi-GPU bench runs — speculative batches, the fused peer-store
halo, the three-round-trip rebuild with NCCL-style migration and ghost
exchange, load-aware re-cuts — driven by the in-process transport (LocalComm,
tmd_comm.cuh): every rank's context in this process, one host thread per
rank, collectives as stream-event rendezvous (no kernel waits on another
rank's kernel). The same code path as NCCL except the transport object.

Parity: the reference's golden vectors (pair sets bit-exact, PE 1e-12,
trajectories 1e-9 with equal rebuild counts — the decomposition invariance of
test_engine.cpp:242-260 / acceptance.cpp:121-150), the single-context engine,
and bitwise equality with the Python protocol over the same slabs."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import E_RTOL, assert_forces_close, assert_rel, load

pytestmark = pytest.mark.gpu


def system(g):
    inter = E.Interactions()
    bonds = g["bonds"] if "bonds" in g else None
    if "lj" in g:
        eps, sig, rc, sh = g["lj"]
        inter = E.Interactions(lj=E.LjParams(float(eps), float(sig), float(rc), bool(sh)))
    if "fene" in g:
        inter.fene = E.FeneParams(*map(float, g["fene"]))
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"], bonds=bonds)
    cfg = {}
    if "thermostat" in g:
        gamma, temp, seed = g["thermostat"]
        cfg["thermostat"] = E.LangevinParams(float(gamma), float(temp), int(seed))
    return flat, inter, E.EngineConfig(dt=float(g["dt"]), **cfg)


def native(g, R, halo="fused", **kw):
    flat, inter, cfg = system(g)
    return DecomposedEngine(flat, inter, float(g["r_skin"]), cfg, comm=InProcessComm(R),
                            native=True, halo=halo, **kw)


GOLDEN_CASES = [("fcc8_jit", 2), ("fcc8_jit", 3), ("fcc8_jit", 4), ("aniso", 2), ("aniso", 5),
                ("aniso", 8), ("kg_lattice10", 2), ("kg_lattice10", 3), ("kg_lattice10", 6),
                ("langevin_fcc8", 2), ("langevin_fcc8", 4), ("fene_lj8", 3)]


@pytest.mark.parametrize("halo", ["fused", "nccl"])
@pytest.mark.parametrize("name,R", GOLDEN_CASES)
def test_native_loop_vs_golden(name, R, halo):
    g = load(name)
    eng = native(g, R, halo)
    try:
        np.testing.assert_array_equal(eng.local_pairs(), g["pairs"])
        ids, pos, vel, f = eng.local_state()
        np.testing.assert_array_equal(ids, np.sort(g["ids"]))
        assert_forces_close(f, g["forces"])
        if "thermostat" not in g:
            o = eng.observe()
            assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
            assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial")
        steps = int(g["steps"])
        eng.run(steps)
        ids, pos, vel, _ = eng.local_state()
        assert np.abs(pos - g["final_pos"]).max() < 1e-9
        assert np.abs(vel - g["final_vel"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])
        sizes = eng.slab_sizes()
        assert sum(s["n_own"] for s in sizes.values()) == len(g["ids"])
    finally:
        eng.close()


@pytest.mark.parametrize("halo", ["fused", "nccl"])
@pytest.mark.parametrize("name,R", [("fcc8_jit", 3), ("kg_lattice10", 3), ("aniso", 5)])
def test_native_loop_is_bitwise_the_python_protocol(name, R, halo):
    """The C++ loop and decomp.py's protocol over the same slabs take the same
    decisions and produce bitwise identical states, step for step."""
    g = load(name)
    flat, inter, cfg = system(g)
    a = native(g, R, halo)
    b = DecomposedEngine(flat, inter, float(g["r_skin"]), cfg, comm=InProcessComm(R))
    try:
        for k in (1, 9, 30):
            a.run(k)
            b.run(k)
            sa, sb = a.local_state(), b.local_state()
            for x, y in zip(sa, sb):
                np.testing.assert_array_equal(x, y)
            assert a.rebuild_count() == b.rebuild_count()
            np.testing.assert_array_equal(a.local_pairs(), b.local_pairs())
        oa, ob = a.observe(), b.observe()
        assert oa.potential == ob.potential and oa.kinetic == ob.kinetic
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("R", [2, 4, 8])
def test_native_loop_matches_single_context_fcc20(R):
    """32 000 particles, 150 steps with migrations, R slabs (8: 1-2 cell
    layers each) against the single-context engine."""
    flat = E.gen_fcc(20, 0.8442, 1.0, 12345)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R),
                           native=True)
    try:
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
        for k in (1, 49, 100):
            one.run(k)
            dec.run(k)
            o1, o2 = one.observe(), dec.observe()
            assert o2.step == o1.step
            assert_rel(o2.potential, o1.potential, 1e-10, "PE")
            assert_rel(o2.kinetic, o1.kinetic, 1e-10, "KE")
            ids, pos, vel, f = dec.local_state()
            ids1, f1 = one.forces()
            np.testing.assert_array_equal(ids, ids1)
            assert_forces_close(f, f1, rtol=1e-8)
            assert dec.rebuild_count() == one.rebuild_count()
        assert dec.rebuild_count() > 0
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
    finally:
        dec.close()
        one.close()


@pytest.mark.parametrize("R", [3, 4])
def test_native_loop_load_aware_cuts(R):
    """BASELINE configs[3]'s shape: count-balanced cut planes re-evaluated
    at every rebuild inside the native loop (layer histograms all-reduced),
    slabs re-cut, the run tracks the single-context engine."""
    flat = E.gen_fcc_slab(8, 0.8442, 0.7, 5)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R),
                           balance="count", native=True)
    try:
        assert dec.recuts >= 1
        pop = [s["n_own"] for s in dec.slab_sizes().values()]
        assert max(pop) <= 1.5 * flat.size() / R
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
        one.run(100)
        dec.run(100)
        assert_rel(dec.observe().potential, one.observe().potential, 1e-10, "PE")
        ids, pos, vel, f = dec.local_state()
        ids1, f1 = one.forces()
        np.testing.assert_array_equal(ids, ids1)
        assert_forces_close(f, f1, rtol=1e-8)
        assert dec.rebuild_count() == one.rebuild_count()
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
    finally:
        dec.close()
        one.close()


def test_native_run_observed_rows_at_three_ranks():
    g = load("fcc8_jit")
    a = native(g, 3)
    b = native(g, 3)
    try:
        rows = a.run_observed(40, stride=3)
        assert rows[:, 0].tolist() == list(range(3, 41, 3))
        assert a.rebuild_count() > 0
        done = 0
        for r in rows:
            b.run(int(r[0]) - done)
            done = int(r[0])
            o = b.observe()
            assert_rel(r[1], o.kinetic, 1e-12, f"KE at {done}")
            assert_rel(r[2], o.potential, 1e-12, f"PE at {done}")
            assert_rel(r[4], o.virial, 1e-12, f"W at {done}")
    finally:
        a.close()
        b.close()


def test_a_failing_rank_releases_its_peers():
    """Two coincident particles inside one slab: that rank raises the
    reference's overlap PhysicsError; its peers, waiting in a collective, are
    released ("a peer rank failed") and the engine reports the real error."""
    g = load("fcc8_jit")
    pos = g["pos"].copy()
    pos[1] = pos[0]
    flat = E.FlatConfig(g["box"], g["ids"], pos, g["vel"])
    with pytest.raises(E.PhysicsError, match="overlapping particles"):
        DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                         E.EngineConfig(dt=float(g["dt"])), comm=InProcessComm(3), native=True)


def test_native_loop_section_timers():
    """SectionTimers of the native loop (CUDA-event phases on each rank's
    stream): Forces, Comm (rebuild-test all-reduce, migration, ghosts),
    Integrate, Neigh (decision, list build) and Resort are filled and add up
    to about the elapsed time."""
    flat = E.gen_fcc(10, 0.8442, 1.0, 3)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3,
                           E.EngineConfig(dt=0.005, section_timers=True),
                           comm=InProcessComm(3), native=True)
    try:
        dec.run(120)
        t = dec.timers()
        assert dec.rebuild_count() > 5
        for sec in E.Section:
            assert t[sec] > 0.0, sec
        assert 0.5 * t.elapsed <= t.section_sum() <= 1.05 * t.elapsed, t
    finally:
        dec.close()


def test_local_state_into_caller_buffers():
    """local_state(out=...) (one rank per process: the bench's pinned
    download buffers, sized for the whole system) equals local_state()."""
    g = load("fcc8_jit")
    eng = native(g, 1)
    try:
        eng.run(30)
        ids, pos, vel, _ = eng.local_state()
        n = len(g["ids"])
        out = (np.empty(n + 5, np.int64), np.empty((n + 5, 3)), np.empty((n + 5, 3)))
        i2, p2, v2, f2 = eng.local_state(out=out)
        assert f2 is None
        np.testing.assert_array_equal(i2, ids)
        np.testing.assert_array_equal(p2, pos)
        np.testing.assert_array_equal(v2, vel)
    finally:
        eng.close()


@pytest.mark.parametrize("bad", [0, 2])
def test_fused_halo_falls_back_when_a_rank_cannot_map_its_peers(bad, monkeypatch, capfd):
    """One rank fails to map a neighbour's position buffers (injected): every
    rank agrees to use the message halo, and the run is bitwise the
    halo="nccl" run (same rebuild steps, same states). With
    TMD_HALO_STRICT=1 (the test suite's default) the same failure raises."""
    g = load("fcc8_jit")
    monkeypatch.setenv("TMD_HALO_FAIL_INJECT", str(bad))
    with pytest.raises(E.CudaError, match="fused halo unavailable"):
        native(g, 3, "fused")
    monkeypatch.setenv("TMD_HALO_STRICT", "0")
    a = native(g, 3, "fused")
    monkeypatch.delenv("TMD_HALO_FAIL_INJECT")
    b = native(g, 3, "nccl")
    try:
        err = capfd.readouterr().err
        assert "fused peer-store halo unavailable" in err and f"rank {bad}" in err
        for k in (1, 9, 30):
            a.run(k)
            b.run(k)
            for x, y in zip(a.local_state(), b.local_state()):
                np.testing.assert_array_equal(x, y)
            assert a.rebuild_count() == b.rebuild_count()
    finally:
        a.close()
        b.close()


def _planted_far_slab(seed, n_pairs=400, L=200.0, rv=2.8):
    """Pairs planted at |r - r_v| of a few ulps in a large box, all in its
    upper half (the slabs of the high ranks) and many along z: the FP32
    prefilter must use coordinates relative to the brick's GLOBAL origin on
    every slab, or its rounding error (~1e-5 at |z| ~ 150) outgrows the exact
    band and membership goes wrong."""
    rng = np.random.default_rng(seed)
    deltas = np.array([0.0, 1e-16, -1e-16, 2e-16, -2e-16, 1e-13, -1e-13, 1e-9, -1e-9])
    p = rng.uniform(0.0, L, (n_pairs, 3))
    p[:, 2] = rng.uniform(0.55 * L, 0.98 * L, n_pairs)
    u = rng.normal(size=(n_pairs, 3)) * np.array([0.3, 0.3, 1.0])
    u /= np.linalg.norm(u, axis=1)[:, None]
    d = rv * (1.0 + deltas[rng.integers(0, len(deltas), n_pairs)])
    q = p + d[:, None] * u
    pos = np.concatenate([p, q]).reshape(-1, 3) % L
    ids = np.arange(1, 2 * n_pairs + 1, dtype=np.int64)
    return np.array([L, L, L]), ids, pos, np.zeros_like(pos)


@pytest.mark.parametrize("seed", [1, 2])
def test_native_slab_rounding_band_far_from_origin(ref, seed):
    box, ids, pos, vel = _planted_far_slab(seed)
    want = ref.RefEngine(box, ids, pos, vel, r_skin=0.3).pairs()
    eng = DecomposedEngine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3,
                           E.EngineConfig(dt=0.005), comm=InProcessComm(4), native=True)
    try:
        np.testing.assert_array_equal(eng.local_pairs(), want)
    finally:
        eng.close()


def test_native_loop_matches_single_context_1m_r8():
    """configs[1] (1,048,576 particles) as 8 slabs on one GPU against the
    single context: the same pair set, the same rebuild steps, energies to
    1e-10 and forces to 1e-8 after 60 steps of the melting lattice."""
    flat = E.gen_fcc(64, 0.8442, 1.0, 12345)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(8), native=True)
    try:
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
        one.run(60)
        dec.run(60)
        o1, o2 = one.observe(), dec.observe()
        assert_rel(o2.potential, o1.potential, 1e-10, "PE")
        assert_rel(o2.kinetic, o1.kinetic, 1e-10, "KE")
        assert dec.rebuild_count() == one.rebuild_count() > 0
        ids, pos, vel, f = dec.local_state()
        ids1, f1 = one.forces()
        np.testing.assert_array_equal(ids, ids1)
        assert_forces_close(f, f1, rtol=1e-8)
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
    finally:
        dec.close()
        one.close()
