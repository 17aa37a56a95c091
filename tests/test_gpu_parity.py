"""GPU parity: libtmd_gpu.so (through the Python mirror of the C ABI) against
the golden vectors of the reference and against the live reference engine
(oracle/_ref, a prebuilt .so that travels to the GPU box).

Tolerances (north star): pair sets and cells bit-exact; forces 1e-10
relative to max(|F|max, rms F); PE and virial 1e-12 relative to the
exactly-rounded (fsum) sums of the reference's per-pair terms."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from tests._util import (E_RTOL, SYSTEMS, assert_forces_close, assert_rel, load,
                         load_json)

pytestmark = pytest.mark.gpu


def gpu_engine(g, dt=None, **cfg):
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    return E.Engine(flat, E.Interactions(), float(g["r_skin"]),
                    E.EngineConfig(dt=float(dt if dt is not None else g["dt"]), **cfg))


@pytest.mark.parametrize("name", SYSTEMS)
@pytest.mark.parametrize("build", [3, 5, 6])
def test_initial_state_vs_golden(name, build):
    """build 3: warp-per-cell brick kernel; 5: thread-per-particle kernel (the
    choice for sparse cells); 6: warp per cell over the culled candidate
    stream; all must emit the reference's pair set."""
    g = load(name)
    eng = gpu_engine(g, build=build)
    np.testing.assert_array_equal(eng.pairs(), g["pairs"])
    _, cell = eng.cell_of()
    np.testing.assert_array_equal(cell, g["cell"])
    ids, f = eng.forces()
    np.testing.assert_array_equal(ids, np.sort(g["ids"]))
    assert_forces_close(f, g["forces"])
    o = eng.observe()
    assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
    assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial")
    assert_rel(o.kinetic, float(g["ke_ref"]), 1e-13, "KE")
    st = eng.list_stats()
    assert st["entries"] == 2 * len(g["pairs"])
    assert st["in_cut"] == 2 * int(g["n_incut"])
    assert tuple(st["dims"]) == tuple(g["dims"].tolist())
    flat = eng.flatten()
    np.testing.assert_array_equal(flat.pos, g["wrapped"])


@pytest.mark.parametrize("name", SYSTEMS)
def test_builds_emit_the_same_list_order(name):
    """The three list builds emit every particle's entries in the reference's
    stencil order: forces (summed in list order) are bit-identical, so are the
    states after a run with rebuilds."""
    g = load(name)
    outs = []
    for build in (3, 5, 6):
        eng = gpu_engine(g, build=build)
        f0 = eng.forces()[1]
        eng.run(40)
        flat = eng.flatten()
        outs.append((f0, flat.pos, flat.vel, eng.rebuild_count()))
        eng.close()
    for o in outs[1:]:
        np.testing.assert_array_equal(o[0], outs[0][0])
        np.testing.assert_array_equal(o[1], outs[0][1])
        np.testing.assert_array_equal(o[2], outs[0][2])
        assert o[3] == outs[0][3]


@pytest.mark.parametrize("name", ["jit6_s101", "random500_s1", "random500_s2", "random500_s3"])
def test_forces_vs_brute_force_oracle(name):
    """acceptance criterion 1: forces vs oracle_forces_energy <= 1e-10 abs and the
    listed pairs == oracle_pair_set."""
    g = load(name)
    eng = gpu_engine(g)
    _, f = eng.forces()
    order = np.argsort(g["ids"])
    assert np.abs(f - g["oracle_forces"][order]).max() <= 1e-10
    np.testing.assert_array_equal(eng.pairs(), g["oracle_pairs"])


@pytest.mark.parametrize("name", ["jit6_s41_T08", "fcc8_jit", "aniso", "thin"])
@pytest.mark.parametrize("build", [3, 5, 6])
def test_trajectory_vs_golden(name, build):
    g = load(name)
    eng = gpu_engine(g, build=build)
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


def test_fcc20_known_answers():
    s = load_json("fcc20_summary.json")
    f = E.gen_fcc(20, 0.8442, 1.0, 12345)
    eng = E.Engine(f, E.Interactions(), 0.3)
    pr = eng.pairs()
    assert len(pr) == s["pairs"]
    assert int(((pr[:, 0] * 1000003 + pr[:, 1]) % 2147483647).sum()) == s["pair_checksum"]
    _, cell = eng.cell_of()
    assert int((cell.astype(np.int64) * (np.arange(len(cell)) % 9973 + 1)).sum()) == \
        s["cell_checksum"]
    o = eng.observe()
    assert_rel(o.potential, s["pe_fsum"], E_RTOL, "PE")
    assert_rel(o.virial, s["w_fsum"], E_RTOL, "virial")
    assert abs(o.potential / 32000 + 6.3328119926) < 5e-10


# -- live reference engine (oracle/_ref) -------------------------------------------

def test_random_configs_criterion_1(ref):
    """10 random N=500 configs (acceptance.cpp:88-118) against the live
    reference: pair sets exact, forces 1e-10 vs the brute-force oracle."""
    for seed in range(1, 11):
        box, ids, pos, vel = ref.gen_random(500, 0.8442, 0.8, 0.72, seed)
        eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3)
        np.testing.assert_array_equal(eng.pairs(), ref.oracle_pairs(box, ids, pos, 2.8))
        f_or, pe_or = ref.oracle_forces(box, ids, pos)
        _, f = eng.forces()
        assert np.abs(f - f_or).max() <= 1e-10
        assert_rel(eng.observe().potential, pe_or, 1e-11, "PE vs oracle_forces_energy")


def test_one_step_matches_reference(ref):
    """criterion 2 analog: one NVE step from a lattice, positions within 1e-10
    of the reference at n_sub 1, 8 and 64."""
    box, ids, pos, vel = ref.gen_lattice(4096, 0.8442, 0.72, 11)
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3)
    eng.run(1)
    mine = eng.flatten()
    for n_sub in (1, 8, 64):
        r = ref.RefEngine(box, ids, pos, vel, n_sub=n_sub)
        r.run(1)
        rid, rp, _ = r.flatten()
        np.testing.assert_array_equal(mine.id, rid)
        assert np.abs(mine.pos - rp).max() <= 1e-10


def test_nve_drift_criterion_3():
    """acceptance criterion 3: SC lattice N=4000, T=0.6 seed 3, 1000 steps:
    worst drift <= 1e-3 at dt=0.005 and >= 10x smaller at dt=0.001, and
    comparable to the reference's own (fixture)."""
    g = load("lattice4000_s3")
    worst = {}
    for dt in (0.005, 0.001):
        eng = E.Engine(E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"]),
                       E.Interactions(), 0.3, E.EngineConfig(dt=dt))
        o = eng.observe()
        e0 = o.kinetic + o.potential
        assert_rel(e0, float(g[f"e0_dt{dt}"]), 1e-12, "E0")
        tr = []
        for _ in range(100):
            eng.run(10)
            o = eng.observe()
            tr.append(o.kinetic + o.potential)
        tr = np.array(tr)
        worst[dt] = np.abs(tr - e0).max() / abs(e0)
        ref_tr = g[f"dt{dt}"]
        assert np.abs(tr - ref_tr).max() / abs(e0) < 1e-6
    assert worst[0.005] <= 1e-3
    assert worst[0.005] / worst[0.001] >= 10.0
    assert abs(worst[0.005] / float(g["worst_dt0.005"]) - 1.0) < 0.05


def test_free_streaming_through_resorts():
    """test_engine.cpp:66-99: force-free particles move in straight lines,
    unchanged by >= 5 resorts."""
    f = E.FlatConfig(np.full(3, 12.0), np.array([0, 1]),
                     np.array([[1.0, 2.0, 3.0], [7.0, 9.0, 4.0]]),
                     np.array([[0.8, -0.3, 0.5], [-0.2, 0.4, -0.7]]))
    eng = E.Engine(f, E.Interactions(), 0.4, E.EngineConfig(dt=0.01))
    eng.run(400)
    assert eng.rebuild_count() >= 5
    out = eng.flatten()
    t = 0.01 * 400
    want = f.pos + f.vel * t
    want -= 12.0 * np.floor(want / 12.0)
    assert np.abs(out.pos - want).max() <= 1e-9
    np.testing.assert_array_equal(out.vel, f.vel)


def _jittered(side, edge, seed, jitter, temperature):
    from oracle import make_golden as mg
    return mg.jittered_lattice(side, edge, seed, jitter, temperature)


def test_velocity_flip_retraces():
    """test_engine.cpp:165-197: 40 steps, flip velocities, 40 steps back,
    within 1e-12."""
    box, ids, pos, vel = _jittered(4, 6.0, 3, 0.05, 0.3)
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.4,
                   E.EngineConfig(dt=0.002))
    start = eng.flatten()
    eng.run(40)
    assert eng.rebuild_count() == 0
    mid = eng.flatten()
    eng.set_velocities(mid.id, -mid.vel)
    eng.run(40)
    back = eng.flatten()
    np.testing.assert_array_equal(back.id, start.id)
    assert np.abs(back.pos - start.pos).max() <= 1e-12
    assert np.abs(back.vel + start.vel).max() <= 1e-12


def test_energy_conserved_200_steps():
    """test_engine.cpp:199-212."""
    box, ids, pos, vel = _jittered(6, 7.2, 17, 0.05, 0.8)
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3,
                   E.EngineConfig(dt=0.002))
    o = eng.observe()
    e0 = o.kinetic + o.potential
    worst = 0.0
    for _ in range(200):
        eng.step()
        o = eng.observe()
        worst = max(worst, abs(o.kinetic + o.potential - e0))
    assert worst / abs(e0) <= 1e-3


def test_zero_steps_and_timers():
    """test_engine.cpp:284-321."""
    box, ids, pos, vel = _jittered(4, 6.0, 61, 0.05, 0.5)
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3)
    eng.run(0)
    assert eng.step_count() == 0
    t = eng.timers()
    assert t.elapsed == 0.0 and t.section_sum() == 0.0
    out = eng.flatten()
    want = pos - 6.0 * np.floor(pos / 6.0)
    np.testing.assert_array_equal(out.pos, want)
    assert eng.potential_energy() != 0.0

    box, ids, pos, vel = _jittered(4, 6.0, 71, 0.02, 0.0)
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.4,
                   E.EngineConfig(dt=0.001))
    eng.run(5)
    t = eng.timers()
    assert eng.rebuild_count() == 0
    assert t[E.Section.kResort] == 0.0
    assert t[E.Section.kForces] > 0.0
    assert t[E.Section.kIntegrate] > 0.0
    assert t[E.Section.kNeigh] > 0.0
    assert t.elapsed > 0.0
    assert t.section_sum() <= t.elapsed * 1.5 + 1e-3


def test_rebuild_trigger_half_skin():
    """test_neighbor.cpp:185-201 in engine form: a displacement of 0.21 > skin/2
    = 0.2 triggers exactly one rebuild; 0.19 does not."""
    for v, want in ((0.19, 0), (0.21, 1)):
        f = E.FlatConfig(np.full(3, 12.0), np.array([0, 1]),
                         np.array([[1.0, 2.0, 3.0], [7.0, 9.0, 4.0]]),
                         np.array([[v, 0.0, 0.0], [0.0, 0.0, 0.0]]))
        eng = E.Engine(f, E.Interactions(), 0.4, E.EngineConfig(dt=1.0))
        eng.run(1)
        assert eng.rebuild_count() == want


def test_overlap_is_a_physics_error():
    """test_neighbor.cpp:254-268: coincident particles raise PhysicsError."""
    f = E.FlatConfig(np.full(3, 8.5), np.array([0, 1]),
                     np.array([[4.0, 4.0, 4.0], [4.0, 4.0, 4.0]]), None)
    with pytest.raises(E.PhysicsError, match="overlapping particles: ids 0 and 1"):
        E.Engine(f, E.Interactions(), 0.3)


def test_non_finite_dynamics_name_the_step():
    """test_engine.cpp:369-382 analog: a velocity that overflows positions is
    reported as a PhysicsError carrying the step number."""
    box, ids, pos, vel = _jittered(4, 6.0, 83, 0.05, 0.1)
    vel[5] = [np.inf, 0.0, 0.0]
    eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3)
    with pytest.raises(E.PhysicsError, match=r"non-finite.*\(at step \d+\)"):
        eng.run(3)


def test_flatten_into_caller_buffers():
    """flatten(out=...) fills caller-owned (e.g. pinned) arrays in place with
    exactly what flatten() returns; wrong shapes or dtypes are ConfigError."""
    f = E.gen_fcc(6, 0.8442, 1.0, 99)
    eng = E.Engine(f, E.Interactions(), 0.3)
    eng.run(30)
    n = f.size()
    out = E.FlatConfig(f.box, np.zeros(n, np.int64), np.zeros((n, 3)), np.zeros((n, 3)))
    pos_buf = out.pos
    got = eng.flatten(out=out)
    want = eng.flatten()
    assert got is out and out.pos is pos_buf
    np.testing.assert_array_equal(out.id, want.id)
    np.testing.assert_array_equal(out.pos, want.pos)
    np.testing.assert_array_equal(out.vel, want.vel)
    bad = E.FlatConfig(f.box, np.zeros(n, np.int64), np.zeros((n + 1, 3)), np.zeros((n, 3)))
    with pytest.raises(E.ConfigError):
        eng.flatten(out=bad)
    eng.close()


def test_deterministic_bitwise():
    """acceptance criterion 9 analog: two identical runs are bit-identical."""
    f = E.gen_fcc(8, 0.8442, 1.0, 4242)
    outs = []
    for _ in range(2):
        eng = E.Engine(f, E.Interactions(), 0.3)
        eng.run(150)
        outs.append(eng.flatten())
    np.testing.assert_array_equal(outs[0].pos, outs[1].pos)
    np.testing.assert_array_equal(outs[0].vel, outs[1].vel)


def test_fixed_capacity_overflow_rolls_back_and_grows():
    """A list capacity far too small forces the overflow/rollback path; the
    result must equal the auto-capacity run bit for bit."""
    f = E.gen_fcc(8, 0.8442, 1.0, 99)
    a = E.Engine(f, E.Interactions(), 0.3)
    a.run(60)
    b = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(nbr_capacity=8))
    b.run(60)
    fa, fb = a.flatten(), b.flatten()
    assert np.abs(fa.pos - fb.pos).max() < 1e-9
    assert b.list_stats()["capacity"] >= b.list_stats()["max_count"]


@pytest.mark.slow
def test_32k_1000_steps_vs_reference(ref):
    """Config 1 (BASELINE.json configs[0]) end to end against the live reference."""
    f = E.gen_fcc(20, 0.8442, 1.0, 12345)
    eng = E.Engine(f, E.Interactions(), 0.3)
    r = ref.RefEngine(f.box, f.id, f.pos, f.vel, r_skin=0.3)
    o0 = eng.observe()
    e0 = o0.kinetic + o0.potential
    worst = 0.0
    for _ in range(100):
        eng.run(10)
        o = eng.observe()
        worst = max(worst, abs(o.kinetic + o.potential - e0) / abs(e0))
    r.run(1000)
    ro = r.observe()
    o = eng.observe()
    assert_rel((o.kinetic + o.potential), ro["kinetic"] + ro["potential"], 1e-7, "E(1000)")
    assert abs(o.temperature - ro["temperature"]) < 1e-3
    assert abs(eng.rebuild_count() - r.rebuild_count()) <= 3
    assert worst < 2e-4  # reference: 1.154e-4


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("name", ["random500_s1", "fcc8_jit", "aniso", "thin"])
def test_kernel_variants_agree(name, variant):
    """Both force/list kernel variants (thread-per-particle L1 gathers and the
    brick-staged shared-memory kernels) meet the same parity bar."""
    g = load(name)
    eng = gpu_engine(g, variant=variant)
    np.testing.assert_array_equal(eng.pairs(), g["pairs"])
    _, f = eng.forces()
    assert_forces_close(f, g["forces"])
    o = eng.observe()
    assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
    assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial")
    eng.run(25)
    o = eng.observe()
    assert o.step == 25


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["random500_s1", "fcc8_jit", "aniso", "thin"])
def test_force_lanes_agree(name, lanes):
    """Variant 3 with 1, 2, 4 or 8 threads per particle (k_forces_l1 /
    k_forces_lanes; small systems default to more lanes): the same parity bar
    at the initial state and along the golden trajectory."""
    g = load(name)
    eng = gpu_engine(g, lanes=lanes)
    _, f = eng.forces()
    assert_forces_close(f, g["forces"])
    o = eng.observe()
    assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
    assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial")
    if "final_pos" in g:
        eng.run(int(g["steps"]))
        assert np.abs(eng.flatten().pos - g["final_pos"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])


@pytest.mark.parametrize("lanes", [1, 2, 4, 8])
def test_force_lanes_report_overlap(lanes):
    """Coincident particles raise PhysicsError whichever lane of the particle
    holds the r2 == 0 entry (test_neighbor.cpp:254-268)."""
    box, ids, pos, vel = _jittered(4, 6.0, 91, 0.05, 0.1)
    pos[17] = pos[3]
    f = E.FlatConfig(box, ids, pos, vel)
    with pytest.raises(E.PhysicsError, match="overlapping particles"):
        E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(lanes=lanes))


def test_force_lanes_bitwise_graph_vs_eager():
    f = E.gen_fcc(8, 0.8442, 1.0, 778)
    for lanes in (2, 8):
        eager = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(lanes=lanes))
        graph = E.Engine(f, E.Interactions(), 0.3,
                         E.EngineConfig(lanes=lanes, section_timers=False))
        eager.run(60)
        graph.run(60)
        np.testing.assert_array_equal(eager.flatten().pos, graph.flatten().pos)
        eager.close()
        graph.close()


def test_variants_bitwise_same_list_membership_1m_scale():
    """At a 256K-particle FCC (64^3 cells... 40^3x4) the two variants list the
    same pairs and agree on energies to 1e-12."""
    f = E.gen_fcc(40, 0.8442, 1.0, 5)
    a = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(variant=1))
    b = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(variant=2))
    a.run(30)
    b.run(30)
    np.testing.assert_array_equal(a.pairs(), b.pairs())
    oa, ob = a.observe(), b.observe()
    assert_rel(ob.potential, oa.potential, 1e-12, "PE v1 vs v2")
    assert_rel(ob.virial, oa.virial, 1e-12, "virial v1 vs v2")


@pytest.mark.parametrize("cells,steps", [(8, 120), (24, 40)])
def test_staged_forces_bitwise_equal_to_global_gathers(cells, steps):
    """Variant 2 (neighbour positions gathered from shared memory, list
    entries = brick staging indices) and variant 3 (gathers from global
    memory, entries = global slots) list the same entries in the same order
    and evaluate them with the same arithmetic: forces, energies and whole
    trajectories are bitwise equal (k_forces_staged vs k_forces_l1)."""
    f = E.gen_fcc(cells, 0.8442, 1.0, 4242)
    a = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(variant=3, lanes=1))
    b = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(variant=2))
    assert b.kernel_config()["variant"] == 2
    np.testing.assert_array_equal(a.pairs(), b.pairs())
    np.testing.assert_array_equal(a.forces()[1], b.forces()[1])
    a.run(steps)
    b.run(steps)
    fa, fb = a.flatten(), b.flatten()
    np.testing.assert_array_equal(fa.pos, fb.pos)
    np.testing.assert_array_equal(fa.vel, fb.vel)
    oa, ob = a.observe(), b.observe()  # (partial sums per brick vs per 128 particles)
    assert_rel(ob.potential, oa.potential, 1e-13, "PE staged vs global")
    assert_rel(ob.virial, oa.virial, 1e-13, "virial staged vs global")
    assert a.rebuild_count() == b.rebuild_count() > 0
    a.close()
    b.close()


def test_default_kernel_choice():
    """Dense systems run the global-gather kernel with one thread per particle
    (measured fastest), small ones several threads per particle;
    a staged-kernel request for a sparse system falls back to it."""
    big = E.Engine(E.gen_fcc(32, 0.8442, 1.0, 1), E.Interactions(), 0.3, E.EngineConfig())
    assert big.kernel_config() == dict(variant=3, lanes=1, build_kind=6)
    big.close()
    small = E.Engine(E.gen_fcc(8, 0.8442, 1.0, 1), E.Interactions(), 0.3, E.EngineConfig())
    assert small.kernel_config()["variant"] == 3 and small.kernel_config()["lanes"] > 1
    small.close()


@pytest.mark.parametrize("variant", [1, 2, 3])
def test_graph_mode_is_bitwise_identical_to_eager(variant):
    """With section timers off a run executes as CUDA graphs whose rebuild
    branch is a device-evaluated conditional node; the result must equal the
    eagerly launched run bit for bit (same kernels, same order)."""
    f = E.gen_fcc(8, 0.8442, 1.0, 777)
    eager = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(variant=variant, graphs=False))
    graph = E.Engine(f, E.Interactions(), 0.3,
                     E.EngineConfig(variant=variant, section_timers=False))
    for chunk in (40, 15, 3, 97):
        eager.run(chunk)
        graph.run(chunk)
    a, b = eager.flatten(), graph.flatten()
    np.testing.assert_array_equal(a.pos, b.pos)
    np.testing.assert_array_equal(a.vel, b.vel)
    assert eager.rebuild_count() == graph.rebuild_count() > 0
    oa, ob = eager.observe(), graph.observe()
    assert oa.potential == ob.potential and oa.kinetic == ob.kinetic


def test_graph_mode_trajectory_vs_golden():
    g = load("fcc8_jit")
    eng = gpu_engine(g, section_timers=False)
    eng.run(int(g["steps"]))
    flat = eng.flatten()
    assert np.abs(flat.pos - g["final_pos"]).max() < 1e-9
    assert eng.rebuild_count() == int(g["rebuilds"])


def test_run1_loop_equals_one_run():
    """Checkpoints every 256 steps, not every call: run(1) x N is the same
    computation as run(N), bit for bit, and observe() reuses the kick's
    kinetic partials."""
    f = E.gen_fcc(8, 0.8442, 1.0, 7)
    a = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(section_timers=False))
    a.run(40)
    b = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(section_timers=False))
    for _ in range(40):
        b.run(1)
        ob = b.observe()
    oa = a.observe()
    fa, fb = a.flatten(), b.flatten()
    np.testing.assert_array_equal(fa.pos, fb.pos)
    np.testing.assert_array_equal(fa.vel, fb.vel)
    assert (oa.kinetic, oa.potential) == (ob.kinetic, ob.potential)
    assert a.rebuild_count() == b.rebuild_count()


def test_overflow_inside_a_run1_loop_replays_from_the_checkpoint():
    f = E.gen_fcc(8, 0.8442, 1.0, 99)
    a = E.Engine(f, E.Interactions(), 0.3)
    a.run(60)
    b = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(nbr_capacity=8))
    for _ in range(60):
        b.run(1)
    assert b.step_count() == 60
    assert np.abs(a.flatten().pos - b.flatten().pos).max() < 1e-9


@pytest.mark.parametrize("timers", [False, True])
def test_run_observed_rows_equal_observe_after_each_run(timers):
    """run_observed records on the device exactly what observe() reports
    after run(stride) calls (golden trajectory system, with rebuilds)."""
    g = load("fcc8_jit")
    a = gpu_engine(g, section_timers=timers)
    rows = a.run_observed(60, stride=4)
    assert rows[:, 0].tolist() == list(range(4, 61, 4))
    b = gpu_engine(g, section_timers=timers)
    for r in rows:
        b.run(4)
        o = b.observe()
        assert (o.step, o.kinetic, o.potential, o.temperature, o.virial) == tuple(r)
    # stride 1 continues from step 60, and rows match the golden trace steps
    rows1 = a.run_observed(140, stride=1)
    assert rows1[0, 0] == 61 and rows1[-1, 0] == 200 and len(rows1) == 140
    for row in g["trace"]:
        if row[0] > 60:
            k = int(row[0]) - 61
            assert_rel(rows1[k, 1] + rows1[k, 2], row[1] + row[2], 1e-10, "E")


@pytest.mark.parametrize("timers", [True, False])
def test_empty_system(timers):
    """No particles: the engine builds, steps and observes zeros (the
    reference's KineticResult reports T = 0 for no particles)."""
    f = E.FlatConfig(np.full(3, 12.0), np.zeros(0, np.int64), np.zeros((0, 3)), None)
    eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(section_timers=timers))
    o = eng.observe()
    assert (o.kinetic, o.potential, o.virial, o.temperature) == (0.0, 0.0, 0.0, 0.0)
    eng.run(10)
    assert eng.step_count() == 10 and eng.observe().temperature == 0.0
    assert eng.flatten().size() == 0 and len(eng.pairs()) == 0


def test_closed_engine_blocks_are_reused_safely():
    """A closed engine's device blocks go to the process cache and back out to
    the next engine: that engine starts from its own state (no leftovers of
    the previous list or arrays), before and after the cache is released."""
    g = load("jit6_s41_T08")
    ref_eng = gpu_engine(g)
    ref_eng.run(30)
    want = ref_eng.flatten()
    ref_eng.close()
    for release in (False, True):
        big = E.Engine(E.gen_fcc(12, 0.8442, 1.0, 5), E.Interactions(), 0.3)
        big.run(5)
        big.close()
        if release:
            E.release_cache()
        eng = gpu_engine(g)
        eng.run(30)
        got = eng.flatten()
        np.testing.assert_array_equal(got.pos, want.pos)
        np.testing.assert_array_equal(got.vel, want.vel)
        eng.close()


@pytest.mark.parametrize("n,rho,min_d", [(1154, 0.8442, 0.8), (1641, 1.2, 0.7)])
def test_cells_of_more_than_a_warp(ref, n, rho, min_d):
    """Cells holding more than 32 particles (3x3x3 grid of 3.7-sigma cells):
    the warp-per-cell builds take them in several passes of 32 lanes, with the
    culled stream's bounding box per pass; every build kind must still emit
    the reference's pair set, in the same order (bitwise forces)."""
    box, ids, pos, vel = ref.gen_random(n, rho, min_d, 0.72, 7)
    want_pairs = ref.oracle_pairs(box, ids, pos, 2.8)
    want_f, want_pe = ref.oracle_forces(box, ids, pos)
    forces = []
    for build in (3, 5, 6):
        eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3,
                       E.EngineConfig(build=build))
        assert tuple(eng.list_stats()["dims"]) == (3, 3, 3)
        _, cell = eng.cell_of()
        assert np.bincount(cell).max() > 32
        np.testing.assert_array_equal(eng.pairs(), want_pairs)
        _, f = eng.forces()
        assert np.abs(f - want_f).max() <= 1e-10
        assert_rel(eng.observe().potential, want_pe, 1e-11, "PE")
        forces.append(f)
        eng.close()
    np.testing.assert_array_equal(forces[0], forces[1])
    np.testing.assert_array_equal(forces[0], forces[2])


def planted_pairs(seed, n_pairs=300, L=20.0, rv=2.8):
    """A dilute gas of planted pairs at separations straddling r_v by a few
    ulps (and exactly r_v as written in decimal), many of them across the
    periodic boundary: every one of them lands in the FP32 prefilter's
    rounding band, where membership is the exact FP64 decision."""
    rng = np.random.default_rng(seed)
    deltas = np.array([0.0, 1e-16, -1e-16, 2e-16, -2e-16, 5e-16, -5e-16, 1e-13, -1e-13,
                       1e-9, -1e-9])
    p = rng.uniform(0.0, L, (n_pairs, 3))
    near = rng.random(n_pairs) < 0.4  # put some pairs at a face of the box
    p[near, rng.integers(0, 3, near.sum())] = rng.uniform(0.0, 0.5, near.sum())
    u = rng.normal(size=(n_pairs, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    d = rv * (1.0 + deltas[rng.integers(0, len(deltas), n_pairs)])
    q = p + d[:, None] * u
    pos = np.concatenate([p, q]).reshape(-1, 3)
    ids = np.arange(1, 2 * n_pairs + 1, dtype=np.int64)
    return np.array([L, L, L]), ids, pos, np.zeros_like(pos)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_rounding_band_pairs_match_the_reference(ref, seed):
    """Pairs at |r - r_v| of a few ulps: the pair set of every build kind is
    the reference engine's own (its rounding, its image-shift orientation)."""
    box, ids, pos, vel = planted_pairs(seed)
    want = ref.RefEngine(box, ids, pos, vel, r_skin=0.3).pairs()
    n = len(ids) // 2
    kept = set(map(tuple, want.tolist()))
    planted_in = sum((k + 1, k + 1 + n) in kept for k in range(n))
    assert 0.3 * n < planted_in < 0.8 * n  # the band really splits them
    for build in (3, 5, 6):
        eng = E.Engine(E.FlatConfig(box, ids, pos, vel), E.Interactions(), 0.3,
                       E.EngineConfig(build=build))
        np.testing.assert_array_equal(eng.pairs(), want)
        eng.close()


def test_section_timers_in_graph_mode():
    """SectionTimers on the production path (CUDA graphs): the device stamps
    each phase of each step (%globaltimer), so the five sections are filled
    without eager launches — they add up to the elapsed time, Resort is
    booked only on rebuild steps, and the split agrees with the eager
    (CUDA-event) timers."""
    f = E.gen_fcc(12, 0.8442, 1.0, 4)
    res = {}
    for graphs in (True, False):
        eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(section_timers=True,
                                                                graphs=graphs))
        eng.run(300)
        t = eng.timers()
        assert eng.rebuild_count() > 10
        for sec in E.Section:
            if sec != E.Section.kComm:
                assert t[sec] > 0.0, (graphs, sec)
        assert t[E.Section.kComm] == 0.0
        assert 0.7 * t.elapsed <= t.section_sum() <= 1.02 * t.elapsed, (graphs, t)
        res[graphs] = t
        eng.close()
    g, e = res[True], res[False]
    # the graph run is the faster one, and its Forces share is the larger
    assert g.elapsed < e.elapsed
    assert g[E.Section.kForces] / g.section_sum() > 0.5 * e[E.Section.kForces] / e.section_sum()
