"""GPU parity of the z-slab decomposition (decomp.py).

All ranks' slab contexts live on one GPU (InProcessComm: the exchanges are
device copies made by the host between kernel launches; no kernel waits on
another rank). The decomposed engine must reproduce the reference's golden
vectors exactly like the single-context engine does: pair sets bit-exact,
forces 1e-10 relative, PE / virial 1e-12 relative, and the golden
trajectories (energy trace, final state, rebuild count)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import E_RTOL, assert_forces_close, assert_rel, load

pytestmark = pytest.mark.gpu


def slab_engine(g, R, **cfg):
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    return DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                            E.EngineConfig(dt=float(g["dt"]), **cfg), comm=InProcessComm(R))


CASES = [("fcc8_jit", 1), ("fcc8_jit", 2), ("fcc8_jit", 3), ("fcc8_jit", 4), ("aniso", 1),
         ("aniso", 2), ("aniso", 5), ("aniso", 10)]


@pytest.mark.parametrize("name,R", CASES)
def test_initial_state_vs_golden(name, R):
    g = load(name)
    eng = slab_engine(g, R)
    try:
        np.testing.assert_array_equal(eng.local_pairs(), g["pairs"])
        ids, pos, vel, f = eng.local_state()
        np.testing.assert_array_equal(ids, np.sort(g["ids"]))
        assert_forces_close(f, g["forces"])
        np.testing.assert_array_equal(pos, g["wrapped"])
        o = eng.observe()
        assert_rel(o.potential, float(g["pe_fsum"]), E_RTOL, "PE")
        assert_rel(o.virial, float(g["w_fsum"]), E_RTOL, "virial")
        assert_rel(o.kinetic, float(g["ke_ref"]), 1e-13, "KE")
        sizes = eng.slab_sizes()
        assert sum(s["n_own"] for s in sizes.values()) == len(g["ids"])
    finally:
        eng.close()


@pytest.mark.parametrize("name,R", [("fcc8_jit", 1), ("fcc8_jit", 2), ("fcc8_jit", 4),
                                    ("aniso", 3)])
def test_trajectory_vs_golden(name, R):
    g = load(name)
    eng = slab_engine(g, R)
    try:
        steps = int(g["steps"])
        every = max(1, steps // len(g["trace"]))
        for row in g["trace"]:
            eng.run(every)
            o = eng.observe()
            assert o.step == int(row[0])
            assert_rel(o.kinetic + o.potential, row[1] + row[2], 1e-10, f"E at step {o.step}")
        ids, pos, vel, f = eng.local_state()
        assert np.abs(pos - g["final_pos"]).max() < 1e-9
        assert np.abs(vel - g["final_vel"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])
    finally:
        eng.close()


@pytest.mark.parametrize("R", [2, 4, 8])
def test_matches_single_context_fcc20(R):
    """32 000 particles, 150 steps with migrations: the decomposed run tracks
    the single-context engine (same pair set after every check, forces and
    energies to the north-star tolerances)."""
    flat = E.gen_fcc(20, 0.8442, 1.0, 12345)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R))
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
        assert dec.exchanged_bytes > 0
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
    finally:
        dec.close()
        one.close()


def test_slab_config_errors():
    g = load("thin")  # 2 z cell layers: too thin to cut
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    with pytest.raises(E.ConfigError):
        DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                         E.EngineConfig(dt=float(g["dt"])), comm=InProcessComm(2))


def _mp_worker(rank, world, port, q):
    """One rank of a multi-process decomposition on GPU 0 (gloo moves the
    buffers through host memory; no kernel waits on another rank)."""
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                init_method=f"tcp://127.0.0.1:{port}")
        from paper_2109_10876_b200.decomp import TorchDistComm
        g = load("fcc8_jit")
        flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
        eng = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                               E.EngineConfig(dt=float(g["dt"])), comm=TorchDistComm(),
                               device_of=lambda r: 0)
        pairs0 = eng.local_pairs()
        eng.run(int(g["steps"]))
        o = eng.observe()
        st = eng.local_state()
        objs = [None] * world
        dist.all_gather_object(objs, (pairs0, st, eng.rebuild_count(), o.kinetic + o.potential))
        eng.close()
        dist.destroy_process_group()
        q.put((rank, "ok", objs if rank == 0 else None))
    except BaseException:
        import traceback
        q.put((rank, "err", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_torch_distributed(world):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r[1] != "ok"]
    assert not errs, errs[0][2]
    objs = res[0][2]
    g = load("fcc8_jit")
    pairs = np.concatenate([o[0] for o in objs])
    pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
    np.testing.assert_array_equal(pairs, g["pairs"])
    ids = np.concatenate([o[1][0] for o in objs])
    order = np.argsort(ids)
    np.testing.assert_array_equal(ids[order], np.sort(g["ids"]))
    pos = np.concatenate([o[1][1] for o in objs])[order]
    vel = np.concatenate([o[1][2] for o in objs])[order]
    assert np.abs(pos - g["final_pos"]).max() < 1e-9
    assert np.abs(vel - g["final_vel"]).max() < 1e-9
    assert all(o[2] == int(g["rebuilds"]) for o in objs)


@pytest.mark.parametrize("R", [3, 4])
def test_load_aware_cuts_on_a_liquid_slab(R):
    """SURVEY §8f f3 on BASELINE configs[3]'s shape (liquid FCC slab in the
    middle third of z): count-balanced cuts re-cut the slabs, and the
    decomposed run still tracks the single-context engine."""
    flat = E.gen_fcc_slab(8, 0.8442, 0.7, 5)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R),
                           balance="count")
    static = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R))
    try:
        assert dec.recuts >= 1
        pop = [s["n_own"] for s in dec.slab_sizes().values()]
        pop_static = [s["n_own"] for s in static.slab_sizes().values()]
        assert max(pop) < max(pop_static)
        assert max(pop) <= 1.5 * flat.size() / R
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
        one.run(100)
        dec.run(100)
        o1, o2 = one.observe(), dec.observe()
        assert_rel(o2.potential, o1.potential, 1e-10, "PE")
        ids, pos, vel, f = dec.local_state()
        ids1, f1 = one.forces()
        np.testing.assert_array_equal(ids, ids1)
        assert_forces_close(f, f1, rtol=1e-8)
        assert dec.rebuild_count() == one.rebuild_count()
        np.testing.assert_array_equal(dec.local_pairs(), one.pairs())
    finally:
        dec.close()
        static.close()
        one.close()


@pytest.mark.parametrize("halo", ["fused", "nccl"])
@pytest.mark.parametrize("name", ["fcc8_jit", "kg_lattice10"])
def test_native_nccl_loop_in_process(name, halo):
    """The C++ step loop (tmd_slab_nccl.cuh) with a one-rank NCCL
    communicator: the slab exchanges its boundary layers with itself."""
    g = load(name)
    inter = E.Interactions()
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    if "bonds" in g:
        eps, sig, rc, sh = g["lj"]
        inter = E.Interactions(lj=E.LjParams(float(eps), float(sig), float(rc), bool(sh)),
                               fene=E.FeneParams(*map(float, g["fene"])))
        flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"], bonds=g["bonds"])
    eng = DecomposedEngine(flat, inter, float(g["r_skin"]), E.EngineConfig(dt=float(g["dt"])),
                           comm=InProcessComm(1), native=True, halo=halo)
    try:
        np.testing.assert_array_equal(eng.local_pairs(), g["pairs"])
        assert_rel(eng.observe().potential, float(g["pe_fsum"]), E_RTOL, "PE")
        eng.run(int(g["steps"]))
        ids, pos, vel, _ = eng.local_state()
        assert np.abs(pos - g["final_pos"]).max() < 1e-9
        assert np.abs(vel - g["final_vel"]).max() < 1e-9
        assert eng.rebuild_count() == int(g["rebuilds"])
    finally:
        eng.close()


@pytest.mark.parametrize("native", [True, False])
def test_decomposed_run_observed_rows(native):
    """run_observed on the decomposed engine (the native loop records rows
    on the device, across speculative batches and the rebuilds that halt
    them): each recorded row equals observe() after running to that step."""
    g = load("fcc8_jit")
    flat = E.FlatConfig(g["box"], g["ids"], g["pos"], g["vel"])
    cfg = E.EngineConfig(dt=float(g["dt"]))
    a = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]), cfg,
                         comm=InProcessComm(1), native=native)
    b = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]), cfg,
                         comm=InProcessComm(1), native=native)
    try:
        rows = a.run_observed(40, stride=3)
        rows = np.vstack([rows, a.run_observed(7, stride=3)])
        assert rows[:, 0].tolist() == list(range(3, 48, 3))
        assert a.rebuild_count() > 0
        done = 0
        for r in rows:
            b.run(int(r[0]) - done)
            done = int(r[0])
            o = b.observe()
            assert o.step == int(r[0])
            assert_rel(r[1], o.kinetic, 1e-12, f"KE at {done}")
            assert_rel(r[2], o.potential, 1e-12, f"PE at {done}")
            assert_rel(r[4], o.virial, 1e-12, f"W at {done}")
            assert_rel(r[3], o.temperature, 1e-12, f"T at {done}")
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("native", [False, True])
def test_nccl_one_rank_decomposition(native):
    """The NCCL transport itself (torchrun, one process): the single slab
    sends its boundary layers to itself through NCCL point-to-point batches,
    plus the all-reduces and all-gathers of the protocol."""
    import socket
    import subprocess
    import sys
    from pathlib import Path
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), str(root / "scripts" / "nccl_selftest.py"),
                        *(["--native"] if native else [])],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok=True" in r.stdout


def test_native_loop_with_load_aware_cuts_runs_the_rebalance_path():
    """balance = "count" in the native loop: layer histograms summed by an
    NCCL all-reduce and the C++ cut rule at every rebuild (one rank: the
    cuts stay [0, dims_z]); the run tracks the single-context engine."""
    flat = E.gen_fcc_slab(8, 0.8442, 0.7, 5)
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(flat, E.Interactions(), 0.3, cfg)
    dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(1),
                           balance="count", native=True)
    try:
        one.run(60)
        dec.run(60)
        assert dec.recuts == 0 and dec.rebuild_count() == one.rebuild_count() > 0
        assert_rel(dec.observe().potential, one.observe().potential, 1e-10, "PE")
        ids, pos, vel, f = dec.local_state()
        assert np.abs(pos - one.flatten().pos).max() < 1e-9
    finally:
        dec.close()
        one.close()
