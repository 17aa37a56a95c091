"""Host-side logic of the z-slab decomposition on CPU.

paper_2109_10876_b200/decomp.py drives the slab protocol; here every slab is
the numpy stand-in tests/_slab_mock.py, and the ranks talk over
torch.distributed's gloo backend (world sizes 2 and 3, 127.0.0.1) or all live
in one process (InProcessComm). Checked after every run: each particle is
owned by exactly one rank, by the one owning its z layer at the last rebuild;
each ghost layer is its neighbour's boundary layer (same ids, same order, the
owner's current positions); every rank took the same rebuild decisions.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_10876_b200.decomp import (DecomposedEngine, InProcessComm, TorchDistComm,
                                          slab_range)
from paper_2109_10876_b200.engine import EngineConfig, FlatConfig, Interactions

from tests._slab_mock import MockSlab

R_CUT, R_SKIN, DT = 1.0, 0.3, 0.05


def _system(n=600, seed=3, box=(5.4, 4.0, 11.8)):
    rng = np.random.default_rng(seed)
    L = np.asarray(box)
    pos = rng.random((n, 3)) * L
    vel = rng.normal(size=(n, 3))
    ids = rng.permutation(10 * n)[:n].astype(np.int64)  # non-contiguous ids
    return FlatConfig(L, ids, pos, vel)


def _make(flat, comm, balance="static"):
    rv = R_CUT + R_SKIN
    inter = Interactions()
    inter.lj.r_cut = R_CUT
    return DecomposedEngine(flat, inter, R_SKIN, EngineConfig(dt=DT), comm=comm,
                            ctx_factory=lambda r: MockSlab(flat, rv, DT, r, comm.nranks),
                            balance=balance)


def _slab_system(n=900, seed=4, box=(5.4, 4.0, 23.5)):
    """Particles only in the middle third of z (config 4's liquid slab shape)."""
    rng = np.random.default_rng(seed)
    L = np.asarray(box)
    pos = rng.random((n, 3)) * L
    pos[:, 2] = L[2] / 3 + rng.random(n) * L[2] / 3
    vel = 0.5 * rng.normal(size=(n, 3))
    return FlatConfig(L, np.arange(n, dtype=np.int64) * 3 + 1, pos, vel)


def _snapshot(eng):
    """Per local rank: everything the invariant check needs (picklable)."""
    out = {}
    for r, c in eng.ctx.items():
        out[r] = dict(z0=c.z0, z1=c.z1, ids=c.id.copy(), pos=c.pos.copy(),
                      cellz=(c.cellkey // c.dxy).copy(),
                      b_ids=[c.id[c.bidx[s]].copy() for s in (0, 1)],
                      g_ids=[c.g_lo[1].numpy().copy(), c.g_hi[1].numpy().copy()],
                      g_pos=[c.g_lo[2].numpy()[:, :3].copy(), c.g_hi[2].numpy()[:, :3].copy()],
                      g_cnt=[c.g_lo[0].numpy().copy(), c.g_hi[0].numpy().copy()],
                      b_cnt=[c.bexp[s][0].numpy().copy() for s in (0, 1)],
                      decisions=list(c.decisions))
    return out


def _check(snaps, all_ids, dims_z, cuts=None):
    R = len(snaps)
    owned = np.concatenate([snaps[r]["ids"] for r in range(R)])
    assert len(owned) == len(all_ids)
    np.testing.assert_array_equal(np.sort(owned), np.sort(all_ids))
    for r in range(R):
        s = snaps[r]
        z0, z1 = (slab_range(r, R, dims_z) if cuts is None else (cuts[r], cuts[r + 1]))
        assert (s["z0"], s["z1"]) == (z0, z1)
        # membership as of the last rebuild
        assert np.all((s["cellz"] >= z0) & (s["cellz"] < z1))
        lo, hi = snaps[(r - 1) % R], snaps[(r + 1) % R]
        # lower ghost = lower neighbour's highest layer, upper = upper's lowest
        np.testing.assert_array_equal(s["g_ids"][0], lo["b_ids"][1])
        np.testing.assert_array_equal(s["g_ids"][1], hi["b_ids"][0])
        np.testing.assert_array_equal(s["g_cnt"][0], lo["b_cnt"][1])
        np.testing.assert_array_equal(s["g_cnt"][1], hi["b_cnt"][0])
        for k, nbr in ((0, lo), (1, hi)):
            where = {int(i): j for j, i in enumerate(nbr["ids"])}
            idx = np.array([where[int(i)] for i in s["g_ids"][k]], dtype=np.int64)
            if len(idx):
                np.testing.assert_array_equal(s["g_pos"][k], nbr["pos"][idx])
    dec = [snaps[r]["decisions"] for r in range(R)]
    assert all(d == dec[0] for d in dec)


def _run_and_check(eng, flat, steps_seq, gather):
    dims_z = int(np.floor(flat.box[2] / (R_CUT + R_SKIN)))
    total_rebuilds = 0
    for k in steps_seq:
        eng.run(k)
        snaps = gather(_snapshot(eng))
        _check(snaps, flat.id, dims_z, eng.cuts)
        total_rebuilds = eng.rebuild_count()
    return total_rebuilds


@pytest.mark.parametrize("R", [2, 3, 4])
def test_inprocess_protocol(R):
    flat = _system()
    eng = _make(flat, InProcessComm(R))
    rebuilds = _run_and_check(eng, flat, [0, 1, 5, 17], lambda s: s)
    assert rebuilds >= 3  # particles move ~0.05/step vs a 0.15 half-skin
    assert eng.exchanged_bytes > 0
    # kinetic energy is conserved by ballistic motion and summed over ranks
    ke = 0.5 * float(np.sum(flat.vel ** 2))
    assert eng.observe().kinetic == pytest.approx(ke, rel=1e-12)


def test_inprocess_migration_happens():
    flat = _system(seed=5)
    eng = _make(flat, InProcessComm(3))
    before = {r: set(c.id.tolist()) for r, c in eng.ctx.items()}
    eng.run(30)
    after = {r: set(c.id.tolist()) for r, c in eng.ctx.items()}
    assert any(before[r] != after[r] for r in before)


@pytest.mark.parametrize("R", [2, 3, 4])
def test_load_aware_cuts_balance_an_inhomogeneous_slab(R):
    """with the liquid in the middle third of z the static
    range rule leaves ranks idle; count-balanced cuts spread the particles."""
    flat = _slab_system()
    static = _make(flat, InProcessComm(R))
    pop_static = [len(c.id) for c in static.ctx.values()]
    eng = _make(flat, InProcessComm(R), balance="count")
    pop = [len(c.id) for c in eng.ctx.values()]
    if R > 2:  # at R = 2 the static halves already split the slab evenly
        assert eng.recuts >= 1
    assert max(pop) <= max(pop_static)
    assert max(pop) < 1.6 * len(flat.id) / R
    _run_and_check(eng, flat, [3, 20], lambda s: s)


def test_balanced_cuts_are_optimal():
    import itertools
    from paper_2109_10876_b200.decomp import balanced_cuts, max_load
    rng = np.random.default_rng(0)
    for _ in range(200):
        dz = int(rng.integers(3, 9))
        R = int(rng.integers(2, dz + 1))
        c = rng.choice([0, 0, 1, 5, 20, 100], size=dz)
        cuts = balanced_cuts(c, R)
        assert cuts[0] == 0 and cuts[-1] == dz and len(cuts) == R + 1
        assert all(b > a for a, b in zip(cuts, cuts[1:]))
        best = min(max_load(c, [0, *m, dz]) for m in itertools.combinations(range(1, dz), R - 1))
        assert max_load(c, cuts) == best


def test_single_slab_exchanges_with_itself():
    """R = 1: the slab's ghost layers are its own boundary layers (periodic
    images); every message goes to and comes from rank 0."""
    flat = _system()
    eng = _make(flat, InProcessComm(1))
    _run_and_check(eng, flat, [1, 9], lambda s: s)
    assert eng.rebuild_count() >= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, balance="static"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                init_method=f"tcp://127.0.0.1:{port}")
        flat = _system(n=500, seed=11) if balance == "static" else _slab_system()
        comm = TorchDistComm()
        eng = _make(flat, comm, balance)

        def gather(local):
            objs = [None] * world
            dist.all_gather_object(objs, local)
            merged = {}
            for o in objs:
                merged.update(o)
            return merged

        rebuilds = _run_and_check(eng, flat, [1, 4, 20], gather)
        obs = eng.observe()
        q.put((rank, "ok", rebuilds, obs.kinetic))
        dist.destroy_process_group()
    except BaseException as e:  # report, never hang the parent
        import traceback
        q.put((rank, "err", traceback.format_exc(), 0.0))


@pytest.mark.parametrize("world,balance", [(2, "static"), (3, "static"), (3, "count")])
def test_gloo_protocol(world, balance):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, balance))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r[1] != "ok"]
    assert not errs, errs[0][2]
    assert len({r[2] for r in res}) == 1 and res[0][2] >= 2
    flat = _system(n=500, seed=11) if balance == "static" else _slab_system()
    ke = 0.5 * float(np.sum(flat.vel ** 2))
    for r in res:
        assert r[3] == pytest.approx(ke, rel=1e-12)


def test_native_balanced_cuts_match_the_python_rule():
    """tmd_balanced_cuts (the native loop's choice, C++) == decomp.balanced_cuts."""
    import ctypes
    from paper_2109_10876_b200 import _abi
    from paper_2109_10876_b200.decomp import balanced_cuts
    rng = np.random.default_rng(1)
    for _ in range(300):
        dz = int(rng.integers(3, 40))
        R = int(rng.integers(1, min(dz, 9) + 1))
        c = rng.choice([0, 0, 1, 5, 20, 100, 1000], size=dz).astype(np.int64)
        out = np.zeros(R + 1, np.int32)
        rc = _abi.lib().tmd_balanced_cuts(c.ctypes.data_as(ctypes.c_void_p), dz, R,
                                          out.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        assert out.tolist() == balanced_cuts(c, R)


def test_run_observed_rows_match_observe_in_process():
    """DecomposedEngine.run_observed (Python protocol): one row per stride-th
    step, each equal to observe() after running to that step, across calls."""
    flat = _system()
    a = _make(flat, InProcessComm(2))
    b = _make(flat, InProcessComm(2))
    rows = np.vstack([a.run_observed(11, stride=4), a.run_observed(6, stride=4)])
    assert rows[:, 0].tolist() == [4, 8, 12, 16]
    done = 0
    for r in rows:
        b.run(int(r[0]) - done)
        done = int(r[0])
        o = b.observe()
        assert o.step == done
        assert np.allclose(r[1:], [o.kinetic, o.potential, o.temperature, o.virial],
                           rtol=1e-13, atol=0.0)
    assert a.step_count() == 17
