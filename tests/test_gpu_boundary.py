"""The drop-in boundary's state round trip (flatten_domain, domain.hpp:193-207):
every particle's type and mass come back as created, through both download
paths (dense ids: id order assembled on the device; arbitrary ids: host
ordering) and from slab contexts; a flatten -> re-create round trip with
non-unit masses continues the reference's trajectory."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import ref
from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import load

pytestmark = pytest.mark.gpu


def mixed(ids_shift=None):
    g = load("fcc8_jit")
    n = len(g["ids"])
    ids = g["ids"].copy()
    if ids_shift is not None:  # sparse, unordered ids: the host download path
        ids = ids * 7 + 3
        perm = np.random.default_rng(ids_shift).permutation(n)
        return g, E.FlatConfig(g["box"], ids[perm], g["pos"][perm], g["vel"][perm],
                               mass=(1.0 + 0.5 * (ids[perm] % 3)),
                               type=(ids[perm] % 4).astype(np.int32))
    return g, E.FlatConfig(g["box"], ids, g["pos"], g["vel"], mass=1.0 + 0.5 * (ids % 3),
                           type=(ids % 4).astype(np.int32))


@pytest.mark.parametrize("sparse", [None, 5])
def test_flatten_returns_types_and_masses(sparse):
    g, flat = mixed(sparse)
    eng = E.Engine(flat, E.Interactions(), float(g["r_skin"]), E.EngineConfig(dt=0.005))
    try:
        eng.run(20)
        f = eng.flatten()
        o = np.argsort(flat.id)
        np.testing.assert_array_equal(f.id, flat.id[o])
        np.testing.assert_array_equal(f.type, flat.type[o])
        np.testing.assert_array_equal(f.mass, flat.mass[o])
    finally:
        eng.close()


def test_mixed_mass_round_trip_continues_the_reference_trajectory():
    """flatten -> new Engine keeps the masses (checkpoint/restart): 30 + 30
    steps equal the reference engine's 60 steps with the same masses."""
    g, flat = mixed()
    dt, rs = 0.005, float(g["r_skin"])
    r = ref.RefEngine(flat.box, flat.id, flat.pos, flat.vel, flat.mass, r_skin=rs, dt=dt)
    r.run(60)
    ids_r, pos_r, vel_r = r.flatten()
    r.close()
    a = E.Engine(flat, E.Interactions(), rs, E.EngineConfig(dt=dt))
    a.run(30)
    mid = a.flatten()
    a.close()
    b = E.Engine(mid, E.Interactions(), rs, E.EngineConfig(dt=dt))
    b.run(30)
    out = b.flatten()
    b.close()
    np.testing.assert_array_equal(out.id, ids_r)
    np.testing.assert_array_equal(out.mass, mid.mass)
    np.testing.assert_array_equal(out.type, mid.type)
    assert np.abs(out.pos - pos_r).max() < 1e-9
    assert np.abs(out.vel - vel_r).max() < 1e-9


def test_flatten_into_pinned_buffers_with_types_and_masses():
    g, flat = mixed()
    n = flat.size()
    eng = E.Engine(flat, E.Interactions(), float(g["r_skin"]), E.EngineConfig(dt=0.005))
    try:
        out = E.FlatConfig(flat.box, np.empty(n, np.int64), np.empty((n, 3)), np.empty((n, 3)),
                           mass=np.empty(n), type=np.empty(n, np.int32))
        eng.flatten(out=out)
        np.testing.assert_array_equal(out.type, flat.type)
        np.testing.assert_array_equal(out.mass, flat.mass)
        with pytest.raises(E.ConfigError):
            eng.flatten(out=E.FlatConfig(flat.box, out.id, out.pos, out.vel,
                                         type=np.empty(n + 1, np.int32)))
    finally:
        eng.close()


def test_slab_download_carries_types_and_masses():
    g, flat = mixed(3)
    dec = DecomposedEngine(flat, E.Interactions(), float(g["r_skin"]),
                           E.EngineConfig(dt=0.005), comm=InProcessComm(3), native=True)
    try:
        dec.run(40)
        L = __import__("paper_2109_10876_b200._abi", fromlist=["lib"]).lib()
        import ctypes as C
        got_t, got_m, got_i = [], [], []
        for c in dec.ctx.values():
            m = c.size()
            ids, t, ms = np.empty(m, np.int64), np.empty(m, np.int32), np.empty(m)
            assert L.tmd_gpu_download(c._h, ids.ctypes.data_as(C.c_void_p), None, None, None,
                                      t.ctypes.data_as(C.c_void_p),
                                      ms.ctypes.data_as(C.c_void_p)) == 0
            got_i.append(ids)
            got_t.append(t)
            got_m.append(ms)
        ids = np.concatenate(got_i)
        o = np.argsort(ids)
        ref_o = np.argsort(flat.id)
        np.testing.assert_array_equal(ids[o], flat.id[ref_o])
        np.testing.assert_array_equal(np.concatenate(got_t)[o], flat.type[ref_o])
        np.testing.assert_array_equal(np.concatenate(got_m)[o], flat.mass[ref_o])
    finally:
        dec.close()
