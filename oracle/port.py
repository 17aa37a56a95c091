"""TEST INFRASTRUCTURE ONLY — ctypes driver for oracle/_ref/libtmd_oracle.so,
the plain-C restatement of the reference LJ path (oracle/taskmd_oracle.c).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_ref" / "libtmd_oracle.so"

_lib = None


def available() -> bool:
    return PORT_LIB.exists()


def build() -> None:
    subprocess.run(["make", "-C", str(HERE), "port"], check=True, capture_output=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not PORT_LIB.exists():
            build()
        L = C.CDLL(str(PORT_LIB))
        P, D = C.c_void_p, C.c_double
        L.tmo_lj_prepare.argtypes = [D, D, D, C.c_int, P]
        L.tmo_lj_prepare.restype = None
        L.tmo_lj_eval.argtypes = [D, P, P, P]
        L.tmo_lj_eval.restype = None
        L.tmo_wrap1.argtypes = [D, D]
        L.tmo_wrap1.restype = D
        L.tmo_cell_grid.argtypes = [P, D, D, P, P]
        L.tmo_cell_of.argtypes = [P, P, P]
        for nm in ("tmo_counter_uniform3", "tmo_counter_normal3"):
            getattr(L, nm).argtypes = [C.c_uint64] * 4 + [P]
            getattr(L, nm).restype = None
        L.tmo_thermal_velocities.argtypes = [C.c_int64, P, P, D, C.c_uint64, P]
        L.tmo_thermal_velocities.restype = None
        L.tmo_gen_fcc.argtypes = [C.c_int, D, D, P, P, P]
        L.tmo_create.argtypes = [C.c_int64, P, P, P, P, P, D, D, D, C.c_int, D, D,
                                 C.POINTER(C.c_int)]
        L.tmo_create.restype = P
        L.tmo_step.argtypes = [P, C.c_int64]
        L.tmo_observe.argtypes = [P, P]
        L.tmo_observe.restype = None
        L.tmo_pairs.argtypes = [P, P, C.c_int64]
        L.tmo_pairs.restype = C.c_int64
        for nm in ("tmo_cell_of_all", "tmo_forces"):
            getattr(L, nm).argtypes = [P, P, P]
            getattr(L, nm).restype = None
        L.tmo_flatten.argtypes = [P, P, P, P]
        L.tmo_flatten.restype = None
        L.tmo_rebuild_count.argtypes = [P]
        L.tmo_rebuild_count.restype = C.c_uint64
        L.tmo_size.argtypes = [P]
        L.tmo_size.restype = C.c_int64
        L.tmo_error.argtypes = [P]
        L.tmo_error.restype = C.c_char_p
        L.tmo_destroy.argtypes = [P]
        L.tmo_destroy.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"status {code}: {msg}")
        self.code = code


class PortSystem:
    """Single-subnode restated engine with compensated sums."""

    def __init__(self, box, ids, pos, vel=None, mass=None, *, eps=1.0, sigma=1.0,
                 r_cut=2.5, shifted=True, r_skin=0.3, dt=0.005):
        L = lib()
        ids = _c(ids, np.int64)
        self._n = int(ids.shape[0])
        st = C.c_int()
        h = L.tmo_create(self._n, _p(ids), _p(_c(mass, np.float64)), _p(_c(pos, np.float64)),
                         _p(_c(vel, np.float64)), _p(_c(box, np.float64)), eps, sigma,
                         r_cut, 1 if shifted else 0, r_skin, dt, C.byref(st))
        self._h = h
        if st.value != 0:
            msg = L.tmo_error(h).decode()
            self.close()
            raise OracleError(st.value, msg)

    def close(self):
        if getattr(self, "_h", None):
            lib().tmo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, steps):
        rc = lib().tmo_step(self._h, int(steps))
        if rc:
            raise OracleError(rc, lib().tmo_error(self._h).decode())

    def observe(self) -> dict:
        o = np.empty(5)
        lib().tmo_observe(self._h, _p(o))
        return dict(step=int(o[0]), kinetic=o[1], potential=o[2], virial=o[3],
                    temperature=o[4])

    def pairs(self):
        m = lib().tmo_pairs(self._h, None, 0)
        out = np.empty((max(m, 1), 2), np.int64)
        lib().tmo_pairs(self._h, _p(out), m)
        return out[:m]

    def cell_of(self):
        ids, cell = np.empty(self._n, np.int64), np.empty(self._n, np.int32)
        lib().tmo_cell_of_all(self._h, _p(ids), _p(cell))
        return ids, cell

    def forces(self):
        ids, f = np.empty(self._n, np.int64), np.empty((self._n, 3))
        lib().tmo_forces(self._h, _p(ids), _p(f))
        return ids, f

    def flatten(self):
        ids, pos, vel = np.empty(self._n, np.int64), np.empty((self._n, 3)), np.empty((self._n, 3))
        lib().tmo_flatten(self._h, _p(ids), _p(pos), _p(vel))
        return ids, pos, vel

    def rebuild_count(self):
        return int(lib().tmo_rebuild_count(self._h))


def lj_eval(r2, eps=1.0, sigma=1.0, rc=2.5, shifted=True):
    q = np.empty(5)
    lib().tmo_lj_prepare(eps, sigma, rc, 1 if shifted else 0, _p(q))
    e, ff = C.c_double(), C.c_double()
    lib().tmo_lj_eval(r2, _p(q), C.byref(e), C.byref(ff))
    return e.value, ff.value


def lj_prepare(eps=1.0, sigma=1.0, rc=2.5, shifted=True):
    q = np.empty(5)
    lib().tmo_lj_prepare(eps, sigma, rc, 1 if shifted else 0, _p(q))
    return q


def cell_grid(box, rc, skin):
    box = _c(box, np.float64)
    dims, cl = np.empty(3, np.int32), np.empty(3)
    rc_ = lib().tmo_cell_grid(_p(box), rc, skin, _p(dims), _p(cl))
    if rc_:
        raise OracleError(1, "invalid cell grid")
    return dims, cl


def cell_of(p, dims, cell_len):
    return int(lib().tmo_cell_of(_p(_c(p, np.float64)), _p(_c(dims, np.int32)),
                                 _p(_c(cell_len, np.float64))))


def wrap1(p, L):
    return float(lib().tmo_wrap1(p, L))


def counter_normal3(seed, ctx, step, pid):
    out = np.empty(3)
    lib().tmo_counter_normal3(seed, ctx, step, pid, _p(out))
    return out


def counter_uniform3(seed, ctx, step, pid):
    out = np.empty(3)
    lib().tmo_counter_uniform3(seed, ctx, step, pid, _p(out))
    return out


def thermal_velocities(ids, temperature, seed, mass=None):
    ids = _c(ids, np.int64)
    vel = np.empty((ids.shape[0], 3))
    lib().tmo_thermal_velocities(ids.shape[0], _p(ids), _p(_c(mass, np.float64)),
                                 temperature, seed, _p(vel))
    return vel


def gen_fcc(cells, rho, offset=0.25):
    n = 4 * cells ** 3
    ids, pos, box = np.empty(n, np.int64), np.empty((n, 3)), np.empty(3)
    lib().tmo_gen_fcc(cells, rho, offset, _p(ids), _p(pos), _p(box))
    return box, ids, pos
