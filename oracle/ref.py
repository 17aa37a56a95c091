"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes driver for oracle/_ref/libtaskmd_ref.so: the UNMODIFIED reference
engine (`taskmd`, /root/reference/proj/include) compiled by oracle/Makefile
through the extern "C" shim oracle/ref_shim.cpp. Only tests/, the golden
generator (oracle/make_golden.py), __graft_entry__.smoke() and bench.py's
CPU-baseline leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libtaskmd_ref.so"

STATUS_NAMES = {0: "ok", 1: "ConfigError", 2: "PhysicsError", 3: "VerifyError",
                4: "StateError", 9: "error"}


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


_lib = None


class RefOpts(C.Structure):
    """ref_shim.cpp's ref_opts: thermostat and FENE bonds."""
    _fields_ = [("thermostat", C.c_int), ("gamma", C.c_double),
                ("temperature", C.c_double), ("seed", C.c_uint64),
                ("n_bonds", C.c_int64), ("bonds", C.c_void_p), ("fene", C.c_int),
                ("fene_k", C.c_double), ("fene_rmax", C.c_double)]


def available() -> bool:
    return REF_LIB.exists()


def build() -> None:
    subprocess.run(["make", "-C", str(HERE), "ref"], check=True, capture_output=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref)")
        L = C.CDLL(str(REF_LIB))
        P = C.c_void_p
        D = C.c_double
        L.ref_create.argtypes = [C.c_int64, P, P, P, P, P, D, D, D, C.c_int, D,
                                 C.c_int, C.c_int, D, C.POINTER(P), C.c_char_p, C.c_int]
        L.ref_create_ex.argtypes = [C.c_int64, P, P, P, P, P, D, D, D, C.c_int, D,
                                    C.c_int, C.c_int, D, C.POINTER(RefOpts),
                                    C.POINTER(P), C.c_char_p, C.c_int]
        L.ref_clone.argtypes = [P, C.c_int, C.POINTER(P), C.c_char_p, C.c_int]
        L.ref_destroy.argtypes = [P]
        L.ref_destroy.restype = None
        L.ref_step.argtypes = [P, C.c_int64, C.c_char_p, C.c_int]
        L.ref_observe.argtypes = [P, P]
        L.ref_observe.restype = None
        L.ref_size.argtypes = [P]
        L.ref_size.restype = C.c_int64
        L.ref_flatten.argtypes = [P, P, P, P]
        L.ref_flatten.restype = None
        L.ref_forces.argtypes = [P, P, P]
        L.ref_forces.restype = None
        L.ref_cell_of.argtypes = [P, P, P]
        L.ref_cell_of.restype = None
        L.ref_pairs.argtypes = [P, P, C.c_int64]
        L.ref_pairs.restype = C.c_int64
        L.ref_timers.argtypes = [P, P, C.POINTER(D)]
        L.ref_timers.restype = None
        L.ref_rebuild_count.argtypes = [P]
        L.ref_rebuild_count.restype = C.c_uint64
        L.ref_grid.argtypes = [P, P, P]
        L.ref_grid.restype = None
        L.ref_lj_prepare.argtypes = [D, D, D, C.c_int, P]
        L.ref_lj_prepare.restype = None
        L.ref_lj_eval.argtypes = [D, D, D, D, C.c_int, P]
        L.ref_lj_eval.restype = None
        L.ref_build_cell_grid.argtypes = [P, D, D, P, P, C.c_char_p, C.c_int]
        L.ref_wrap_and_bin.argtypes = [C.c_int64, P, P, D, D, P, P, C.c_char_p, C.c_int]
        L.ref_cell_coords.argtypes = [P, D, D, P, P]
        L.ref_cell_coords.restype = None
        L.ref_wrap1.argtypes = [D, D]
        L.ref_wrap1.restype = D
        for nm in ("ref_counter_uniform3", "ref_counter_normal3"):
            getattr(L, nm).argtypes = [C.c_uint64] * 4 + [P]
            getattr(L, nm).restype = None
        L.ref_thermal_velocities.argtypes = [C.c_int64, P, P, D, C.c_uint64, P]
        L.ref_thermal_velocities.restype = None
        L.ref_gen_lattice.argtypes = [C.c_int64, D, D, C.c_uint64, P, P, P, P,
                                      C.c_char_p, C.c_int]
        L.ref_gen_spherical.argtypes = [D, D, D, D, D, C.c_uint64, C.c_int64, P, P, P,
                                        C.POINTER(C.c_int64), C.c_char_p, C.c_int]
        L.ref_gen_random.argtypes = [C.c_int64, D, D, D, C.c_uint64, P, P, P, P,
                                     C.c_char_p, C.c_int]
        L.ref_oracle_forces.argtypes = [C.c_int64, P, P, P, D, D, D, C.c_int, P,
                                        C.POINTER(D), C.c_char_p, C.c_int]
        L.ref_oracle_pairs.argtypes = [C.c_int64, P, P, P, D, P, C.c_int64]
        L.ref_oracle_pairs.restype = C.c_int64
        L.ref_autotune.argtypes = [C.c_int64, P, P, P, P, P, D, D, D, C.c_int, D,
                                   C.c_int, D, C.c_int, C.POINTER(C.c_int),
                                   C.c_char_p, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def _raise(rc: int, buf) -> None:
    if rc != 0:
        raise RefError(rc, buf.value.decode(errors="replace"))


class RefEngine:
    """build_domain + Engine of the reference, on the host cores."""

    def __init__(self, box, ids, pos, vel=None, mass=None, *, eps=1.0, sigma=1.0,
                 r_cut=2.5, shifted=True, r_skin=0.3, n_sub=1, workers=1, dt=0.005,
                 thermostat=None, bonds=None, fene=None):
        """thermostat: None (NVE) or (gamma, temperature, seed); bonds: (n, 2)
        ids; fene: None or (k, r_max)."""
        L = lib()
        self._ids = _c(ids, np.int64)
        self._n = int(self._ids.shape[0])
        box = _c(box, np.float64)
        pos = _c(pos, np.float64)
        vel = _c(vel, np.float64)
        mass = _c(mass, np.float64)
        err = C.create_string_buffer(512)
        h = C.c_void_p()
        o = RefOpts()
        if thermostat is not None:
            o.thermostat = 1
            o.gamma, o.temperature, o.seed = float(thermostat[0]), float(thermostat[1]), \
                int(thermostat[2])
        self._bonds = None
        if bonds is not None and len(bonds):
            self._bonds = _c(bonds, np.int64)
            o.n_bonds = int(self._bonds.shape[0])
            o.bonds = _p(self._bonds)
        if fene is not None:
            o.fene = 1
            o.fene_k, o.fene_rmax = float(fene[0]), float(fene[1])
        rc = L.ref_create_ex(self._n, _p(self._ids), _p(mass), _p(pos), _p(vel), _p(box),
                             eps, sigma, r_cut, 1 if shifted else 0, r_skin, n_sub, workers,
                             dt, C.byref(o), C.byref(h), err, 512)
        _raise(rc, err)
        self._h = h

    def clone(self, workers: int) -> "RefEngine":
        """A second reference Engine over a copy of this one's Domain with
        `workers` worker threads (ref_clone: Engine(Domain, EngineConfig),
        engine.hpp:68-77; the same subnode layout)."""
        err = C.create_string_buffer(512)
        h = C.c_void_p()
        _raise(lib().ref_clone(self._h, int(workers), C.byref(h), err, 512), err)
        c = RefEngine.__new__(RefEngine)
        c._ids, c._n, c._bonds, c._h = self._ids, self._n, getattr(self, "_bonds", None), h
        return c

    def close(self):
        if getattr(self, "_h", None):
            lib().ref_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, steps: int) -> None:
        err = C.create_string_buffer(512)
        _raise(lib().ref_step(self._h, int(steps), err, 512), err)

    def observe(self) -> dict:
        o = np.empty(4)
        lib().ref_observe(self._h, _p(o))
        return dict(step=int(o[0]), kinetic=o[1], potential=o[2], temperature=o[3])

    def flatten(self):
        n = self._n
        ids, pos, vel = np.empty(n, np.int64), np.empty((n, 3)), np.empty((n, 3))
        lib().ref_flatten(self._h, _p(ids), _p(pos), _p(vel))
        return ids, pos, vel

    def forces(self):
        n = self._n
        ids, f = np.empty(n, np.int64), np.empty((n, 3))
        lib().ref_forces(self._h, _p(ids), _p(f))
        return ids, f

    def cell_of(self):
        n = self._n
        ids, cell = np.empty(n, np.int64), np.empty(n, np.int32)
        lib().ref_cell_of(self._h, _p(ids), _p(cell))
        return ids, cell

    def pairs(self) -> np.ndarray:
        m = lib().ref_pairs(self._h, None, 0)
        out = np.empty((max(m, 1), 2), np.int64)
        lib().ref_pairs(self._h, _p(out), m)
        return out[:m]

    def timers(self):
        sec = np.empty(5)
        el = C.c_double()
        lib().ref_timers(self._h, _p(sec), C.byref(el))
        return sec, el.value

    def rebuild_count(self) -> int:
        return int(lib().ref_rebuild_count(self._h))

    def grid(self):
        dims = np.empty(3, np.int32)
        cl = np.empty(3)
        lib().ref_grid(self._h, _p(dims), _p(cl))
        return dims, cl


# ---- standalone reference functions -----------------------------------------

def lj_prepare(eps=1.0, sigma=1.0, rc=2.5, shifted=True) -> np.ndarray:
    out = np.empty(5)
    lib().ref_lj_prepare(eps, sigma, rc, 1 if shifted else 0, _p(out))
    return out


def lj_eval(r2, eps=1.0, sigma=1.0, rc=2.5, shifted=True):
    out = np.empty(2)
    lib().ref_lj_eval(r2, eps, sigma, rc, 1 if shifted else 0, _p(out))
    return float(out[0]), float(out[1])


def build_cell_grid(box, rc, skin):
    box = _c(box, np.float64)
    dims, cl = np.empty(3, np.int32), np.empty(3)
    err = C.create_string_buffer(512)
    _raise(lib().ref_build_cell_grid(_p(box), rc, skin, _p(dims), _p(cl), err, 512), err)
    return dims, cl


def wrap_and_bin(pos, box, rc, skin):
    pos = _c(pos, np.float64).reshape(-1, 3)
    box = _c(box, np.float64)
    n = pos.shape[0]
    w, cell = np.empty((n, 3)), np.empty(n, np.int32)
    err = C.create_string_buffer(512)
    _raise(lib().ref_wrap_and_bin(n, _p(pos), _p(box), rc, skin, _p(w), _p(cell), err, 512), err)
    return w, cell


def counter_normal3(seed, ctx, step, pid):
    out = np.empty(3)
    lib().ref_counter_normal3(seed, ctx, step, pid, _p(out))
    return out


def counter_uniform3(seed, ctx, step, pid):
    out = np.empty(3)
    lib().ref_counter_uniform3(seed, ctx, step, pid, _p(out))
    return out


def thermal_velocities(ids, temperature, seed, mass=None):
    ids = _c(ids, np.int64)
    vel = np.empty((ids.shape[0], 3))
    lib().ref_thermal_velocities(ids.shape[0], _p(ids), _p(_c(mass, np.float64)),
                                 temperature, seed, _p(vel))
    return vel


def gen_lattice(n, rho, temperature, seed):
    ids, pos, vel, box = np.empty(n, np.int64), np.empty((n, 3)), np.empty((n, 3)), np.empty(3)
    err = C.create_string_buffer(512)
    _raise(lib().ref_gen_lattice(n, rho, temperature, seed, _p(ids), _p(pos), _p(vel),
                                 _p(box), err, 512), err)
    return box, ids, pos, vel


def gen_random(n, rho, min_d, temperature, seed):
    ids, pos, vel, box = np.empty(n, np.int64), np.empty((n, 3)), np.empty((n, 3)), np.empty(3)
    err = C.create_string_buffer(512)
    _raise(lib().ref_gen_random(n, rho, min_d, temperature, seed, _p(ids), _p(pos), _p(vel),
                                _p(box), err, 512), err)
    return box, ids, pos, vel


def gen_spherical(box_length, frac, rho_in, alpha, temperature, seed):
    err = C.create_string_buffer(512)
    n = C.c_int64()
    _raise(lib().ref_gen_spherical(box_length, frac, rho_in, alpha, temperature, seed, 0, None,
                                   None, None, C.byref(n), err, 512), err)
    ids, pos, vel = np.empty(n.value, np.int64), np.empty((n.value, 3)), np.empty((n.value, 3))
    _raise(lib().ref_gen_spherical(box_length, frac, rho_in, alpha, temperature, seed, n.value,
                                   _p(ids), _p(pos), _p(vel), C.byref(n), err, 512), err)
    return np.full(3, float(box_length)), ids, pos, vel


def oracle_forces(box, ids, pos, eps=1.0, sigma=1.0, rc=2.5, shifted=True):
    ids = _c(ids, np.int64)
    pos = _c(pos, np.float64)
    box = _c(box, np.float64)
    n = ids.shape[0]
    f = np.empty((n, 3))
    pe = C.c_double()
    err = C.create_string_buffer(512)
    _raise(lib().ref_oracle_forces(n, _p(ids), _p(pos), _p(box), eps, sigma, rc,
                                   1 if shifted else 0, _p(f), C.byref(pe), err, 512), err)
    return f, pe.value


def oracle_pairs(box, ids, pos, r_verlet):
    ids = _c(ids, np.int64)
    pos = _c(pos, np.float64)
    box = _c(box, np.float64)
    n = ids.shape[0]
    m = lib().ref_oracle_pairs(n, _p(ids), _p(pos), _p(box), r_verlet, None, 0)
    out = np.empty((max(m, 1), 2), np.int64)
    lib().ref_oracle_pairs(n, _p(ids), _p(pos), _p(box), r_verlet, _p(out), m)
    return out[:m]


def autotune(box, ids, pos, vel, *, r_skin=0.3, workers=1, dt=0.005, probe_steps=20,
             eps=1.0, sigma=1.0, r_cut=2.5, shifted=True):
    ids = _c(ids, np.int64)
    sel = C.c_int()
    err = C.create_string_buffer(512)
    _raise(lib().ref_autotune(ids.shape[0], _p(ids), None, _p(_c(pos, np.float64)),
                              _p(_c(vel, np.float64)), _p(_c(box, np.float64)), eps, sigma,
                              r_cut, 1 if shifted else 0, r_skin, workers, dt, probe_steps,
                              C.byref(sel), err, 512), err)
    return sel.value
