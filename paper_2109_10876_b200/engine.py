"""Python mirror of the reference engine's public API, backed by libtmd_gpu.so.

The names, argument meanings and error behaviour follow the reference
`taskmd` C++ API (/root/reference/proj/include/taskmd/):

  FlatConfig        flat_config.hpp:18-40     decomposition-free snapshot
  LjParams          potentials.hpp:21-26
  Interactions      domain.hpp:19-23          (FENE / angles: not on this path)
  EngineConfig      engine.hpp:19-26
  StepObservables   engine.hpp:43-48          (+ virial)
  SectionTimers     timers.hpp:36-62
  Engine            engine.hpp:66-290         build_domain + Engine in one ctor
  ConfigError, PhysicsError, VerifyError, StateError   errors.hpp:19-43

Every numeric call goes through the C ABI (include/tmd_gpu.h) to the sm_100a
kernels; nothing here computes physics on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi


class ConfigError(ValueError):
    """taskmd::ConfigError (errors.hpp:21-26)."""


class PhysicsError(RuntimeError):
    """taskmd::PhysicsError (errors.hpp:28-34)."""


class VerifyError(RuntimeError):
    """taskmd::VerifyError (errors.hpp:36-40)."""


class StateError(RuntimeError):
    """taskmd::StateError (errors.hpp:42-47)."""


class CudaError(RuntimeError):
    """Device or driver failure (no reference analog)."""


_ERRORS = {
    _abi.TMD_ERR_CONFIG: ConfigError,
    _abi.TMD_ERR_PHYSICS: PhysicsError,
    _abi.TMD_ERR_VERIFY: VerifyError,
    _abi.TMD_ERR_STATE: StateError,
    _abi.TMD_ERR_CUDA: CudaError,
}


def _check(rc: int, ctx) -> None:
    if rc != _abi.TMD_OK:
        msg = _abi.lib().tmd_gpu_last_error(ctx)
        raise _ERRORS.get(rc, CudaError)((msg or b"").decode(errors="replace"))


class Section(enum.IntEnum):
    """taskmd::Section (timers.hpp:11-17)."""
    kForces = 0
    kComm = 1
    kIntegrate = 2
    kNeigh = 3
    kResort = 4


SECTION_NAMES = ("Forces", "Comm", "Integrate", "Neigh", "Resort")


@dataclass
class SectionTimers:
    seconds: np.ndarray = field(default_factory=lambda: np.zeros(5))
    elapsed: float = 0.0

    def __getitem__(self, s: Section) -> float:
        return float(self.seconds[int(s)])

    def section_sum(self) -> float:
        return float(self.seconds.sum())


@dataclass
class LjParams:
    epsilon: float = 1.0
    sigma: float = 1.0
    r_cut: float = 2.5
    energy_shifted: bool = True


@dataclass
class FeneParams:
    k: float = 30.0
    r_max: float = 1.5


@dataclass
class AngleParams:
    k: float = 1.0
    theta0: float = 0.0


@dataclass
class LangevinParams:
    gamma: float = 1.0
    temperature: float = 1.0
    seed: int = 0


@dataclass
class Interactions:
    lj: LjParams = field(default_factory=LjParams)
    fene: Optional[FeneParams] = None
    angle: Optional[AngleParams] = None


@dataclass
class EngineConfig:
    dt: float = 0.005
    steps: int = 0
    thermostat: Optional[LangevinParams] = None
    n_sub: int = 1              # CPU subnode count: accepted, no GPU meaning
    worker_threads: int = 1     # CPU workers: accepted, no GPU meaning
    observable_stride: int = 100
    # GPU-only knobs
    section_timers: bool = True
    device: int = -1
    nbr_capacity: int = 0
    # kernel variant: 0 = library default (3); 1 = thread-per-particle ELL list +
    # 2x LDG.128 gathers; 2 = sector-chunked list of brick staging indices,
    # neighbour positions gathered from shared memory; 3 = sector-chunked list
    # of global slots + 256-bit LDG gathers
    variant: int = 0
    # list build of variants 2/3: 0 = by cell occupancy, 3 = warp per cell
    # (brick-staged), 5 = thread per particle (sparse cells; variant 3 only),
    # 6 = warp per cell over a culled candidate stream
    build: int = 0
    # variant-3 force kernel: threads per particle (1, 2, 4, 8; 0 = by
    # particle count, more lanes for small systems)
    lanes: int = 0
    # variant-3 force kernel: neighbour gathers in flight per thread (1, 2, 4,
    # 8; 0 = by cell occupancy: 1 for dense cells, 2 for sparse ones)
    unroll: int = 0
    # > 0: cap each LJ pair force at this magnitude (overlap warm-up of a fresh
    # polymer melt, BASELINE configs[2]); 0 = off
    force_cap: float = 0.0
    # step blocks run as CUDA graphs (section timers, when on, from device
    # phase stamps); False: every kernel launched eagerly (timers from CUDA
    # events) — bitwise the same results
    graphs: bool = True


@dataclass
class StepObservables:
    step: int = 0
    kinetic: float = 0.0
    potential: float = 0.0
    temperature: float = 0.0
    virial: float = 0.0


@dataclass
class FlatConfig:
    """Parallel arrays + box (flat_config.hpp:18-40). pos/vel are (n, 3)."""
    box: np.ndarray
    id: np.ndarray
    pos: np.ndarray
    vel: np.ndarray
    mass: Optional[np.ndarray] = None
    type: Optional[np.ndarray] = None
    bonds: Optional[np.ndarray] = None   # Topology::bonds as (n_bonds, 2) ids

    def __post_init__(self):
        self.box = np.ascontiguousarray(self.box, dtype=np.float64).reshape(3)
        self.id = np.ascontiguousarray(self.id, dtype=np.int64)
        self.pos = np.ascontiguousarray(self.pos, dtype=np.float64).reshape(-1, 3)
        if self.vel is None:
            self.vel = np.zeros_like(self.pos)
        self.vel = np.ascontiguousarray(self.vel, dtype=np.float64).reshape(-1, 3)
        if self.mass is not None:
            self.mass = np.ascontiguousarray(self.mass, dtype=np.float64)
        if self.type is not None:
            self.type = np.ascontiguousarray(self.type, dtype=np.int32)
        if self.bonds is not None:
            self.bonds = np.ascontiguousarray(self.bonds, dtype=np.int64).reshape(-1, 2)

    def size(self) -> int:
        return int(self.id.shape[0])


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def validate_engine_config(c: EngineConfig) -> None:
    """validate_engine_config (engine.hpp:28-41) + GPU-path scope checks."""
    if not np.isfinite(c.dt) or c.dt == 0.0:
        raise ConfigError("time step must be finite and nonzero")
    if c.steps < 0:
        raise ConfigError("step count must be non-negative")
    if c.n_sub < 1:
        raise ConfigError("n_sub must be at least 1")
    if c.worker_threads < 1:
        raise ConfigError("worker_threads must be at least 1")
    if c.observable_stride < 1:
        raise ConfigError("observable stride must be at least 1")
    if not np.isfinite(c.force_cap) or c.force_cap < 0.0:
        raise ConfigError("force cap must be finite and non-negative")
    if c.thermostat is not None:
        validate_langevin(c.thermostat)


def validate_langevin(p: LangevinParams) -> None:
    """validate_langevin (potentials.hpp:180-189)."""
    if not (p.gamma >= 0.0) or not np.isfinite(p.gamma):
        raise ConfigError("langevin gamma must be finite and >= 0")
    if not (p.temperature >= 0.0) or not np.isfinite(p.temperature):
        raise ConfigError("langevin temperature must be finite and >= 0")


def _system(flat: FlatConfig) -> "_abi.TmdSystem":
    sys = _abi.TmdSystem()
    sys.box[:] = list(flat.box)
    sys.n = flat.size()
    sys.id = _ptr(flat.id)
    sys.type = _ptr(flat.type)
    sys.mass = _ptr(flat.mass)
    sys.pos = _ptr(flat.pos)
    sys.vel = _ptr(flat.vel)
    if flat.bonds is not None and len(flat.bonds):
        sys.n_bonds = int(flat.bonds.shape[0])
        sys.bonds = _ptr(flat.bonds)
    return sys


def _interactions(inter: Interactions):
    if inter.angle is not None:
        raise ConfigError("angle terms are not on the GPU LJ path")
    lj = _abi.TmdLjParams(inter.lj.epsilon, inter.lj.sigma, inter.lj.r_cut,
                          1 if inter.lj.energy_shifted else 0)
    fene = None
    if inter.fene is not None:
        fene = _abi.TmdFeneParams(float(inter.fene.k), float(inter.fene.r_max))
    return lj, fene


def _engine_params(cfg: EngineConfig, r_skin: float, device: int) -> "_abi.TmdEngineParams":
    p = _abi.TmdEngineParams()
    p.dt = cfg.dt
    p.r_skin = r_skin
    p.device = device
    p.section_timers = 1 if cfg.section_timers else 0
    p.nbr_capacity = cfg.nbr_capacity
    p.reserved[0] = int(cfg.variant)
    p.reserved[3] = int(cfg.build)
    p.reserved[4] = int(cfg.lanes)
    p.reserved[1] = int(cfg.unroll)
    p.reserved[2] = 0 if cfg.graphs else 1
    p.force_cap = float(cfg.force_cap)
    if cfg.thermostat is not None:
        p.thermostat = 1
        p.gamma = float(cfg.thermostat.gamma)
        p.temperature = float(cfg.thermostat.temperature)
        p.seed = int(cfg.thermostat.seed) & 0xFFFFFFFFFFFFFFFF
    return p


class Engine:
    """build_domain (domain.hpp:134) + Engine (engine.hpp:66) on one B200.

    Engine(flat, inter, r_skin, cfg): validates, uploads, bins, builds the
    full Verlet list and runs the untimed initial force evaluation.
    """

    def __init__(self, flat: FlatConfig, inter: Interactions, r_skin: float,
                 cfg: Optional[EngineConfig] = None):
        cfg = cfg or EngineConfig()
        validate_engine_config(cfg)
        L = _abi.lib()
        self._cfg = cfg
        self._n = flat.size()
        self._keep = flat
        sys = _system(flat)
        lj, fene = _interactions(inter)
        p = _engine_params(cfg, r_skin, cfg.device)
        h = C.c_void_p()
        rc = L.tmd_gpu_create(C.byref(sys), C.byref(lj), C.byref(fene) if fene else None,
                              C.byref(p), C.byref(h))
        _check(rc, None)
        self._h = h
        self.box = flat.box.copy()
        self.r_skin = float(r_skin)
        self.inter = inter

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().tmd_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- Engine surface (engine.hpp:80-149) -----------------------------------
    def step(self) -> None:
        self.run(1)

    def run(self, steps: int) -> None:
        _check(_abi.lib().tmd_gpu_step(self._h, int(steps)), self._h)

    def run_observed(self, steps: int, stride: int = 1) -> np.ndarray:
        """run(steps) recording (step, kinetic, potential, temperature, virial)
        every `stride` steps on the device (tmd_gpu_run_observed)."""
        steps, stride = int(steps), int(stride)
        cap = steps // max(stride, 1) + 1
        rows = (_abi.TmdObservables * max(cap, 1))()
        n = C.c_int64()
        _check(_abi.lib().tmd_gpu_run_observed(self._h, steps, stride, rows, cap,
                                                C.byref(n)), self._h)
        out = np.empty((n.value, 5))
        for k in range(n.value):
            r = rows[k]
            out[k] = (r.step, r.kinetic, r.potential, r.temperature, r.virial)
        return out

    def observe(self) -> StepObservables:
        o = _abi.TmdObservables()
        _check(_abi.lib().tmd_gpu_observe(self._h, C.byref(o)), self._h)
        return StepObservables(int(o.step), o.kinetic, o.potential, o.temperature,
                               o.virial)

    def config(self) -> EngineConfig:
        return self._cfg

    def timers(self) -> SectionTimers:
        sec = np.zeros(5)
        el = C.c_double()
        _check(_abi.lib().tmd_gpu_timers(self._h, _ptr(sec), C.byref(el)), self._h)
        return SectionTimers(sec, el.value)

    def step_count(self) -> int:
        return int(_abi.lib().tmd_gpu_step_count(self._h))

    def potential_energy(self) -> float:
        return self.observe().potential

    def rebuild_count(self) -> int:
        return int(_abi.lib().tmd_gpu_rebuild_count(self._h))

    def steal_count(self) -> int:
        return 0  # no work-stealing pool on the GPU path

    def size(self) -> int:
        return self._n

    # -- state access ----------------------------------------------------------
    def flatten(self, out: Optional[FlatConfig] = None) -> FlatConfig:
        """flatten_domain (domain.hpp:193-207): sorted by id, wrapped, with each
        particle's type and mass as created.

        out: a FlatConfig whose id/pos/vel arrays (C-contiguous int64 (n,),
        float64 (n, 3)) — and type (int32 (n,)) / mass (float64 (n,)) when not
        None — receive the state in place, e.g. buffers in pinned host memory
        reused across downloads; it is returned."""
        n = self._n
        if out is None:
            ids = np.empty(n, np.int64)
            pos = np.empty((n, 3))
            vel = np.empty((n, 3))
            typ = np.empty(n, np.int32)
            mass = np.empty(n)
        else:
            ids, pos, vel, typ, mass = out.id, out.pos, out.vel, out.type, out.mass
            for a, dt, shape in ((ids, np.int64, (n,)), (pos, np.float64, (n, 3)),
                                 (vel, np.float64, (n, 3)), (typ, np.int32, (n,)),
                                 (mass, np.float64, (n,))):
                if a is None:
                    continue
                if a.dtype != dt or a.shape != shape or not a.flags.c_contiguous \
                        or not a.flags.writeable:
                    raise ConfigError("flatten(out=...): id (n,) int64, pos/vel (n, 3) "
                                      "float64, type (n,) int32, mass (n,) float64, "
                                      "C-contiguous and writeable")
        _check(_abi.lib().tmd_gpu_download(self._h, _ptr(ids), _ptr(pos), _ptr(vel), None,
                                           _ptr(typ), _ptr(mass)), self._h)
        if out is not None:
            out.box = self.box.copy()
            return out
        bonds = None if self._keep.bonds is None else self._keep.bonds.copy()
        return FlatConfig(self.box.copy(), ids, pos, vel, mass=mass, type=typ, bonds=bonds)

    def forces(self):
        """(ids, forces) of the last evaluation, sorted by id."""
        n = self._n
        ids = np.empty(n, np.int64)
        f = np.empty((n, 3))
        _check(_abi.lib().tmd_gpu_download(self._h, _ptr(ids), None, None, _ptr(f), None, None),
               self._h)
        return ids, f

    def set_velocities(self, ids: np.ndarray, vel: np.ndarray) -> None:
        ids = np.ascontiguousarray(ids, np.int64)
        vel = np.ascontiguousarray(vel, np.float64).reshape(-1, 3)
        _check(_abi.lib().tmd_gpu_set_velocities(self._h, _ptr(ids), _ptr(vel)), self._h)

    def compute_forces(self):
        """One force evaluation at the current positions: (pe, virial)."""
        pe, w = C.c_double(), C.c_double()
        _check(_abi.lib().tmd_gpu_compute_forces(self._h, C.byref(pe), C.byref(w)), self._h)
        return pe.value, w.value

    # -- PairIndexList (neighbor_list.hpp:193-268) ----------------------------------
    def build_pair_index_list(self) -> int:
        """build_pair_index_list (neighbor_list.hpp:196-247) from the current
        neighbour list: each unordered pair once. Valid until the next
        re-sort. Returns the number of pairs."""
        m = C.c_int64()
        _check(_abi.lib().tmd_gpu_build_pair_index_list(self._h, C.byref(m)), self._h)
        return m.value

    def pair_index_list(self) -> np.ndarray:
        """The built pair list as (id_i, id_j) rows, list order."""
        L = _abi.lib()
        n = C.c_size_t()
        _check(L.tmd_gpu_pair_index_list(self._h, None, 0, C.byref(n)), self._h)
        out = np.empty((max(n.value, 1), 2), np.int64)
        _check(L.tmd_gpu_pair_index_list(self._h, _ptr(out), n.value, C.byref(n)), self._h)
        return out[: n.value]

    def compute_forces_pairs(self):
        """compute_pair_forces(const PairIndexList&, ...) (neighbor_list.hpp:
        250-268): forces over the explicit pair list; returns (pe, virial)."""
        pe, w = C.c_double(), C.c_double()
        _check(_abi.lib().tmd_gpu_compute_forces_pairs(self._h, C.byref(pe), C.byref(w)),
               self._h)
        return pe.value, w.value

    def time_pair_traversal(self, reps: int) -> float:
        ms = C.c_double()
        _check(_abi.lib().tmd_gpu_time_pair_traversal(self._h, int(reps), C.byref(ms)),
               self._h)
        return ms.value

    # -- parity taps -------------------------------------------------------------
    def cell_of(self):
        n = self._n
        ids = np.empty(n, np.int64)
        cell = np.empty(n, np.int32)
        _check(_abi.lib().tmd_gpu_cell_of(self._h, _ptr(ids), _ptr(cell)), self._h)
        return ids, cell

    def pairs(self) -> np.ndarray:
        L = _abi.lib()
        n = C.c_size_t()
        _check(L.tmd_gpu_pairs(self._h, None, 0, C.byref(n)), self._h)
        out = np.empty((max(n.value, 1), 2), np.int64)
        _check(L.tmd_gpu_pairs(self._h, _ptr(out), n.value, C.byref(n)), self._h)
        return out[: n.value]

    def list_stats(self) -> dict:
        s = _abi.TmdListStats()
        _check(_abi.lib().tmd_gpu_list_stats(self._h, C.byref(s)), self._h)
        return dict(n=s.n, entries=s.entries, in_cut=s.in_cut, max_count=s.max_count,
                    capacity=s.capacity, dims=tuple(s.dims), cell_len=tuple(s.cell_len))

    def kernel_config(self) -> dict:
        """Which kernels this engine runs: force/list variant, threads per
        particle of the variant-3 force kernel, list build kind."""
        v, l, b = C.c_int(), C.c_int(), C.c_int()
        _abi.lib().tmd_gpu_kernel_config(self._h, C.byref(v), C.byref(l), C.byref(b))
        return dict(variant=v.value, lanes=l.value, build_kind=b.value)

    def launch_count(self) -> int:
        return int(_abi.lib().tmd_gpu_launch_count(self._h))

    def stream_handle(self) -> int:
        return int(_abi.lib().tmd_gpu_stream(self._h) or 0)

    def time_list_build(self, reps: int) -> float:
        ms = C.c_double()
        _check(_abi.lib().tmd_gpu_time_list_build(self._h, int(reps), C.byref(ms)), self._h)
        return ms.value

    def time_step_kernel(self, reps: int) -> float:
        """Mean ms per launch of the production step kernel (forces + fused
        velocity-Verlet epilogue); the state is restored afterwards."""
        ms = C.c_double()
        _check(_abi.lib().tmd_gpu_time_step_kernel(self._h, int(reps), C.byref(ms)),
               self._h)
        return ms.value

    def prepare_graphs(self, obs_stride: int = 0) -> None:
        """Capture the CUDA graphs the next run(s) will launch (no steps run)."""
        _check(_abi.lib().tmd_gpu_prepare_graphs(self._h, int(obs_stride)), self._h)

    def time_force_kernel(self, reps: int) -> float:
        ms = C.c_double()
        _check(_abi.lib().tmd_gpu_time_force_kernel(self._h, int(reps), C.byref(ms)),
               self._h)
        return ms.value


def release_cache() -> None:
    """Return the device blocks closed engines left in the process cache."""
    _abi.lib().tmd_gpu_release_cache()


# -- setup helpers (host-side, C ABI) --------------------------------------------

def gen_fcc(cells: int, rho: float, temperature: float, seed: int,
            offset: float = 0.25) -> FlatConfig:
    """FCC cells^3 x 4 lattice with thermal velocities."""
    L = _abi.lib()
    n = 4 * cells ** 3
    ids = np.empty(n, np.int64)
    pos = np.empty((n, 3))
    box = np.empty(3)
    rc = L.tmd_gen_fcc(int(cells), float(rho), float(offset), _ptr(ids), _ptr(pos), _ptr(box))
    if rc != 0:
        raise ConfigError("fcc generator: cells >= 1 and rho > 0 required")
    vel = np.empty((n, 3))
    L.tmd_thermal_velocities(n, _ptr(ids), None, float(temperature), int(seed), _ptr(vel))
    return FlatConfig(box, ids, pos, vel)


def gen_fcc_box(nx: int, ny: int, nz: int, rho: float, temperature: float, seed: int,
                offset: float = 0.25) -> FlatConfig:
    """FCC nx x ny x nz x 4 lattice (the weak-scaling boxes of BASELINE.json
    configs[4]: 2.048M particles per GPU, the 160^3 box at 8 GPUs). A cube is
    exactly gen_fcc; otherwise lattice constant a = cbrt(4 / rho), box =
    (nx, ny, nz) * a, ids in z, y, x, basis order, positions (i + b + offset) a,
    the same velocity draw."""
    if min(nx, ny, nz) < 1 or not rho > 0.0:
        raise ConfigError("fcc generator: cells >= 1 and rho > 0 required")
    if nx == ny == nz:
        return gen_fcc(nx, rho, temperature, seed, offset)
    a = float(np.cbrt(4.0 / rho))
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cell = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1).astype(np.float64)
    pos = ((cell[:, None, :] + basis[None, :, :] + offset) * a).reshape(-1, 3)
    n = pos.shape[0]
    ids = np.arange(n, dtype=np.int64)
    vel = np.empty((n, 3))
    _abi.lib().tmd_thermal_velocities(n, _ptr(ids), None, float(temperature), int(seed),
                                      _ptr(vel))
    return FlatConfig(np.array([nx * a, ny * a, nz * a]), ids, np.ascontiguousarray(pos), vel)


def gen_lattice(n: int, rho: float, temperature: float, seed: int) -> FlatConfig:
    """gen_lattice (generators.hpp:47-81): simple cubic, x-fastest, tail empty."""
    if n < 1:
        raise ConfigError("lattice generator needs at least 1 particle")
    if not rho > 0.0:
        raise ConfigError("density must be positive")
    if temperature < 0.0:
        raise ConfigError("temperature must be non-negative")
    ids = np.empty(n, np.int64)
    pos = np.empty((n, 3))
    vel = np.empty((n, 3))
    box = np.empty(3)
    _abi.lib().tmd_gen_lattice(int(n), float(rho), float(temperature), int(seed), _ptr(ids),
                               _ptr(pos), _ptr(vel), _ptr(box))
    return FlatConfig(box, ids, pos, vel)


def gen_spherical(box_length: float, diameter_fraction: float, rho_in: float, alpha: float,
                  temperature: float, seed: int) -> FlatConfig:
    """gen_spherical (generators.hpp:83-135): dense sphere in a dilute background."""
    if not box_length > 0.0:
        raise ConfigError("box length must be positive")
    if not diameter_fraction > 0.0 or diameter_fraction > 1.0:
        raise ConfigError("sphere diameter fraction must be in (0, 1]")
    if not rho_in > 0.0:
        raise ConfigError("density must be positive")
    if alpha < 0.0 or alpha > 1.0:
        raise ConfigError("density factor alpha must be in [0, 1]")
    if temperature < 0.0:
        raise ConfigError("temperature must be non-negative")
    L = _abi.lib()
    n = C.c_int64()
    box = np.empty(3)
    args = (float(box_length), float(diameter_fraction), float(rho_in), float(alpha),
            float(temperature), int(seed))
    L.tmd_gen_spherical(*args, None, None, None, C.byref(n), _ptr(box))
    ids = np.empty(n.value, np.int64)
    pos = np.empty((n.value, 3))
    vel = np.empty((n.value, 3))
    L.tmd_gen_spherical(*args, _ptr(ids), _ptr(pos), _ptr(vel), C.byref(n), _ptr(box))
    return FlatConfig(box, ids, pos, vel)


def gen_random(n: int, rho: float, min_distance: float, temperature: float,
               seed: int) -> FlatConfig:
    """gen_random (generators.hpp:212-258): rejection-sampled uniform positions."""
    if n < 1:
        raise ConfigError("random generator needs at least 1 particle")
    if not rho > 0.0:
        raise ConfigError("density must be positive")
    if min_distance < 0.0:
        raise ConfigError("minimum distance must be non-negative")
    if temperature < 0.0:
        raise ConfigError("temperature must be non-negative")
    ids = np.empty(n, np.int64)
    pos = np.empty((n, 3))
    vel = np.empty((n, 3))
    box = np.empty(3)
    rc = _abi.lib().tmd_gen_random(int(n), float(rho), float(min_distance), float(temperature),
                                   int(seed), _ptr(ids), _ptr(pos), _ptr(vel), _ptr(box))
    if rc != 0:
        raise ConfigError("random placement failed: density too high for the requested "
                          "minimum distance")
    return FlatConfig(box, ids, pos, vel)


def brute_force(flat: FlatConfig, inter: Interactions, r_verlet: float, device: int = -1):
    """All-pairs minimum-image LJ forces, PE and pair set on the GPU (the CLI's
    verify reference; oracle.hpp:31-160's role). Returns (forces in input
    order, pe, sorted (min id, max id) pairs)."""
    L = _abi.lib()
    sys = _system(flat)
    lj, _ = _interactions(Interactions(lj=inter.lj))
    n = flat.size()
    f = np.empty((n, 3))
    pe = C.c_double()
    npairs = C.c_size_t()
    _check(L.tmd_gpu_brute_force(C.byref(sys), C.byref(lj), float(r_verlet), int(device),
                                 _ptr(f), C.byref(pe), None, 0, C.byref(npairs)), None)
    pairs = np.empty((max(npairs.value, 1), 2), np.int64)
    _check(L.tmd_gpu_brute_force(C.byref(sys), C.byref(lj), float(r_verlet), int(device),
                                 None, None, _ptr(pairs), npairs.value, C.byref(npairs)), None)
    return f, pe.value, pairs[: npairs.value]


def gen_chains(n_chains: int, chain_len: int, rho: float = 0.85, bond: float = 0.97,
               seed: int = 1, temperature: float = 1.0) -> FlatConfig:
    """Kremer-Grest melt shape (BASELINE.json configs[2]): linear random-walk
    chains, bond length 0.97, bead density 0.85 (tmd_gen_chains), with
    thermal velocities at `temperature`. Overlapping beads need the
    force-capped warm-up (`kg_warmup`) before NVE."""
    L = _abi.lib()
    n = int(n_chains) * int(chain_len)
    ids = np.empty(n, np.int64)
    pos = np.empty((n, 3))
    bonds = np.empty((max(0, n_chains * (chain_len - 1)), 2), np.int64)
    box = np.empty(3)
    rc = L.tmd_gen_chains(int(n_chains), int(chain_len), float(rho), float(bond), int(seed),
                          _ptr(ids), _ptr(pos), _ptr(bonds), _ptr(box))
    if rc != 0:
        raise ConfigError("chain generator: n_chains, chain_len >= 1, rho, bond > 0 required")
    f = FlatConfig(box, ids, pos, None, bonds=bonds)
    thermal_velocities(f, temperature, seed)
    return f


def kg_interactions() -> Interactions:
    """Kremer-Grest: WCA (LJ cut at 2^(1/6) sigma, shifted) + FENE K=30, R0=1.5."""
    return Interactions(lj=LjParams(1.0, 1.0, 2.0 ** (1.0 / 6.0), True),
                        fene=FeneParams(30.0, 1.5))


def kg_warmup(flat: FlatConfig, r_skin: float = 0.4, caps=(5.0, 10.0, 20.0, 50.0, 100.0,
              300.0, 1000.0), steps_per_cap: int = 200, dt: float = 0.002,
              equilibrate_steps: int = 2000, equilibrate_dt: float = 0.005,
              temperature: float = 1.0, seed: int = 7, device: int = -1) -> FlatConfig:
    """Overlap-capped warm-up of a fresh melt (new; the reference has none,
    SURVEY §8c): Langevin dynamics (gamma = 1) with the LJ pair force capped at
    each value of `caps` in turn, then `equilibrate_steps` uncapped Langevin
    steps that carry off the heat the overlaps released. Returns the relaxed
    snapshot (bonds kept)."""
    cur = flat
    stages = [(float(c), steps_per_cap, dt) for c in caps]
    stages.append((0.0, equilibrate_steps, equilibrate_dt))
    for k, (cap, steps, h) in enumerate(stages):
        cfg = EngineConfig(dt=h, device=device, section_timers=False, force_cap=cap,
                           thermostat=LangevinParams(1.0, temperature, seed + k))
        with Engine(cur, kg_interactions(), r_skin, cfg) as eng:
            eng.run(steps)
            cur = eng.flatten()
    return cur


def gen_fcc_slab(cells: int, rho: float, temperature: float, seed: int,
                 n: Optional[int] = None) -> FlatConfig:
    """BASELINE.json configs[3] shape: a liquid FCC slab at density rho filling
    the middle third of a box with Lz = 3 Lx = 3 Ly (vacuum elsewhere).

    The slab is a cells^3 x 4 FCC block of side Lx = (4 cells^3 / rho)^(1/3)
    shifted to z in [Lx, 2 Lx). With `n` set, only the first n sites in id
    order are kept (2,097,152 particles is not 4 k^3, so an
    81^3-cell block is filled in id order with its tail left empty —
    gen_lattice's convention, generators.hpp:48-81)."""
    f = gen_fcc(cells, rho, temperature, seed)
    box = f.box.copy()
    pos = f.pos.copy()
    pos[:, 2] += box[2]
    box[2] *= 3.0
    ids, vel = f.id, f.vel
    if n is not None:
        if not 1 <= n <= len(ids):
            raise ConfigError(f"slab generator: 1 <= n <= {len(ids)} required")
        keep = np.argsort(ids, kind="stable")[:n]
        ids, pos = ids[keep], pos[keep]
        out = FlatConfig(box, ids, pos, None)
        thermal_velocities(out, temperature, seed)
        return out
    return FlatConfig(box, ids, pos, vel)


def thermal_velocities(flat: FlatConfig, temperature: float, seed: int) -> None:
    """gen_detail::thermal_velocities + zero_net_momentum (generators.hpp:19-39)."""
    vel = np.empty((flat.size(), 3))
    _abi.lib().tmd_thermal_velocities(flat.size(), _ptr(flat.id), _ptr(flat.mass),
                                      float(temperature), int(seed), _ptr(vel))
    flat.vel = vel


def fp64_peak_tflops(device: int = -1) -> float:
    """Measured DFMA throughput (TFLOP/s) — the FP64 roofline denominator."""
    t = C.c_double()
    _check(_abi.lib().tmd_gpu_fp64_peak(int(device), C.byref(t)), None)
    return t.value


def counter_uniform3(seed: int, ctx: int, step: int, pid: int) -> np.ndarray:
    out = np.empty(3)
    _abi.lib().tmd_counter_uniform3(seed, ctx, step, pid, _ptr(out))
    return out


def counter_normal3(seed: int, ctx: int, step: int, pid: int) -> np.ndarray:
    out = np.empty(3)
    _abi.lib().tmd_counter_normal3(seed, ctx, step, pid, _ptr(out))
    return out
