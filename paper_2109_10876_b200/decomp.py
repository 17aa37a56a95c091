"""Multi-GPU z-slab decomposition of the LJ hot path.

The reference decomposes the box into subnodes inside one process
(decomp.hpp:47-118 make_subnode_decomposition / make_subnode_layouts) and
keeps ghost cells current by copying positions across subnode stores
(decomp.hpp:142-200 build_ghost_plan / update_ghost_positions), re-binning
every particle at a resort (domain.hpp:54-92 distribute_records). Here one
process (or one context) per GPU owns a slab of whole z cell layers, cut with
the reference's range rule i*dims/s (decomp.hpp:87-93), plus one ghost layer
per side:

  * rebuild (the reference's resort + rebuild_all_lists, engine.hpp:195-215):
    leavers are packed into 64-byte records and sent to the rank owning their
    new z layer; each slab resorts its owned particles and exports its lowest
    and highest layer (per-cell counts, ids, positions) to the neighbour
    slabs, whose ghost layers they become; then each slab builds its list.
  * step: after the fused force + integrator kernel, each slab sends the
    current positions of its two boundary layers (32 B per particle) — the
    only per-step traffic. The full neighbour list makes the reference's
    reverse force pass (collect_ghost_forces, decomp.hpp:202-224) unnecessary.
  * the rebuild test is the reference's global one (needs_rebuild,
    neighbor_list.hpp:141-145: max displacement^2 > skin^2 / 4) as a MAX
    all-reduce of one double per step.

The byte buffers live on the device (C ABI tmd_gpu_slab_*, include/tmd_gpu.h)
and move between ranks through a `Comm`:

  * `TorchDistComm`: one process per GPU, torch.distributed (NCCL for CUDA
    buffers; the gloo backend drives the same protocol on CPU buffers in the
    host-logic tests);
  * `InProcessComm`: every rank's context in this process (device copies).
    Used to check the decomposition on one GPU; ranks never wait on one
    another inside a kernel.

Slot layout of a slab context: owned particles [0, n_own) cell-sorted
(brick-major), lower ghost layer [n_own, n_own + n_lo), upper ghost layer
after it, each ghost layer cell-sorted x-fastest exactly as the neighbour
exported it.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .engine import (ConfigError, EngineConfig, FlatConfig, Interactions, StateError,
                     StepObservables,
                     _check, _engine_params, _interactions, _ptr, _system,
                     validate_engine_config)

# message tags (both ends of a transfer agree on them; NCCL matches by order)
TAG_MIGRATE = 100
TAG_GHOST_LO = 0    # into the receiver's lower ghost layer (+0 counts, +1 ids, +2 pos)
TAG_GHOST_HI = 10   # into the receiver's upper ghost layer
TAG_HALO_LO = 20    # per-step positions into the receiver's lower ghost layer
TAG_HALO_HI = 30


def slab_range(rank: int, nranks: int, dims_z: int) -> Tuple[int, int]:
    """Owned z layers [z0, z1) of slab `rank` (decomp.hpp:87-93's rule)."""
    return rank * dims_z // nranks, (rank + 1) * dims_z // nranks


def default_cuts(nranks: int, dims_z: int) -> List[int]:
    return [r * dims_z // nranks for r in range(nranks + 1)]


def max_load(counts: Sequence[int], cuts: Sequence[int]) -> int:
    return max(int(sum(counts[cuts[r]:cuts[r + 1]])) for r in range(len(cuts) - 1))


def balanced_cuts(counts: Sequence[int], nranks: int) -> List[int]:
    """Cut planes over the z layers minimising the largest slab population,
    every slab >= 1 layer: binary search on the bound with a greedy fill, then
    the widest slabs are halved until there are `nranks` (halving never raises
    the maximum). Deterministic, so every rank computes the same cuts."""
    c = [int(x) for x in counts]
    dz = len(c)
    if nranks > dz:
        raise ConfigError(f"more ranks ({nranks}) than z cell layers ({dz})")

    def greedy(bound: int) -> List[int]:
        starts, acc = [0], 0
        for z in range(dz):
            if z > starts[-1] and acc + c[z] > bound:
                starts.append(z)
                acc = 0
            acc += c[z]
        return starts

    lo, hi = max(c), max(sum(c), max(c))
    while lo < hi:
        mid = (lo + hi) // 2
        if len(greedy(mid)) <= nranks:
            hi = mid
        else:
            lo = mid + 1
    starts = greedy(lo)
    while len(starts) < nranks:
        ends = starts[1:] + [dz]
        widths = [e - b for b, e in zip(starts, ends)]
        i = widths.index(max(widths))
        starts.insert(i + 1, starts[i] + widths[i] // 2)
    return starts + [dz]


# ---------------------------------------------------------------------------
# device buffers as tensors (zero copy)

class _DevArray:
    """__cuda_array_interface__ view of a device pointer owned by the context."""

    def __init__(self, ptr: int, shape: Tuple[int, ...], typestr: str):
        self.__cuda_array_interface__ = {
            "shape": shape, "typestr": typestr, "data": (int(ptr or 0), False),
            "version": 2, "strides": None,
        }


def _tensor(ptr, shape, typestr: str, device: int):
    import torch
    if int(np.prod(shape)) == 0:
        dt = {"<i4": torch.int32, "<i8": torch.int64, "<f8": torch.float64,
              "|u1": torch.uint8}[typestr]
        return torch.empty(shape, dtype=dt, device=f"cuda:{device}")
    return torch.as_tensor(_DevArray(ptr, tuple(shape), typestr), device=f"cuda:{device}")


class SlabContext:
    """One slab of the decomposition on one GPU (C ABI tmd_gpu_slab_*)."""

    def __init__(self, flat: FlatConfig, inter: Interactions, r_skin: float,
                 cfg: EngineConfig, rank: int, nranks: int, device: int):
        validate_engine_config(cfg)
        L = _abi.lib()
        self._keep = flat
        sys = _system(flat)
        lj, fene = _interactions(inter)
        p = _engine_params(cfg, r_skin, device)
        p.section_timers = 1 if cfg.section_timers else 0  # native loop: CUDA-event phases
        p.reserved[0] = 0
        h = C.c_void_p()
        _check(L.tmd_gpu_create_slab(C.byref(sys), C.byref(lj),
                                     C.byref(fene) if fene else None, C.byref(p),
                                     int(rank), int(nranks), C.byref(h)), None)
        self._h = h
        self.rank, self.nranks, self.device = rank, nranks, device
        self.box = flat.box.copy()
        info = self.info()
        self.dxy = info["dxy"]
        self.rec_bytes = info["rec_bytes"]

    # -- lifetime
    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().tmd_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, rc: int) -> None:
        _check(rc, self._h)

    # -- protocol
    def info(self) -> dict:
        a = np.zeros(11, np.int64)
        self._c(_abi.lib().tmd_gpu_slab_info(self._h, _ptr(a)))
        keys = ("rank", "nranks", "z0", "zown", "n_own", "n_lo", "n_hi", "dxy", "n_cap",
                "rec_bytes", "recuts")
        return dict(zip(keys, (int(v) for v in a)))

    def max_d2(self) -> float:
        m = C.c_double()
        self._c(_abi.lib().tmd_gpu_slab_max_d2(self._h, C.byref(m)))
        return m.value

    def decide(self, rebuild: bool, advance: bool) -> None:
        self._c(_abi.lib().tmd_gpu_slab_decide(self._h, int(bool(rebuild)), int(bool(advance))))

    def migrate_out(self):
        counts = np.zeros(self.nranks, np.int64)
        ptr = C.c_void_p()
        self._c(_abi.lib().tmd_gpu_slab_migrate_out(self._h, _ptr(counts), C.byref(ptr)))
        total = int(counts.sum())
        return counts, _tensor(ptr.value, (total * self.rec_bytes,), "|u1", self.device)

    def migrate_in(self, nrecv: int):
        ptr = C.c_void_p()
        self._c(_abi.lib().tmd_gpu_slab_migrate_in(self._h, int(nrecv), C.byref(ptr)))
        return _tensor(ptr.value, (int(nrecv) * self.rec_bytes,), "|u1", self.device)

    def commit(self) -> Tuple[int, int]:
        nb = np.zeros(2, np.int64)
        self._c(_abi.lib().tmd_gpu_slab_commit(self._h, _ptr(nb)))
        return int(nb[0]), int(nb[1])

    def border(self, side: int, nb: int):
        c_, i_, p_ = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._c(_abi.lib().tmd_gpu_slab_border(self._h, int(side), C.byref(c_), C.byref(i_),
                                                C.byref(p_)))
        return (_tensor(c_.value, (self.dxy,), "<i4", self.device),
                _tensor(i_.value, (nb,), "<i8", self.device),
                _tensor(p_.value, (nb, 4), "<f8", self.device))

    def ghost_in(self, n_lo: int, n_hi: int):
        lo, hi = (C.c_void_p * 3)(), (C.c_void_p * 3)()
        self._c(_abi.lib().tmd_gpu_slab_ghost_in(self._h, int(n_lo), int(n_hi), lo, hi))

        def views(a, n):
            return (_tensor(a[0], (self.dxy,), "<i4", self.device),
                    _tensor(a[1], (n,), "<i8", self.device),
                    _tensor(a[2], (n, 4), "<f8", self.device))
        return views(lo, n_lo), views(hi, n_hi)

    def ghosts_ready(self) -> None:
        self._c(_abi.lib().tmd_gpu_slab_ghosts_ready(self._h))

    def kick_drift(self) -> None:
        self._c(_abi.lib().tmd_gpu_slab_kick_drift(self._h))

    def forces(self, mode: int) -> None:
        self._c(_abi.lib().tmd_gpu_slab_forces(self._h, int(mode)))

    def halo(self, nb: Tuple[int, int], n_lo: int, n_hi: int):
        send, recv = (C.c_void_p * 2)(), (C.c_void_p * 2)()
        self._c(_abi.lib().tmd_gpu_slab_halo(self._h, send, recv))
        return ([_tensor(send[0], (nb[0], 4), "<f8", self.device),
                 _tensor(send[1], (nb[1], 4), "<f8", self.device)],
                [_tensor(recv[0], (n_lo, 4), "<f8", self.device),
                 _tensor(recv[1], (n_hi, 4), "<f8", self.device)])

    def sums(self) -> np.ndarray:
        out = np.zeros(3)
        self._c(_abi.lib().tmd_gpu_slab_sums(self._h, _ptr(out)))
        return out

    def layer_counts(self, dims_z: int) -> np.ndarray:
        out = np.zeros(dims_z, np.int64)
        self._c(_abi.lib().tmd_gpu_slab_layer_counts(self._h, _ptr(out)))
        return out

    def recut(self, cuts: Sequence[int]) -> None:
        a = np.ascontiguousarray(cuts, dtype=np.int32)
        self._c(_abi.lib().tmd_gpu_slab_recut(self._h, _ptr(a)))

    def sync(self) -> None:
        import torch
        torch.cuda.synchronize(self.device)

    # -- state taps (owned particles)
    def size(self) -> int:
        return int(_abi.lib().tmd_gpu_size(self._h))

    def download(self, out=None):
        """(ids, pos, vel, forces) of the owned particles, sorted by id. out:
        caller buffers (ids int64, pos / vel float64 (rows, 3), C-contiguous,
        rows >= the owned count — e.g. pinned staging kept across calls) that
        receive ids / positions / velocities in their first rows (forces are
        not downloaded then); views of those rows are returned."""
        n = self.size()
        if out is not None:
            ids, pos, vel = out
            for a, dt, cols in ((ids, np.int64, None), (pos, np.float64, 3),
                                (vel, np.float64, 3)):
                if a.dtype != dt or a.shape[0] < n or not a.flags.c_contiguous or \
                        (cols and a.shape[1:] != (cols,)):
                    raise ConfigError("download(out=...): ids (>=n,) int64, pos/vel (>=n, 3) "
                                      "float64, C-contiguous")
            self._c(_abi.lib().tmd_gpu_download(self._h, _ptr(ids), _ptr(pos), _ptr(vel), None,
                                                   None, None))
            return ids[:n], pos[:n], vel[:n], None
        ids = np.empty(n, np.int64)
        pos = np.empty((n, 3))
        vel = np.empty((n, 3))
        f = np.empty((n, 3))
        self._c(_abi.lib().tmd_gpu_download(self._h, _ptr(ids), _ptr(pos), _ptr(vel), _ptr(f),
                                               None, None))
        return ids, pos, vel, f

    def pairs(self) -> np.ndarray:
        L = _abi.lib()
        n = C.c_size_t()
        self._c(L.tmd_gpu_pairs(self._h, None, 0, C.byref(n)))
        out = np.empty((max(n.value, 1), 2), np.int64)
        self._c(L.tmd_gpu_pairs(self._h, _ptr(out), n.value, C.byref(n)))
        return out[: n.value]

    def launch_count(self) -> int:
        return int(_abi.lib().tmd_gpu_launch_count(self._h))

    def rebuild_count(self) -> int:
        return int(_abi.lib().tmd_gpu_rebuild_count(self._h))

    # -- the native NCCL step loop (tmd_slab_nccl.cuh)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_abi.lib().tmd_nccl_unique_id(buf), None)
        return buf.raw

    def attach_nccl(self, uid: bytes, balance_count: bool = False,
                    fused_halo: bool = True) -> None:
        buf = C.create_string_buffer(bytes(uid), 128)
        flags = (1 if balance_count else 0) | (2 if fused_halo else 0)
        self._c(_abi.lib().tmd_gpu_slab_attach_nccl(self._h, buf, flags))

    def attach_host(self, path: str, balance_count: bool = False,
                    fused_halo: bool = True) -> None:
        flags = (1 if balance_count else 0) | (2 if fused_halo else 0)
        self._c(_abi.lib().tmd_gpu_slab_attach_host(self._h, str(path).encode(), flags))

    def attach_local(self, group, balance_count: bool = False, fused_halo: bool = True) -> None:
        """Attach to an in-process group (tmd_local_group_create): the same C++
        loop with every rank's context in this process, one thread per rank."""
        flags = (1 if balance_count else 0) | (2 if fused_halo else 0)
        self._c(_abi.lib().tmd_gpu_slab_attach_local(self._h, group, flags))

    def setup_native(self) -> None:
        self._c(_abi.lib().tmd_gpu_slab_setup(self._h))

    def run_native(self, steps: int) -> None:
        self._c(_abi.lib().tmd_gpu_slab_run(self._h, int(steps)))

    def run_observed_native(self, steps: int, stride: int) -> np.ndarray:
        """run_native(steps) recording every stride-th step's rank-local
        (step, kinetic, potential, virial) sums on the device."""
        cap = int(steps) // max(int(stride), 1) + 1
        rows = (_abi.TmdObservables * cap)()
        n = C.c_int64()
        self._c(_abi.lib().tmd_gpu_slab_run_observed(self._h, int(steps), int(stride), rows,
                                                     cap, C.byref(n)))
        out = np.empty((min(n.value, cap), 4))
        for k in range(out.shape[0]):
            r = rows[k]
            out[k] = (r.step, r.kinetic, r.potential, r.virial)
        return out

    def observe_native(self, n_total: int) -> StepObservables:
        o = _abi.TmdObservables()
        self._c(_abi.lib().tmd_gpu_slab_observe(self._h, int(n_total), C.byref(o)))
        return StepObservables(int(o.step), o.kinetic, o.potential, o.temperature, o.virial)

    def stream_handle(self) -> int:
        return int(_abi.lib().tmd_gpu_stream(self._h) or 0)


# ---------------------------------------------------------------------------
# communication backends

@dataclass
class Transfer:
    """One message: `me` is the local rank, `peer` the remote one."""
    me: int
    peer: int
    tag: int
    tensor: object


class Comm:
    nranks: int
    local_ranks: Sequence[int]

    def allreduce_max(self, vals: Dict[int, float]) -> float:
        raise NotImplementedError

    def allreduce_sum(self, vals: Dict[int, np.ndarray]) -> np.ndarray:
        raise NotImplementedError

    def allgather(self, vals: Dict[int, np.ndarray]) -> np.ndarray:
        """Rows of every rank's int64 vector, stacked in rank order."""
        raise NotImplementedError

    def exchange(self, sends: List[Transfer], recvs: List[Transfer]) -> None:
        raise NotImplementedError

    def barrier(self) -> None:
        pass

    def broadcast_bytes(self, make) -> bytes:
        """make() on rank 0, its bytes on every rank."""
        raise NotImplementedError


class HostFileComm(Comm):
    """One rank per process; the native loop's collectives and messages go
    through host memory shared by mapping one file (tmd_gpu_slab_attach_host).
    Every operation synchronises the stream first, so the ranks may share one
    GPU: the multi-process path of the native loop — CUDA IPC peer buffers of
    the fused halo included — tested on a single-GPU box. Native loop only
    (the Python protocol needs a torch.distributed or in-process Comm)."""

    def __init__(self, path: str, rank: int, nranks: int):
        self.path = str(path)
        self.me = int(rank)
        self.nranks = int(nranks)
        self.local_ranks = [self.me]


class InProcessComm(Comm):
    """All ranks in this process; a transfer is a tensor copy."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.local_ranks = list(range(nranks))

    def allreduce_max(self, vals):
        return max(vals[r] for r in self.local_ranks)

    def allreduce_sum(self, vals):
        return np.sum([np.asarray(vals[r], np.float64) for r in self.local_ranks], axis=0)

    def allgather(self, vals):
        return np.stack([np.asarray(vals[r], np.int64) for r in self.local_ranks])

    def broadcast_bytes(self, make) -> bytes:
        return make()

    def exchange(self, sends, recvs):
        box: Dict[Tuple[int, int, int], object] = {}
        for s in sends:
            key = (s.me, s.peer, s.tag)
            if key in box:
                raise RuntimeError(f"duplicate message {key}")
            box[key] = s.tensor
        for r in recvs:
            src = box.pop((r.peer, r.me, r.tag))
            if src.numel() != r.tensor.numel():
                raise RuntimeError(f"message size mismatch {r.peer}->{r.me} tag {r.tag}: "
                                   f"{src.numel()} vs {r.tensor.numel()}")
            if src.numel():
                r.tensor.copy_(src)
        if box:
            raise RuntimeError(f"unmatched messages: {sorted(box)}")
        _sync_all()


def _sync_all() -> None:
    import torch
    if torch.cuda.is_available():
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)


class TorchDistComm(Comm):
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU).

    Point-to-point messages of one phase are posted as one batch, sends
    ordered by (peer, tag) and receives by (peer, tag), so both ends of each
    rank pair post matching messages in the same order (NCCL matches by
    order, gloo by tag)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nranks = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        self.local_ranks = [self.me]
        self.backend = dist.get_backend(group)

    def _dev(self):
        import torch
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def allreduce_max(self, vals):
        import torch
        t = torch.tensor([float(vals[self.me])], dtype=torch.float64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allreduce_sum(self, vals):
        import torch
        t = torch.tensor(np.asarray(vals[self.me], np.float64), device=self._dev())
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def allgather(self, vals):
        import torch
        v = torch.tensor(np.asarray(vals[self.me], np.int64), device=self._dev())
        out = [torch.empty_like(v) for _ in range(self.nranks)]
        self.dist.all_gather(out, v, group=self.group)
        return torch.stack(out).cpu().numpy()

    def exchange(self, sends, recvs):
        import torch
        # gloo moves host memory only: device buffers are staged through host
        # copies (used by the one-GPU multi-process test; NCCL sends in place)
        stage = self.backend != "nccl"

        def host(t):
            return t.cpu() if (stage and t.is_cuda) else t
        ops, back = [], []
        P2POp = self.dist.P2POp
        for s in sorted(sends, key=lambda t: (t.peer, t.tag)):
            if s.tensor.numel():
                ops.append(P2POp(self.dist.isend, host(s.tensor).reshape(-1), s.peer,
                                 self.group, s.tag))
        for r in sorted(recvs, key=lambda t: (t.peer, t.tag)):
            if r.tensor.numel():
                buf = r.tensor
                if stage and buf.is_cuda:
                    buf = torch.empty(buf.shape, dtype=buf.dtype)
                    back.append((r.tensor, buf))
                ops.append(P2POp(self.dist.irecv, buf.reshape(-1), r.peer, self.group,
                                 r.tag))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for dev_t, host_t in back:
            dev_t.copy_(host_t)
        if self.backend == "nccl" or back:
            torch.cuda.synchronize()

    def barrier(self):
        self.dist.barrier(group=self.group)

    def broadcast_bytes(self, make) -> bytes:
        obj = [make() if self.me == 0 else None]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        return obj[0]


# ---------------------------------------------------------------------------
# the decomposed engine

class DecomposedEngine:
    """Engine (engine.hpp:66-290) over a z-slab decomposition.

    Every rank constructs it with the same whole system (FlatConfig) and
    keeps its slab; `ctx_factory(rank)` creates the per-rank context (a
    `SlabContext` on GPU `device_of(rank)` by default). With `InProcessComm`
    one process holds every rank's context.
    """

    def __init__(self, flat: FlatConfig, inter: Interactions, r_skin: float,
                 cfg: Optional[EngineConfig] = None, comm: Optional[Comm] = None,
                 device_of=None, ctx_factory=None, balance: str = "static",
                 rebalance_tolerance: float = 1.05, native: bool = False,
                 halo: str = "fused"):
        cfg = cfg or EngineConfig()
        validate_engine_config(cfg)
        if comm is None:
            raise ConfigError("DecomposedEngine needs a Comm (InProcessComm / TorchDistComm)")
        if isinstance(comm, HostFileComm) and not native:
            raise ConfigError("HostFileComm drives the native loop only (native=True)")
        self.comm = comm
        self.cfg = cfg
        self.n_total = flat.size()
        self.box = flat.box.copy()
        self.r_skin = float(r_skin)
        self.thr = 0.25 * self.r_skin * self.r_skin  # needs_rebuild (nl.hpp:143)
        R = comm.nranks
        if device_of is None:
            device_of = (lambda r: 0) if isinstance(comm, InProcessComm) else (lambda r: r)
        if ctx_factory is None:
            def ctx_factory(r):
                return SlabContext(flat, inter, r_skin, cfg, r, R, device_of(r))
        if balance not in ("static", "count"):
            raise ConfigError(f"unknown balance mode {balance!r} (static | count)")
        self.balance = balance
        self.rebalance_tolerance = float(rebalance_tolerance)
        rv = inter.lj.r_cut + self.r_skin
        self.dims_z = max(1, int(np.floor(float(flat.box[2]) / rv)))
        self.cuts = default_cuts(R, self.dims_z)
        self.recuts = 0
        self.ctx = {r: ctx_factory(r) for r in comm.local_ranks}
        self.nb: Dict[int, Tuple[int, int]] = {}
        self.ng: Dict[int, Tuple[int, int]] = {}
        self.steps = 0
        self.rebuilds = 0
        self.exchanged_bytes = 0
        self.native = bool(native)
        if self.native:
            # the whole protocol in C++ (tmd_slab_nccl.cuh) with its collectives
            # on each context's stream: NCCL with one slab per process, or the
            # in-process transport with every rank's context here, driven by
            # one thread per rank
            if halo not in ("fused", "nccl"):
                raise ConfigError(f"unknown halo mode {halo!r} (fused | nccl)")
            kw = dict(balance_count=balance == "count", fused_halo=halo == "fused")
            if isinstance(comm, InProcessComm):
                L = _abi.lib()
                g = C.c_void_p()
                _check(L.tmd_local_group_create(int(R), C.byref(g)), None)
                try:
                    for c in self.ctx.values():
                        c.attach_local(g, **kw)
                finally:
                    L.tmd_local_group_destroy(g)
            elif isinstance(comm, HostFileComm):
                (c,) = self.ctx.values()
                c.attach_host(comm.path, **kw)
            else:
                if len(self.ctx) != 1:
                    raise ConfigError("the native NCCL loop runs one slab per process")
                (c,) = self.ctx.values()
                c.attach_nccl(comm.broadcast_bytes(SlabContext.nccl_unique_id), **kw)
            self._par(lambda c: c.setup_native())
            self.recuts = next(iter(self.ctx.values())).info()["recuts"]
            return
        self._rebuild(advance=False)
        for c in self.ctx.values():
            c.forces(0)

    def close(self) -> None:
        for c in self.ctx.values():
            c.close()

    def _par(self, fn) -> Dict[int, object]:
        """fn(ctx) for every local rank, concurrently (one thread per rank: the
        native loop's collectives rendezvous across them). The first error
        that is not a peer's "a peer rank failed" is raised."""
        items = list(self.ctx.items())
        if len(items) == 1:
            r, c = items[0]
            return {r: fn(c)}
        out: Dict[int, object] = {}
        errs: Dict[int, BaseException] = {}

        def work(r, c):
            try:
                out[r] = fn(c)
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errs[r] = e
        ts = [threading.Thread(target=work, args=rc, daemon=True) for rc in items]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            own = [e for e in errs.values() if "a peer rank failed" not in str(e)]
            raise (own or list(errs.values()))[0]
        return out

    # -- protocol phases ---------------------------------------------------------
    def _rebuild(self, advance: bool) -> None:
        R = self.comm.nranks
        for c in self.ctx.values():
            c.decide(True, advance)
        if self.balance == "count":
            self._rebalance()
        # 1. migration of leavers to the owners of their z layers
        out = {r: c.migrate_out() for r, c in self.ctx.items()}
        M = self.comm.allgather({r: out[r][0] for r in self.ctx})  # M[src, dst]
        sends, recvs = [], []
        for r, c in self.ctx.items():
            counts, buf = out[r]
            off = np.concatenate([[0], np.cumsum(counts)]) * c.rec_bytes
            for d in range(R):
                if counts[d]:
                    sends.append(Transfer(r, d, TAG_MIGRATE, buf[off[d]:off[d + 1]]))
            col = M[:, r]
            rbuf = c.migrate_in(int(col.sum()))
            roff = np.concatenate([[0], np.cumsum(col)]) * c.rec_bytes
            for s in range(R):
                if col[s]:
                    recvs.append(Transfer(r, s, TAG_MIGRATE, rbuf[roff[s]:roff[s + 1]]))
            self.exchanged_bytes += int(counts.sum()) * c.rec_bytes
        self.comm.exchange(sends, recvs)
        # 2. resort + boundary-layer export
        for r, c in self.ctx.items():
            self.nb[r] = c.commit()
        NB = self.comm.allgather({r: np.asarray(self.nb[r], np.int64) for r in self.ctx})
        sends, recvs = [], []
        for r, c in self.ctx.items():
            lo_rank, hi_rank = (r - 1) % R, (r + 1) % R
            n_lo, n_hi = int(NB[lo_rank, 1]), int(NB[hi_rank, 0])
            self.ng[r] = (n_lo, n_hi)
            lo, hi = c.ghost_in(n_lo, n_hi)
            b0 = c.border(0, self.nb[r][0])  # my lowest layer -> lower neighbour's upper ghost
            b1 = c.border(1, self.nb[r][1])  # my highest layer -> upper neighbour's lower ghost
            for k in range(3):
                sends.append(Transfer(r, lo_rank, TAG_GHOST_HI + k, b0[k]))
                sends.append(Transfer(r, hi_rank, TAG_GHOST_LO + k, b1[k]))
                recvs.append(Transfer(r, lo_rank, TAG_GHOST_LO + k, lo[k]))
                recvs.append(Transfer(r, hi_rank, TAG_GHOST_HI + k, hi[k]))
            self.exchanged_bytes += (self.nb[r][0] + self.nb[r][1]) * 40 + 8 * c.dxy
        self.comm.exchange(sends, recvs)
        # 3. cell ranges of the ghost layers + list build
        for c in self.ctx.values():
            c.ghosts_ready()

    def _rebalance(self) -> None:
        """Load-aware cut planes: particle counts per z layer
        summed over ranks; re-cut when the current cuts' largest slab exceeds
        the balanced optimum by more than the tolerance."""
        hist = self.comm.allreduce_sum(
            {r: c.layer_counts(self.dims_z).astype(np.float64) for r, c in self.ctx.items()})
        hist = np.rint(hist).astype(np.int64)
        best = balanced_cuts(hist, self.comm.nranks)
        if max_load(hist, self.cuts) > self.rebalance_tolerance * max_load(hist, best):
            for c in self.ctx.values():
                c.recut(best)
            self.cuts = best
            self.recuts += 1

    def _halo(self) -> None:
        R = self.comm.nranks
        sends, recvs = [], []
        for r, c in self.ctx.items():
            send, recv = c.halo(self.nb[r], *self.ng[r])
            lo_rank, hi_rank = (r - 1) % R, (r + 1) % R
            sends.append(Transfer(r, lo_rank, TAG_HALO_HI, send[0]))
            sends.append(Transfer(r, hi_rank, TAG_HALO_LO, send[1]))
            recvs.append(Transfer(r, lo_rank, TAG_HALO_LO, recv[0]))
            recvs.append(Transfer(r, hi_rank, TAG_HALO_HI, recv[1]))
            self.exchanged_bytes += 32 * (self.nb[r][0] + self.nb[r][1])
        self.comm.exchange(sends, recvs)

    # -- Engine surface ------------------------------------------------------------
    def run(self, steps: int) -> None:
        """steps x velocity Verlet (engine.hpp:80-110's loop): kick + drift, then per
        step the global rebuild test, (rebuild,) forces + closing half-kick fused
        with the next opening half-kick + drift, halo exchange."""
        if steps < 0:
            raise ConfigError("step count must be non-negative")
        if steps == 0:
            return
        if self.native:
            self._par(lambda c: c.run_native(steps))
            self.steps += steps
            c = next(iter(self.ctx.values()))
            self.rebuilds = c.rebuild_count()
            self.recuts = c.info()["recuts"]
            return
        for c in self.ctx.values():
            c.kick_drift()
        self._halo()
        for s in range(steps):
            m = self.comm.allreduce_max({r: c.max_d2() for r, c in self.ctx.items()})
            if m > self.thr:
                self._rebuild(advance=True)
                self.rebuilds += 1
            else:
                for c in self.ctx.values():
                    c.decide(False, True)
            last = s + 1 == steps
            for c in self.ctx.values():
                c.forces(1 if last else 2)
            if not last:
                self._halo()
        for c in self.ctx.values():
            c.max_d2()  # drains the stream and raises pending physics errors
        self.steps += steps

    def step(self) -> None:
        self.run(1)

    def run_observed(self, steps: int, stride: int = 1) -> np.ndarray:
        """run(steps) recording (step, kinetic, potential, temperature, virial)
        of every stride-th step, summed over ranks (Engine.run_observed's rows).
        The native loop records rank-local sums on the device as the steps
        run and reduces the whole table once at the end; the Python protocol
        observes after each recorded step."""
        steps, stride = int(steps), int(stride)
        if stride < 1:
            raise ConfigError("observable stride must be at least 1")
        if self.native:
            s0 = self.steps
            local = self._par(lambda c: c.run_observed_native(steps, stride))
            self.steps += steps
            c = next(iter(self.ctx.values()))
            self.rebuilds = c.rebuild_count()
            self.recuts = c.info()["recuts"]
            want = np.arange(s0 + stride - s0 % stride, s0 + steps + 1, stride)
            for rows in local.values():
                if rows.shape[0] != want.size or not np.array_equal(rows[:, 0], want):
                    raise StateError("native loop recorded an unexpected set of steps")
            tot = self.comm.allreduce_sum(
                {r: rows[:, 1:4].ravel() for r, rows in local.items()}).reshape(-1, 3)
            ke, pe, w = tot[:, 0], tot[:, 1], tot[:, 2]
            return np.column_stack([want.astype(np.float64), ke, pe,
                                    2.0 * ke / (3.0 * self.n_total), w])
        rows = []
        done = 0
        while done < steps:
            k = stride - (self.steps % stride)
            k = min(k, steps - done)
            self.run(k)
            done += k
            if self.steps % stride == 0:
                o = self.observe()
                rows.append((o.step, o.kinetic, o.potential, o.temperature, o.virial))
        return np.array(rows, dtype=np.float64).reshape(-1, 5)

    def observe(self) -> StepObservables:
        if self.native:
            obs = self._par(lambda c: c.observe_native(self.n_total))
            o = obs[min(obs)]
            return StepObservables(self.steps, o.kinetic, o.potential, o.temperature, o.virial)
        tot = self.comm.allreduce_sum({r: c.sums() for r, c in self.ctx.items()})
        pe, w, ke = (float(v) for v in tot)
        return StepObservables(self.steps, ke, pe, 2.0 * ke / (3.0 * self.n_total), w)

    def timers(self):
        """SectionTimers of the native loop (engine.hpp:145): those of this
        process's slowest rank (largest elapsed; each rank times its own
        stream with CUDA events, a collective's wait for its peers included
        in Comm). The Python protocol fills none."""
        from .engine import SectionTimers
        best = SectionTimers(np.zeros(5), 0.0)
        for c in self.ctx.values():
            s5 = np.zeros(5)
            e = C.c_double()
            _check(_abi.lib().tmd_gpu_timers(c._h, _ptr(s5), C.byref(e)), c._h)
            if e.value >= best.elapsed:
                best = SectionTimers(s5, e.value)
        return best

    def step_count(self) -> int:
        return self.steps

    def rebuild_count(self) -> int:
        return self.rebuilds

    def size(self) -> int:
        return self.n_total

    # -- local state (this process's ranks) ---------------------------------------
    def local_state(self, out=None):
        """(ids, pos, vel, forces) of the particles this process's ranks own,
        sorted by id. out (one rank per process): caller buffers as in
        SlabContext.download, filled in place (forces None)."""
        if out is not None and len(self.ctx) == 1:
            return next(iter(self.ctx.values())).download(out)
        parts = [c.download() for c in self.ctx.values()]
        ids = np.concatenate([p[0] for p in parts])
        o = np.argsort(ids, kind="stable")
        return tuple(np.concatenate([p[k] for p in parts])[o] for k in range(4))

    def local_pairs(self) -> np.ndarray:
        ps = [c.pairs() for c in self.ctx.values()]
        p = np.concatenate(ps) if ps else np.empty((0, 2), np.int64)
        if len(p):
            p = p[np.lexsort((p[:, 1], p[:, 0]))]
        return p

    def slab_sizes(self) -> Dict[int, dict]:
        return {r: c.info() for r, c in self.ctx.items()}

    def launch_count(self) -> int:
        return sum(c.launch_count() for c in self.ctx.values())
