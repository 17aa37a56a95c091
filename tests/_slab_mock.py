"""CPU stand-in for one slab context (test infrastructure only).

Implements the byte-level contract of the tmd_gpu_slab_* entry points
(include/tmd_gpu.h) with numpy, so the host-side protocol in
paper_2109_10876_b200/decomp.py — who sends what to whom, message sizes and
tags, ghost-layer layout, migration bookkeeping, the global rebuild test —
can be exercised over torch.distributed's gloo backend without a GPU. It does
no force computation: particles drift ballistically.
"""
from __future__ import annotations

import numpy as np
import torch

REC = np.dtype([("id", "<i8"), ("mass", "<f8"), ("x", "<f8"), ("y", "<f8"), ("z", "<f8"),
                ("vx", "<f8"), ("vy", "<f8"), ("vz", "<f8")])
assert REC.itemsize == 64


def wrap1(p, L):
    r = p - L * np.floor(p / L)
    return np.where(r >= L, r - L, r)


class MockSlab:
    def __init__(self, flat, r_verlet: float, dt: float, rank: int, nranks: int):
        self.rank, self.nranks, self.device = rank, nranks, "cpu"
        self.L = np.asarray(flat.box, np.float64)
        self.dims = np.maximum(1, np.floor(self.L / r_verlet).astype(int))
        self.cl = self.L / self.dims
        self.dxy = int(self.dims[0] * self.dims[1])
        dz = int(self.dims[2])
        self.cuts = [r * dz // nranks for r in range(nranks + 1)]
        self.z0, self.z1 = self.cuts[rank], self.cuts[rank + 1]
        self.dt = dt
        self.rec_bytes = 64
        zc = self._cell(wrap1(flat.pos, self.L))[:, 2]
        keep = (zc >= self.z0) & (zc < self.z1)
        self.id = flat.id[keep].copy()
        self.pos = flat.pos[keep].copy()
        self.vel = flat.vel[keep].copy()
        self.mass = np.ones(len(self.id)) if flat.mass is None else flat.mass[keep].copy()
        self.snap = self.pos.copy()
        self.g_lo = self.g_hi = None
        self.decisions = []

    def _cell(self, p):
        c = np.floor(p / self.cl).astype(int)
        return np.clip(c, 0, self.dims - 1)

    def _owner(self, z):
        return np.searchsorted(self.cuts[1:], z, side="right")

    def layer_counts(self, dims_z):
        assert dims_z == int(self.dims[2])
        z = self._cell(wrap1(self.pos, self.L))[:, 2] if len(self.id) else np.zeros(0, int)
        return np.bincount(z, minlength=dims_z).astype(np.int64)

    def recut(self, cuts):
        assert cuts[0] == 0 and cuts[-1] == int(self.dims[2])
        assert all(b > a for a, b in zip(cuts, cuts[1:]))
        self.cuts = [int(x) for x in cuts]
        self.z0, self.z1 = self.cuts[self.rank], self.cuts[self.rank + 1]

    # -- protocol (same names and return shapes as decomp.SlabContext)
    def info(self):
        return dict(rank=self.rank, nranks=self.nranks, z0=self.z0, zown=self.z1 - self.z0,
                    n_own=len(self.id), dxy=self.dxy, rec_bytes=64)

    def max_d2(self):
        if len(self.id) == 0:
            return 0.0
        d = self.pos - self.snap
        return float(np.max(np.sum(d * d, axis=1)))

    def decide(self, rebuild, advance):
        self.decisions.append((bool(rebuild), bool(advance)))

    def migrate_out(self):
        self.pos = wrap1(self.pos, self.L)
        dest = self._owner(self._cell(self.pos)[:, 2])
        leave = dest != self.rank
        order = np.argsort(dest[leave], kind="stable")
        idx = np.nonzero(leave)[0][order]
        rec = np.zeros(len(idx), REC)
        rec["id"], rec["mass"] = self.id[idx], self.mass[idx]
        rec["x"], rec["y"], rec["z"] = self.pos[idx].T
        rec["vx"], rec["vy"], rec["vz"] = self.vel[idx].T
        counts = np.bincount(dest[leave], minlength=self.nranks).astype(np.int64)
        stay = ~leave
        self.id, self.pos, self.vel, self.mass = (self.id[stay], self.pos[stay],
                                                  self.vel[stay], self.mass[stay])
        self._send = rec
        return counts, torch.from_numpy(rec.view(np.uint8).reshape(-1))

    def migrate_in(self, nrecv):
        self._recv = np.zeros(nrecv, REC)
        return torch.from_numpy(self._recv.view(np.uint8).reshape(-1))

    def commit(self):
        r = self._recv
        self.id = np.concatenate([self.id, r["id"]])
        self.mass = np.concatenate([self.mass, r["mass"]])
        self.pos = np.concatenate([self.pos, np.stack([r["x"], r["y"], r["z"]], 1)])
        self.vel = np.concatenate([self.vel, np.stack([r["vx"], r["vy"], r["vz"]], 1)])
        c = self._cell(self.pos)
        if len(self.id) and (c[:, 2].min() < self.z0 or c[:, 2].max() >= self.z1):
            raise AssertionError("particle outside its slab after migration")
        key = c[:, 0] + self.dims[0] * (c[:, 1] + self.dims[1] * c[:, 2])
        o = np.lexsort((self.id, key))
        self.id, self.pos, self.vel, self.mass = (self.id[o], self.pos[o], self.vel[o],
                                                  self.mass[o])
        self.cellkey = key[o]
        self.bidx = []
        self.bexp = []
        for lz in (self.z0, self.z1 - 1):
            sel = np.nonzero(self.cellkey // self.dxy == lz)[0]
            counts = np.bincount(self.cellkey[sel] % self.dxy, minlength=self.dxy)
            p4 = np.zeros((len(sel), 4))
            p4[:, :3] = self.pos[sel]
            self.bidx.append(sel)
            self.bexp.append((torch.from_numpy(counts.astype(np.int32)),
                              torch.from_numpy(self.id[sel].copy()), torch.from_numpy(p4)))
        return len(self.bidx[0]), len(self.bidx[1])

    def border(self, side, nb):
        assert nb == len(self.bidx[side])
        return self.bexp[side]

    def ghost_in(self, n_lo, n_hi):
        def alloc(n):
            return (torch.zeros(self.dxy, dtype=torch.int32), torch.zeros(n, dtype=torch.int64),
                    torch.zeros((n, 4), dtype=torch.float64))
        self.g_lo, self.g_hi = alloc(n_lo), alloc(n_hi)
        return self.g_lo, self.g_hi

    def ghosts_ready(self):
        for g in (self.g_lo, self.g_hi):
            assert int(g[0].sum()) == g[1].numel(), "ghost counts disagree with ghost size"
        self.snap = self.pos.copy()

    def kick_drift(self):
        self.pos = self.pos + self.dt * self.vel

    def forces(self, mode):
        if mode == 2:
            self.kick_drift()

    def halo(self, nb, n_lo, n_hi):
        send = []
        for s in (0, 1):
            p4 = np.zeros((len(self.bidx[s]), 4))
            p4[:, :3] = self.pos[self.bidx[s]]
            send.append(torch.from_numpy(p4))
        return send, [self.g_lo[2], self.g_hi[2]]

    def sums(self):
        ke = 0.5 * float(np.sum(self.mass[:, None] * self.vel * self.vel))
        return np.array([0.0, 0.0, ke])

    def download(self):
        n = len(self.id)
        o = np.argsort(self.id)
        return self.id[o], wrap1(self.pos[o], self.L), self.vel[o], np.zeros((n, 3))

    def pairs(self):
        return np.empty((0, 2), np.int64)

    def launch_count(self):
        return 0

    def close(self):
        pass
