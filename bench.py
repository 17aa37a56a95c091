#!/usr/bin/env python3
"""Throughput bench for the B200 LJ short-range engine (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): LJ fluid, 1,048,576 particles on an FCC
64^3 x 4 lattice, rho 0.8442, eps = sigma = m = 1, r_cut 2.5 shifted, skin
0.3, Gaussian velocities at T = 1.0 (seed 12345, zero net momentum),
dt 0.005, FP64, NVE. A "step" is one velocity-Verlet step of the whole system
(kick, drift, on-device rebuild decision, resort + list build when triggered,
forces, kick). Synthetic input generated on the host (no dataset exists).

One JSON line on rank 0 (see DESIGN.md §Measurement for every field):
  value      device-timed particle-steps/s, inputs resident in HBM
  e2e        the same metric through the public API from host buffers:
             create (H2D) + K x (step + observe D2H) + final download
  roofline   the LJ force kernel against max(B/HBM, F/FP64)
  cpu_baseline  the reference engine (oracle/_ref) on this box's host cores

--impl reference times the reference's own CPU engine (oracle/_ref: the
unmodified taskmd headers compiled by oracle/Makefile) on the same config,
rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LJ particle-steps/sec at 1/2/4/8 B200; force-kernel % of HBM/FP64 roofline"
UNIT = "particle-steps/s"
HBM_FALLBACK_GBS = 6650.0


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, ValueError, KeyError, TypeError):  # absent or another schema
        return {"hbm_gbs": HBM_FALLBACK_GBS, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=3)
            except Exception:
                self.proc.kill()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(cells: int) -> dict:
    n = 4 * cells ** 3
    idx = {20: 0, 64: 1, 160: 4}.get(cells)
    return {"workload": f"LJ fluid FCC {cells}^3x4" +
            (f" (BASELINE.json configs[{idx}])" if idx is not None else ""),
            "n_particles": n, "rho": 0.8442, "r_cut": 2.5, "energy_shifted": True,
            "r_skin": 0.3, "temperature": 1.0, "seed": 12345, "dt": 0.005,
            "ensemble": "NVE"}


class Workload:
    """One BASELINE.json configuration: the synthetic system, its interactions
    and integrator settings, and the reference-engine kwargs for the CPU arm."""

    def __init__(self, kind: str, cells: int, weak_ranks: int = 0):
        from paper_2109_10876_b200 import engine as E
        self.kind = kind
        self.setup_s = 0.0
        t0 = time.perf_counter()
        if kind == "lj" and weak_ranks > 0:
            # configs[4] weak scaling: FCC 80^3 x 4 = 2.048M particles per GPU, the
            # box doubled along x, then y, then z (8 GPUs: the 160^3 configs[4] box)
            dims = [80, 80, 80]
            k = 0
            r = weak_ranks
            while r > 1:
                if r % 2:
                    raise SystemExit("--weak needs a power-of-two GPU count")
                dims[k % 3] *= 2
                k += 1
                r //= 2
            self.flat = E.gen_fcc_box(*dims, 0.8442, 1.0, 12345)
            self.inter, self.r_skin, self.dt = E.Interactions(), 0.3, 0.005
            self.cfg = {"workload": "LJ fluid, weak scaling at 2.048M particles per GPU "
                                    "(BASELINE.json configs[4])",
                        "fcc_cells": dims, "n_particles": self.flat.size(),
                        "n_per_gpu": self.flat.size() // weak_ranks, "rho": 0.8442,
                        "r_cut": 2.5, "energy_shifted": True, "r_skin": 0.3,
                        "temperature": 1.0, "seed": 12345, "dt": 0.005, "ensemble": "NVE"}
            self.ref_kw = {}
        elif kind == "lj":
            self.cfg = workload(cells)
            self.flat = E.gen_fcc(cells, 0.8442, 1.0, 12345)
            self.inter, self.r_skin, self.dt = E.Interactions(), 0.3, 0.005
            self.ref_kw = {}
        elif kind == "kg":
            # configs[2]: 20,000 x 200-bead KG melt (cells scales it: chains = 20000 *
            # (cells/64)^3), random-walk chains + force-capped Langevin warm-up
            chains = max(1, round(20000 * (cells / 64) ** 3))
            raw = E.gen_chains(chains, 200, 0.85, 0.97, seed=12345)
            self.flat = E.kg_warmup(raw)
            self.inter, self.r_skin, self.dt = E.kg_interactions(), 0.4, 0.01
            self.cfg = {"workload": "Kremer-Grest melt (BASELINE.json configs[2])"
                        if chains == 20000 else "Kremer-Grest melt",
                        "chains": chains, "beads_per_chain": 200,
                        "n_particles": self.flat.size(), "rho": 0.85, "bond": 0.97,
                        "lj": "WCA r_cut 2^(1/6) shifted", "fene": [30.0, 1.5],
                        "r_skin": 0.4, "dt": 0.01, "ensemble": "NVE",
                        "warmup": "force-capped Langevin (kg_warmup), untimed"}
            self.ref_kw = dict(r_cut=2.0 ** (1.0 / 6.0), bonds=self.flat.bonds,
                               fene=(30.0, 1.5))
        elif kind == "slab":
            # configs[3]: 2,097,152 particles, liquid FCC slab in the middle third of
            # Lz = 3 Lx (81^3-cell block filled in id order)
            n = 2097152 if cells == 64 else 4 * cells ** 3
            c = 81 if cells == 64 else cells
            self.flat = E.gen_fcc_slab(c, 0.8442, 0.7, 12345, n=n)
            self.inter, self.r_skin, self.dt = E.Interactions(), 0.3, 0.005
            self.cfg = {"workload": "LJ liquid-vapour slab (BASELINE.json configs[3])"
                        if n == 2097152 else "LJ liquid-vapour slab",
                        "n_particles": n, "rho_liquid": 0.8442, "box": list(self.flat.box),
                        "temperature": 0.7, "r_cut": 2.5, "r_skin": 0.3, "dt": 0.005,
                        "ensemble": "NVE"}
            self.ref_kw = {}
        else:
            raise SystemExit(f"unknown config {kind!r}")
        self.setup_s = time.perf_counter() - t0
        self.n = self.flat.size()


# ----------------------------------------------------------------------------------
def cpu_reference_run(w: "Workload", steps_wanted: int, warmup: int, budget_s: float):
    """The reference engine (oracle/_ref) on all host cores. Returns
    (particle-steps/s, cores, sample description, steps timed)."""
    from oracle import ref
    if not ref.available():
        ref.build()
    f = w.flat
    cores = os.cpu_count() or 1
    n_sub = 2 * cores
    t0 = time.perf_counter()
    r = ref.RefEngine(f.box, f.id, f.pos, f.vel, r_skin=w.r_skin, n_sub=n_sub, workers=cores,
                      dt=w.dt, **w.ref_kw)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    r.run(max(1, warmup))
    est = (time.perf_counter() - t0) / max(1, warmup)
    steps = int(max(1, min(steps_wanted, budget_s / max(est, 1e-9))))
    t0 = time.perf_counter()
    r.run(steps)
    t = time.perf_counter() - t0
    n = f.size()
    sample = (f"{n}-particle {w.kind} config, {steps} NVE steps (of {steps_wanted} requested) after "
              f"build_domain ({t_build:.1f} s, untimed) and {max(1, warmup)} warm-up steps; "
              f"reference taskmd Engine, worker_threads={cores}, n_sub={n_sub} (fixed 2x "
              f"workers), g++ -O3 -DNDEBUG")
    r.close()
    return n * steps / t, cores, sample, steps


def run_reference_arm(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        w = Workload(args.config, args.cells, ws if args.weak else 0)
        v, cores, sample, steps = cpu_reference_run(w, args.steps, args.warmup,
                                                    args.ref_budget_s)
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    cfg = dict(w.cfg)
    cfg["parallelism"] = "host threads (reference CPU engine)"
    n = w.n
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / v,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------------
def run_ours(args) -> None:
    import torch
    from paper_2109_10876_b200 import engine as E

    ws, rank, local = dist_env()
    if ws > 1 or args.decomposed:
        run_decomposed(args)
        return
    torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    w = Workload(args.config, args.cells, 1 if args.weak else 0)
    cfg_w, n, flat = w.cfg, w.n, w.flat
    ecfg = E.EngineConfig(dt=w.dt, section_timers=False, device=dev)
    eng = E.Engine(flat, w.inter, w.r_skin, ecfg)

    eng.run(args.warmup)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    rebuilds0 = eng.rebuild_count()
    with ClockSampler(dev) as clocks:
        ev0.record(stream)
        eng.run(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = eng.launch_count() - launches0
    rebuilds = eng.rebuild_count() - rebuilds0
    ms_per_step = ms / args.steps
    value = n * args.steps / (ms * 1e-3)

    # -- roofline of the force kernel -----------------------------
    st = eng.list_stats()
    kc = eng.kernel_config()
    E_ent, P_cut = st["entries"], st["in_cut"]
    t_force_ms = eng.time_force_kernel(args.force_reps)
    B = n * 52 + E_ent * 28
    F = 8 * E_ent + 20 * P_cut
    peaks = measured_peaks()
    fp64 = E.fp64_peak_tflops(dev)
    t_hbm = B / (peaks["hbm_gbs"] * 1e9)
    t_flop = F / (fp64 * 1e12)
    traffic = None
    prof = ROOT / "profiles" / "force_kernel_ncu.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            if pj.get("n_particles") == n:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if t_hbm >= t_flop:
        achieved = B / (t_force_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic}
    else:
        achieved = F / (t_force_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64, "traffic": traffic}
    # The bound the kernel actually sits on: every gathered neighbour of a
    # warp's 32 lanes lies in its own 128-B line, one L1 wavefront each, and
    # an SM's L1 processes one wavefront per clock.
    sm_count, clk_ghz = 148, (clocks_mhz := (clocks.summary().get("sm_mhz") or 1965.0)) / 1e3
    t_l1 = E_ent / (sm_count * clk_ghz * 1e9)
    roof["l1"] = {"model": "one L1 wavefront per gathered list entry, 1 wavefront/clk/SM",
                  "t_ms": 1e3 * t_l1, "frac": 1e3 * t_l1 / t_force_ms, "sm_mhz": clocks_mhz}
    roof.update({
        "kernel": "k_forces_l1" if kc["lanes"] == 1 else f"k_forces_lanes<{kc['lanes']}>",
        "algorithmic_bytes": B, "algorithmic_flops": F,
        "entries": E_ent, "in_cut_entries": P_cut, "kernel_ms": t_force_ms,
        "t_roof_ms": 1e3 * max(t_hbm, t_flop), "fp64_peak_tflops_measured": fp64,
        "peak_source": peaks["source"], "share_of_step": t_force_ms / ms_per_step,
        "definition": "B = N*52 + E*28 bytes, F = 8E + 20P (E full-list entries, P in-cut "
                      "entries); frac = T_roof / T_kernel",
    })
    eng.close()

    # -- e2e through the public API from host buffers ----------------------------------
    # The caller's arrays live in pinned host memory (allocated and filled
    # before the timed region, as a serving process keeps its staging
    # buffers); the upload and the final download are inside it.
    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    flat_in = E.FlatConfig(flat.box, pinned(flat.id), pinned(flat.pos), pinned(flat.vel),
                           mass=None if flat.mass is None else pinned(flat.mass),
                           type=flat.type, bonds=flat.bonds)
    out = E.FlatConfig(flat.box, torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(),
                       torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy(),
                       torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy())
    torch.cuda.synchronize()
    h2d = flat_in.pos.nbytes + flat_in.vel.nbytes + flat_in.id.nbytes + (
        0 if flat_in.mass is None else flat_in.mass.nbytes)
    t0 = time.perf_counter()
    e2 = E.Engine(flat_in, w.inter, w.r_skin, ecfg)
    rows = e2.run_observed(args.steps, stride=1)  # each step's observables land in host memory
    e2.flatten(out=out)
    t_e2e = time.perf_counter() - t0
    assert len(rows) == args.steps
    obs_bytes = 32 * len(rows)  # (step, KE, PE, W) per step, written by the device to host
    d2h = obs_bytes + out.pos.nbytes + out.vel.nbytes + out.id.nbytes
    e2.close()
    e2e = {"value": n * args.steps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
           "seconds": t_e2e,
           "what": "Engine(create from the caller's arrays in pinned host memory: upload, "
                   "bin, build, first forces) + run_observed(K, stride 1): every step's "
                   "(step, KE, PE, W) written by the device into mapped pinned host memory + "
                   "flatten(out=pinned buffers) download"}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, cores, sample, _ = cpu_reference_run(w, args.steps, 2, args.cpu_budget_s)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    cfg = dict(cfg_w)
    cfg.update({"parallelism": "single GPU",
                "l2": "working set > 126 MB L2 (neighbour list alone ~0.4 GB); no flush",
                "rebuilds_in_timed_region": rebuilds, "section_timers": False,
                "nbr_capacity": st["capacity"], "cell_grid": list(st["dims"])})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic", "config": cfg, "roofline": roof, "cpu_baseline": cpu,
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
    }
    print(json.dumps(line))


def run_decomposed(args) -> None:
    """N > 1: the BASELINE config on an N-slab z decomposition (decomp.py), one
    process per GPU, NCCL point-to-point halo/migration + all-reduces
    (strong scaling: the same 1M-particle system at every N; --weak: 2.048M
    particles per GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2109_10876_b200 import engine as E
    from paper_2109_10876_b200.decomp import DecomposedEngine, TorchDistComm

    ws, rank, local = dist_env()
    if args.dist_backend == "gloo":
        # pipeline check on a one-GPU box: every rank on GPU 0, buffers staged
        # through host memory (the numbers are not a scaling measurement)
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    torch.cuda.set_device(dev)
    w = Workload(args.config, args.cells, ws if args.weak else 0)  # identical on every rank
    cfg_w, n, flat = w.cfg, w.n, w.flat
    ecfg = E.EngineConfig(dt=w.dt, section_timers=False, device=dev)
    balance = "count" if args.config == "slab" else "static"

    # the C++ step loop with NCCL on the context stream (tmd_slab_nccl.cuh);
    # the Python protocol for the gloo pipeline check
    native = args.dist_backend == "nccl"

    def make():
        return DecomposedEngine(flat, w.inter, w.r_skin, ecfg, comm=TorchDistComm(),
                                device_of=lambda r: local, balance=balance, native=native)

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    eng = make()
    eng.run(args.warmup)
    ctx = eng.ctx[rank]
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = eng.launch_count()
    rebuilds0 = eng.rebuild_count()
    bytes0 = eng.exchanged_bytes
    with ClockSampler(dev) as clocks:
        ev0.record(stream)
        eng.run(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    dist.barrier()
    launches = eng.launch_count() - launches0
    rebuilds = eng.rebuild_count() - rebuilds0
    xbytes = eng.exchanged_bytes - bytes0
    sizes = eng.slab_sizes()[rank]
    eng.close()

    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    e2 = make()
    # every step's (step, KE, PE, W) recorded by the device (rank-local sums),
    # the table reduced over ranks once at the end
    rows = e2.run_observed(args.steps, stride=1)
    assert rows.shape[0] == args.steps
    ids, pos, vel, _f = e2.local_state()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    e2.close()
    h2d = flat.pos.nbytes + flat.vel.nbytes + flat.id.nbytes
    d2h = 40 * args.steps + pos.nbytes + vel.nbytes + ids.nbytes
    dist.destroy_process_group()
    if rank != 0:
        return
    cfg = dict(cfg_w)
    cfg.update({"parallelism": f"{ws} z-slabs (spatial decomposition, {args.dist_backend} "
                               f"halo + migration, {balance} cuts, "
                               f"{'native C++' if native else 'python'} step loop)",
                "l2": "working set > 126 MB L2 on every rank; no flush",
                "rebuilds_in_timed_region": rebuilds, "section_timers": False,
                "rank0_slab": sizes, "exchanged_bytes_rank0": xbytes})
    line = {
        "metric": METRIC, "value": n * args.steps / (ms * 1e-3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg, "roofline": None, "cpu_baseline": None,
        "e2e": {"value": n * args.steps / t_e2e, "unit": UNIT,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "seconds": t_e2e,
                "what": "DecomposedEngine(create, NCCL init) + run_observed(K, stride 1): every step's rank-local (step, KE, PE, W) written by the device into mapped host memory, the table summed over ranks at the end + local_state()"},
        "gpu_launches": launches * ws, "clocks": clocks.summary(),
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cells", type=int, default=64, help="FCC cells per edge (64 = 1M)")
    ap.add_argument("--config", choices=["lj", "kg", "slab"], default="lj",
                    help="lj: FCC LJ fluid (configs[0,1,4] by --cells 20/64/160); kg: "
                         "Kremer-Grest melt (configs[2]); slab: liquid-vapour slab "
                         "(configs[3])")
    ap.add_argument("--weak", action="store_true",
                    help="lj only: weak scaling at 2.048M particles per GPU (FCC 80^3 x 4 "
                         "per GPU; the box doubles along x, y, z with N; 8 GPUs = the "
                         "configs[4] 160^3 box)")
    ap.add_argument("--force-reps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=90.0)
    ap.add_argument("--decomposed", action="store_true",
                    help="run the slab decomposition even at N = 1 (under torchrun): the "
                         "single slab exchanges its halo with itself over NCCL")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="N > 1 only; gloo = pipeline check with every rank on GPU 0")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
