#!/usr/bin/env python3
"""Throughput bench for the B200 LJ short-range engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config lj|kg|slab] [--cells C] [--weak]

Default workload (BASELINE.json configs[4], the configuration the north-star's
scaling target is stated on, and one that fits one GPU): LJ fluid, 16,384,000
particles on an FCC 160^3 x 4 lattice, rho 0.8442, eps = sigma = m = 1, r_cut
2.5 shifted, skin 0.3, Gaussian velocities at T = 1.0 (seed 12345, zero net
momentum), dt 0.005, FP64, NVE; the same system at every N (strong scaling).
`--cells 64` is configs[1] (1M), `--cells 20` configs[0] (32K), `--config kg`
configs[2], `--config slab` configs[3], `--weak` configs[4]'s weak series
(2.048M particles per GPU). A "step" is one velocity-Verlet step of the whole
system (kick, drift, on-device rebuild decision, resort + list build when
triggered, forces, kick). Synthetic inputs (no dataset exists).

`--gpus N` with N > 1 and no torchrun environment re-launches this script
under `python -m torch.distributed.run --nproc-per-node N`; under torchrun the
world size must equal N. Each rank drives one GPU's slab of the z-slab
decomposition (the native C++ step loop over NCCL).

One JSON line on rank 0:
  value      device-timed particle-steps/s (CUDA events on the engine's
             stream, inputs resident in HBM, max over ranks)
  e2e        the same metric through the public API from host buffers:
             create (H2D) + K x (step + observables D2H) + final download
  roofline   the production step kernel (forces + fused integrator) against
             max(B/HBM, F/FP64) (BASELINE.md §4 / SURVEY §8d), plus the
             L1-wavefront model and ncu's DRAM / L1TEX figures
  cpu_baseline  the reference engine (oracle/_ref) on this box's host cores:
             all-core rate, its five SectionTimers, and a 1-thread rate

--impl reference times the reference's own CPU engine (oracle/_ref: the
unmodified taskmd headers compiled by oracle/Makefile) on the same config
with every host core, rank 0 only. Its inputs are generated without this
repo's library (numpy + the reference's own velocity draw), so that arm
never maps libtmd_gpu.so.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LJ particle-steps/sec at 1/2/4/8 B200; force-kernel % of HBM/FP64 roofline"
UNIT = "particle-steps/s"
HBM_FALLBACK_GBS = 6650.0
L2_BYTES = 126 * 2 ** 20
RHO, SEED = 0.8442, 12345


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


# ----------------------------------------------------------------------------------
# launch: one process per GPU

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return int(s.getsockname()[1])


def relaunch_if_needed(args, argv) -> None:
    """`--gpus N` means N ranks: without a torchrun environment, N > 1 re-runs
    this script under torch.distributed.run (one process per GPU); under
    torchrun the world size must be N."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                   f"--master-port={_free_port()}", str(Path(__file__).resolve()), *argv]
            sys.stdout.flush()
            sys.exit(subprocess.call(cmd))
        return
    if int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started "
                         f"WORLD_SIZE={ws_env} ranks; pass --gpus {ws_env}")


# ----------------------------------------------------------------------------------
# workload description (identical in both arms) and synthetic inputs

def config_index(kind: str, cells: int, weak: bool):
    if kind == "lj":
        if weak:
            return 4
        return {20: 0, 64: 1, 160: 4}.get(cells)
    if kind == "kg":
        return 2 if cells == 64 else None
    if kind == "slab":
        return 3 if cells == 64 else None
    return None


def weak_dims(ranks: int):
    """configs[4] weak scaling: FCC 80^3 x 4 = 2.048M particles per GPU, the box
    doubled along x, then y, then z (8 GPUs: the 160^3 configs[4] box)."""
    dims = [80, 80, 80]
    k, r = 0, ranks
    while r > 1:
        if r % 2:
            raise SystemExit("--weak needs a power-of-two GPU count")
        dims[k % 3] *= 2
        k += 1
        r //= 2
    return dims


def workload_config(kind: str, cells: int, weak: bool, ranks: int) -> dict:
    """The `config` object of the JSON line — a pure function of the command
    line, so both arms print the same dict."""
    idx = config_index(kind, cells, weak)
    tag = f" (BASELINE.json configs[{idx}])" if idx is not None else ""
    if kind == "lj" and weak:
        dims = weak_dims(ranks)
        n = 4 * dims[0] * dims[1] * dims[2]
        return {"workload": "LJ fluid, weak scaling at 2.048M particles per GPU" + tag,
                "fcc_cells": dims, "n_particles": n, "n_per_gpu": n // ranks, "rho": RHO,
                "r_cut": 2.5, "energy_shifted": True, "r_skin": 0.3, "temperature": 1.0,
                "seed": SEED, "dt": 0.005, "ensemble": "NVE"}
    if kind == "lj":
        return {"workload": f"LJ fluid FCC {cells}^3x4" + tag, "n_particles": 4 * cells ** 3,
                "rho": RHO, "r_cut": 2.5, "energy_shifted": True, "r_skin": 0.3,
                "temperature": 1.0, "seed": SEED, "dt": 0.005, "ensemble": "NVE"}
    if kind == "kg":
        chains = max(1, round(20000 * (cells / 64) ** 3))
        return {"workload": "Kremer-Grest melt" + tag, "chains": chains,
                "beads_per_chain": 200, "n_particles": chains * 200, "rho": 0.85,
                "bond": 0.97, "lj": "WCA r_cut 2^(1/6) shifted", "fene": [30.0, 1.5],
                "r_skin": 0.4, "dt": 0.01, "ensemble": "NVE",
                "warmup": "force-capped Langevin (kg_warmup), untimed"}
    if kind == "slab":
        n = 2097152 if cells == 64 else 4 * cells ** 3
        return {"workload": "LJ liquid-vapour slab" + tag, "n_particles": n,
                "rho_liquid": RHO, "box_lz_over_lx": 3, "temperature": 0.7, "r_cut": 2.5,
                "r_skin": 0.3, "dt": 0.005, "ensemble": "NVE"}
    raise SystemExit(f"unknown config {kind!r}")


def fcc_numpy(nx: int, ny: int, nz: int, offset: float = 0.25):
    """The FCC lattice of SURVEY §8(d) in numpy (no repo library): ids in z, y,
    x, basis order, positions (i + b + offset) a; a cube uses a = L / cells
    with L = cbrt(n / rho) (tmd_gen_fcc's rounding), other boxes a =
    cbrt(4 / rho). Bit-identical to the engine's generators
    (tests/test_bench_host.py)."""
    n = 4 * nx * ny * nz
    if nx == ny == nz:
        L = math.cbrt(float(n) / RHO)  # libm cbrt, as tmd_gen_fcc (np.cbrt differs by an ulp)
        a = L / nx
        box = np.array([L, L, L])
    else:
        a = float(np.cbrt(4.0 / RHO))  # gen_fcc_box's rule
        box = np.array([nx * a, ny * a, nz * a])
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cell = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1).astype(np.float64)
    pos = np.ascontiguousarray(((cell[:, None, :] + basis[None, :, :] + offset) * a)
                               .reshape(-1, 3))
    return box, np.arange(n, dtype=np.int64), pos


class Inputs:
    """One system: box, ids, positions, velocities (+ bonds), the interaction
    settings, and the reference-engine kwargs."""

    def __init__(self, box, ids, pos, vel, *, r_skin, dt, bonds=None, ref_kw=None):
        self.box, self.id, self.pos, self.vel = box, ids, pos, vel
        self.bonds = bonds
        self.r_skin, self.dt = r_skin, dt
        self.ref_kw = ref_kw or {}
        self.n = int(ids.shape[0])


def kg_ref_kw(bonds):
    return dict(r_cut=2.0 ** (1.0 / 6.0), bonds=bonds, fene=(30.0, 1.5))


def make_inputs_ours(kind: str, cells: int, weak_ranks: int):
    """Inputs through the engine's own generators (our arm)."""
    from paper_2109_10876_b200 import engine as E
    if kind == "lj":
        if weak_ranks > 0:
            f = E.gen_fcc_box(*weak_dims(weak_ranks), RHO, 1.0, SEED)
        else:
            f = E.gen_fcc(cells, RHO, 1.0, SEED)
        return f, E.Interactions(), Inputs(f.box, f.id, f.pos, f.vel, r_skin=0.3, dt=0.005)
    if kind == "kg":
        chains = max(1, round(20000 * (cells / 64) ** 3))
        f = E.kg_warmup(E.gen_chains(chains, 200, 0.85, 0.97, seed=SEED))
        return f, E.kg_interactions(), Inputs(f.box, f.id, f.pos, f.vel, r_skin=0.4,
                                              dt=0.01, bonds=f.bonds,
                                              ref_kw=kg_ref_kw(f.bonds))
    if kind == "slab":
        n = 2097152 if cells == 64 else 4 * cells ** 3
        c = 81 if cells == 64 else cells
        f = E.gen_fcc_slab(c, RHO, 0.7, SEED, n=n)
        return f, E.Interactions(), Inputs(f.box, f.id, f.pos, f.vel, r_skin=0.3, dt=0.005)
    raise SystemExit(f"unknown config {kind!r}")


def make_inputs_reference(kind: str, cells: int, weak_ranks: int) -> Inputs:
    """Inputs for the reference arm without this repo's library: numpy FCC
    positions + the reference's own velocity draw (gen_detail::
    thermal_velocities + zero_net_momentum, generators.hpp:19-39, through
    oracle/_ref). The KG melt needs the force-capped warm-up (absent from the
    reference), so it is generated by a separate process of this script and
    handed over as a file."""
    from oracle import ref
    if not ref.available():
        ref.build()
    if kind == "lj":
        dims = weak_dims(weak_ranks) if weak_ranks > 0 else [cells] * 3
        box, ids, pos = fcc_numpy(*dims)
        vel = ref.thermal_velocities(ids, 1.0, SEED)
        return Inputs(box, ids, pos, vel, r_skin=0.3, dt=0.005)
    if kind == "slab":
        n = 2097152 if cells == 64 else 4 * cells ** 3
        c = 81 if cells == 64 else cells
        box, ids, pos = fcc_numpy(c, c, c)
        pos = pos.copy()
        pos[:, 2] += box[2]
        box = box.copy()
        box[2] *= 3.0
        ids, pos = ids[:n], np.ascontiguousarray(pos[:n])
        vel = ref.thermal_velocities(ids, 0.7, SEED)
        return Inputs(box, ids, pos, vel, r_skin=0.3, dt=0.005)
    if kind == "kg":
        path = Path(os.environ.get("TMPDIR", "/tmp")) / f"tmd_bench_kg_{cells}.npz"
        if not path.exists():
            subprocess.run([sys.executable, str(Path(__file__).resolve()), "--make-kg-input",
                            str(path), "--cells", str(cells)], check=True,
                           env={k: v for k, v in os.environ.items()
                                if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
        d = np.load(path)
        return Inputs(d["box"], d["id"], d["pos"], d["vel"], r_skin=0.4, dt=0.01,
                      bonds=d["bonds"], ref_kw=kg_ref_kw(d["bonds"]))
    raise SystemExit(f"unknown config {kind!r}")


# ----------------------------------------------------------------------------------
# the reference engine on the host cores

def cpu_reference_run(w: Inputs, steps_wanted: int, warmup: int, budget_s: float,
                      one_thread_budget_s: float = 0.0) -> dict:
    """The reference engine (oracle/_ref) with every host core: particle-steps/s
    over a bounded sample, its five SectionTimers over the timed steps, and
    (one_thread_budget_s > 0) a 1-thread rate from a second Engine over a copy
    of the same Domain (ref_clone)."""
    from oracle import ref
    if not ref.available():
        ref.build()
    cores = os.cpu_count() or 1
    rv = w.ref_kw.get("r_cut", 2.5) + w.r_skin
    cells = int(np.prod([max(1, int(math.floor(float(L) / rv))) for L in w.box]))
    n_sub = max(1, min(2 * cores, cells))
    t0 = time.perf_counter()
    r = ref.RefEngine(w.box, w.id, w.pos, w.vel, r_skin=w.r_skin, n_sub=n_sub, workers=cores,
                      dt=w.dt, **w.ref_kw)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    r.run(max(1, warmup))
    est = (time.perf_counter() - t0) / max(1, warmup)
    steps = int(max(1, min(steps_wanted, budget_s / max(est, 1e-9))))
    sec0, el0 = r.timers()
    t0 = time.perf_counter()
    r.run(steps)
    t = time.perf_counter() - t0
    sec1, el1 = r.timers()
    n = w.n
    out = {"value": n * steps / t, "cores": cores, "steps": steps, "n_sub": n_sub,
           "build_s": t_build,
           "sections_s": dict(zip(("Forces", "Comm", "Integrate", "Neigh", "Resort"),
                                  (float(x) for x in sec1 - sec0))),
           "elapsed_s": float(el1 - el0)}
    out["sample"] = (f"{n}-particle system, {steps} NVE steps (of {steps_wanted} requested) "
                     f"after build_domain + Engine ctor ({t_build:.1f} s, untimed) and "
                     f"{max(1, warmup)} warm-up steps; reference taskmd Engine, "
                     f"worker_threads={cores}, n_sub={n_sub} (fixed 2x workers, at most the cell count), "
                     f"g++ -O3 -DNDEBUG")
    if one_thread_budget_s > 0.0:
        t0 = time.perf_counter()
        r1 = r.clone(1)
        t_clone = time.perf_counter() - t0
        t0 = time.perf_counter()
        r1.run(1)
        est1 = time.perf_counter() - t0
        s1 = int(max(1, min(steps_wanted, one_thread_budget_s / max(est1, 1e-9))))
        t0 = time.perf_counter()
        r1.run(s1)
        t1 = time.perf_counter() - t0
        sec_1, _ = r1.timers()
        r1.close()
        out["one_thread"] = {
            "value": n * s1 / t1, "steps": s1,
            "sample": f"same Domain (n_sub={n_sub}), worker_threads=1, {s1} steps after 1 "
                      f"warm-up step (Engine ctor {t_clone:.1f} s, untimed)"}
    r.close()
    return out


def run_reference_arm(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = workload_config(args.config, args.cells, args.weak, ws)
    try:
        w = make_inputs_reference(args.config, args.cells, ws if args.weak else 0)
        c = cpu_reference_run(w, args.steps, args.warmup, args.ref_budget_s)
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    v = c["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": c["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * w.n / v,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": c["cores"], "kind": "reference",
                         "sample": c["sample"], "sections_s": c["sections_s"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "details": {"parallelism": "host threads (reference CPU engine), rank 0 only",
                    "inputs": "numpy FCC + the reference's thermal_velocities "
                              "(no repo library in this process)"},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------------
# our arm

def ncu_capture(n: int, kernel: str):
    """Per-launch DRAM bytes and the L1TEX / DRAM throughput fractions of the
    step kernel from the committed ncu capture of this workload
    (profiles/force_kernel_ncu.json, written by scripts/ncu_summary.py), or
    None when the capture is of another size or kernel."""
    prof = ROOT / "profiles" / "force_kernel_ncu.json"
    try:
        pj = json.loads(prof.read_text())
    except (OSError, ValueError):
        return None
    for rec in pj if isinstance(pj, list) else [pj]:
        if rec.get("n_particles") == n and rec.get("kernel", kernel) == kernel:
            return rec
    return None


def roofline(eng, n: int, step_ms: float, sm_mhz: float, reps: int) -> dict:
    """The production step kernel (forces + fused velocity-Verlet epilogue)
    against the frozen roofline of SURVEY §8(d) / BASELINE.md §4:
    B = N*52 + E*28 bytes, F = 8E + 20P, T_roof = max(B/HBM, F/FP64)."""
    from paper_2109_10876_b200 import engine as E
    st = eng.list_stats()
    kc = eng.kernel_config()
    E_ent, P_cut = st["entries"], st["in_cut"]
    t_ms = eng.time_step_kernel(reps)
    B = n * 52 + E_ent * 28
    F = 8 * E_ent + 20 * P_cut
    peaks = measured_peaks()
    fp64 = E.fp64_peak_tflops(eng.config().device)
    t_hbm = B / (peaks["hbm_gbs"] * 1e9)
    t_flop = F / (fp64 * 1e12)
    kernel = ("k_forces_l1<kFused>" if kc["lanes"] == 1
              else f"k_forces_lanes<{kc['lanes']}, kFused>")
    cap = ncu_capture(n, kernel)
    if t_hbm >= t_flop:
        achieved = B / (t_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"]}
    else:
        achieved = F / (t_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64}
    roof["traffic"] = None if cap is None else cap.get("dram_bytes_per_launch")
    # what binds it: every gathered neighbour of a warp's 32 lanes lies in its
    # own 128-B line, one L1 wavefront each, one wavefront per clock per SM
    t_l1 = E_ent / (148 * sm_mhz * 1e6)
    roof.update({
        "kernel": kernel, "algorithmic_bytes": B, "algorithmic_flops": F,
        "entries": E_ent, "in_cut_entries": P_cut, "kernel_ms": t_ms,
        "t_roof_ms": 1e3 * max(t_hbm, t_flop), "fp64_peak_tflops_measured": fp64,
        "peak_source": peaks["source"], "share_of_step": t_ms / step_ms,
        "l1": {"model": "one L1 wavefront per gathered list entry, 1 wavefront/clk/SM",
               "t_ms": 1e3 * t_l1, "frac": 1e3 * t_l1 / t_ms, "sm_mhz": sm_mhz},
        "definition": "B = N*52 + E*28 bytes (gathered x_j counted at HBM), F = 8E + 20P "
                      "(E full-list entries, P in-cut entries); frac = achieved / peak = "
                      "T_roof / T_kernel. frac > 1: the gathers are served by L1/L2; the "
                      "binding resource is the L1 (see l1, ncu)",
    })
    if cap is not None:
        roof["ncu"] = {k: cap.get(k) for k in ("dram_bytes_per_launch", "dram_frac_of_peak",
                                               "l1tex_frac_of_peak", "fp64_pipe_frac",
                                               "duration_ms", "source")}
        if cap.get("dram_bytes_per_launch"):
            roof["ncu"]["dram_gbs_live"] = cap["dram_bytes_per_launch"] / (t_ms * 1e-3) / 1e9
    return roof


def pinned_like(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


def run_ours(args) -> None:
    import torch
    from paper_2109_10876_b200 import engine as E

    ws, rank, local = dist_env()
    if ws > 1 or args.decomposed:
        run_decomposed(args)
        return
    torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    cfg = workload_config(args.config, args.cells, args.weak, 1)
    flat, inter, w = make_inputs_ours(args.config, args.cells, 1 if args.weak else 0)
    n = w.n
    ecfg = E.EngineConfig(dt=w.dt, section_timers=False, device=dev)
    eng = E.Engine(flat, inter, w.r_skin, ecfg)

    eng.run(args.warmup)
    eng.prepare_graphs()  # every graph shape the timed run launches, captured now
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
    clk = clocks.summary()

    st = eng.list_stats()
    roof = roofline(eng, n, ms_per_step, clk.get("sm_mhz") or 1965.0, args.force_reps)
    work_set = int(st["capacity"]) * 4 * ((n + 31) // 32 * 32) + n * 180
    eng.close()

    # -- e2e through the public API from host buffers ----------------------------------
    # The caller's arrays live in pinned host memory (allocated and filled
    # before the timed region, as a serving process keeps its staging
    # buffers); the upload and the final download are inside it.
    flat_in = E.FlatConfig(flat.box, pinned_like(flat.id), pinned_like(flat.pos),
                           pinned_like(flat.vel),
                           mass=None if flat.mass is None else pinned_like(flat.mass),
                           type=flat.type, bonds=flat.bonds)
    out = E.FlatConfig(flat.box, torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(),
                       torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy(),
                       torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy())
    torch.cuda.synchronize()
    # (ids lo, lo + 1, ... in input order are generated on the device, not copied)
    ids_iota = bool(n) and bool(np.array_equal(flat_in.id, flat_in.id[0] + np.arange(n)))
    h2d = flat_in.pos.nbytes + flat_in.vel.nbytes + (0 if ids_iota else flat_in.id.nbytes) + (
        0 if flat_in.mass is None else flat_in.mass.nbytes)
    t0 = time.perf_counter()
    e2 = E.Engine(flat_in, inter, w.r_skin, ecfg)
    rows = e2.run_observed(args.steps, stride=1)  # each step's observables land in host memory
    e2.flatten(out=out)
    t_e2e = time.perf_counter() - t0
    assert len(rows) == args.steps
    obs_bytes = 32 * len(rows)  # (step, KE, PE, W) per step, written by the device to host
    # (a dense id range comes back in id order: the host writes the id column)
    ids_dense = bool(n) and int(flat_in.id.max()) - int(flat_in.id.min()) == n - 1
    d2h = obs_bytes + out.pos.nbytes + out.vel.nbytes + (0 if ids_dense else out.id.nbytes)
    e2.close()
    e2e = {"value": n * args.steps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
           "seconds": t_e2e,
           "what": "Engine(create from the caller's arrays in pinned host memory: validate, "
                   "upload, bin, build, first forces) + run_observed(K, stride 1): every "
                   "step's (step, KE, PE, W) written by the device into mapped pinned host "
                   "memory + flatten(out=pinned buffers) download"}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            c = cpu_reference_run(w, args.steps, 2, args.cpu_budget_s, args.cpu1_budget_s)
            cpu = {"value": c["value"], "unit": UNIT, "cores": c["cores"], "kind": "reference",
                   "sample": c["sample"], "sections_s": c["sections_s"]}
            if "one_thread" in c:
                cpu["one_thread"] = c["one_thread"]
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    l2 = (f"working set ~{work_set / 2 ** 30:.2f} GiB > 126 MB L2: no flush needed"
          if work_set > 2 * L2_BYTES else
          f"working set ~{work_set / 2 ** 20:.0f} MiB fits the 126 MB L2: steps run "
          f"L2-warm (a production step re-reads the same state every step); no flush")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": cfg, "roofline": roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "details": {"parallelism": "single GPU", "l2": l2,
                    "rebuilds_in_timed_region": rebuilds, "section_timers": False,
                    "nbr_capacity": st["capacity"], "cell_grid": list(st["dims"]),
                    "graphs": "captured before the timed region (prepare_graphs)"},
    }
    print(json.dumps(line))


def run_decomposed(args) -> None:
    """N > 1: the workload on an N-slab z decomposition (decomp.py), one
    process per GPU, the native C++ step loop: fused peer-store halo, NCCL
    migration + all-reduces (strong scaling: the same system at every N;
    --weak: 2.048M particles per GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2109_10876_b200 import engine as E
    from paper_2109_10876_b200.decomp import DecomposedEngine, TorchDistComm

    ws, rank, local = dist_env()
    if args.dist_backend in ("gloo", "hostfile"):
        # pipeline checks on a one-GPU box, every rank on GPU 0 (the numbers are
        # not a scaling measurement). gloo: the Python protocol, buffers staged
        # through host memory. hostfile: the production C++ loop, one process
        # per rank, collectives through a shared file mapping, the fused halo
        # through CUDA IPC mappings of the other processes' buffers.
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    torch.cuda.set_device(dev)
    cfg = workload_config(args.config, args.cells, args.weak, ws)
    flat, inter, w = make_inputs_ours(args.config, args.cells, ws if args.weak else 0)
    n = w.n
    ecfg = E.EngineConfig(dt=w.dt, section_timers=False, device=dev)
    balance = "count" if args.config == "slab" else "static"

    # the C++ step loop with NCCL on the context stream (tmd_slab_nccl.cuh);
    # the Python protocol for the gloo pipeline check
    native = args.dist_backend != "gloo"
    made = [0]

    def transport():
        if args.dist_backend != "hostfile":
            return TorchDistComm()
        from paper_2109_10876_b200.decomp import HostFileComm

        class HostFileBenchComm(HostFileComm):
            """+ the host-side sum run_observed reduces its table with, over
            the job's gloo group (the transport itself is device-stream only)."""

            def allreduce_sum(self, vals):
                t = torch.from_numpy(np.sum(list(vals.values()), axis=0).astype(np.float64))
                dist.all_reduce(t)
                return t.numpy()

        # a fresh mapping per engine, named by the job's rendezvous port
        made[0] += 1
        path = os.path.join(tempfile.gettempdir(),
                            f"tmd_bench_{os.environ.get('MASTER_PORT', '0')}_{made[0]}.bin")
        if rank == 0 and os.path.exists(path):
            os.unlink(path)
        dist.barrier()
        return HostFileBenchComm(path, rank, ws)

    def make():
        return DecomposedEngine(flat, inter, w.r_skin, ecfg, comm=transport(),
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

    # e2e from the caller's arrays in pinned host memory and into pinned
    # download buffers (sized for the whole system: a slab's share is known
    # only after its run), both prepared before the timed region
    flat_in = E.FlatConfig(flat.box, pinned_like(flat.id), pinned_like(flat.pos),
                           pinned_like(flat.vel), bonds=flat.bonds)
    out = (torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(),
           torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy(),
           torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy())
    e2_comm = transport()
    e2_make = lambda: DecomposedEngine(flat_in, inter, w.r_skin, ecfg, comm=e2_comm,  # noqa: E731
                                       device_of=lambda r: local, balance=balance, native=native)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    e2 = e2_make()
    # every step's (step, KE, PE, W) recorded by the device (rank-local sums),
    # the table reduced over ranks once at the end
    rows = e2.run_observed(args.steps, stride=1)
    assert rows.shape[0] == args.steps
    ids, pos, vel, _f = e2.local_state(out=out)
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    e2.close()
    h2d = flat.pos.nbytes + flat.vel.nbytes + flat.id.nbytes
    d2h = 40 * args.steps + pos.nbytes + vel.nbytes + ids.nbytes
    dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": n * args.steps / (ms * 1e-3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg, "roofline": None, "cpu_baseline": None,
        "e2e": {"value": n * args.steps / t_e2e, "unit": UNIT,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "seconds": t_e2e,
                "what": "DecomposedEngine(create from the caller's pinned arrays: every rank "
                        "stages the whole system on its GPU and keeps its slab; NCCL attach "
                        "(the process's communicator, cached after the device-timed engine) + "
                        "run_observed(K, stride 1): every step's rank-local (step, KE, PE, W) "
                        "written by the device into mapped host memory, the table summed over "
                        "ranks at the end + local_state(out=pinned buffers)"},
        "gpu_launches": launches * ws, "clocks": clocks.summary(),
        "details": {"parallelism": f"{ws} z-slabs (spatial decomposition, {args.dist_backend} "
                                   f"halo + migration, {balance} cuts, "
                                   f"{'native C++' if native else 'python'} step loop)",
                    "l2": "working set > 126 MB L2 on every rank; no flush",
                    "rebuilds_in_timed_region": rebuilds, "section_timers": False,
                    "rank0_slab": sizes, "exchanged_bytes_rank0": xbytes},
    }
    print(json.dumps(line))


def launch_check(args) -> None:
    """CPU check of the launch path (tests/test_bench_host.py): every rank joins
    a gloo group and all-reduces its rank; rank 0 prints the world it saw."""
    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank + 1], dtype=torch.int64)
        dist.all_reduce(t)
        total = int(t.item())
        dist.destroy_process_group()
    else:
        total = 1
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": ws, "gpus_flag": args.gpus,
                          "rank_sum": total,
                          "config": workload_config(args.config, args.cells, args.weak, ws)}))


def make_kg_input(args) -> None:
    """Writes the warmed-up KG melt (our engine's force-capped warm-up) for the
    reference arm, which must not load this repo's library itself."""
    flat, _inter, w = make_inputs_ours("kg", args.cells, 0)
    np.savez(args.make_kg_input, box=flat.box, id=flat.id, pos=flat.pos, vel=flat.vel,
             bonds=flat.bonds)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cells", type=int, default=160,
                    help="FCC cells per edge (160 = 16.4M configs[4], 64 = 1M configs[1], "
                         "20 = 32K configs[0])")
    ap.add_argument("--config", choices=["lj", "kg", "slab"], default="lj",
                    help="lj: FCC LJ fluid (configs[0,1,4] by --cells 20/64/160); kg: "
                         "Kremer-Grest melt (configs[2], --cells 64); slab: liquid-vapour "
                         "slab (configs[3], --cells 64)")
    ap.add_argument("--weak", action="store_true",
                    help="lj only: weak scaling at 2.048M particles per GPU (FCC 80^3 x 4 "
                         "per GPU; the box doubles along x, y, z with N; 8 GPUs = the "
                         "configs[4] 160^3 box)")
    ap.add_argument("--force-reps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--cpu1-budget-s", type=float, default=10.0,
                    help="bounded 1-thread sample of the reference (0 = skip)")
    ap.add_argument("--ref-budget-s", type=float, default=90.0)
    ap.add_argument("--decomposed", action="store_true",
                    help="run the slab decomposition even at N = 1 (under torchrun): the "
                         "single slab exchanges its halo with itself over NCCL")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo", "hostfile"], default="nccl",
                    help="N > 1 only; gloo / hostfile = pipeline checks with every rank on "
                         "GPU 0 (Python protocol / the native C++ loop over the host-staged "
                         "transport with CUDA IPC halo)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--make-kg-input", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.make_kg_input:
        make_kg_input(args)
        return
    relaunch_if_needed(args, argv)
    if args.launch_check:
        launch_check(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
