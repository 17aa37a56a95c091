"""`md`-style command line on the GPU engine.

    python -m paper_2109_10876_b200.cli run      --config FILE [--threads N] [--seed S] [--out DIR]
    python -m paper_2109_10876_b200.cli generate --config FILE ...
    python -m paper_2109_10876_b200.cli verify   --config FILE ...
    python -m paper_2109_10876_b200.cli autotune --config FILE ...

The reference's md_cli.cpp (CLI11, absent here) restated over the B200
engine with its output formats unchanged: observables CSV on stdout
("step,kinetic,potential,temperature", 17 significant digits), the
completion line on stderr, TimingWriter CSVs (io.hpp:54-91), XYZ
trajectories (io.hpp:17-48), generate's system.xyz + resolved.cfg, verify's
report, and the exit codes 0 / 1 config / 2 physics / 3 verify mismatch
(errors.hpp:10-15, md_cli.cpp:333-352). verify compares the list-based
engine with an all-pairs minimum-image evaluation on the GPU (the role of
oracle.hpp in the reference).

engine.n_sub, engine.worker_threads and the autotune keys are accepted and
have no GPU meaning (one context per GPU; `autotune` reports the single
choice and runs). engine.gpus > 1 runs the z-slab decomposition and must be
launched with torchrun, one process per GPU.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path
from typing import Optional, TextIO

import numpy as np

from . import engine as E
from .runconfig import RunConfig, generate_system, parse_run_config, serialize_run_config, \
    with_overrides

EXIT_OK, EXIT_CONFIG, EXIT_PHYSICS, EXIT_VERIFY = 0, 1, 2, 3
VERIFY_CAP = 5000
VERIFY_TOLERANCE = 1e-10


def _f17(v: float) -> str:
    return format(v, ".17g")


def load_config(path: str, threads: int, seed: Optional[int]) -> RunConfig:
    try:
        text = Path(path).read_text()
    except OSError:
        raise E.ConfigError(f"cannot open config file: {path}") from None
    return with_overrides(parse_run_config(text), threads, seed)


def out_path(out_dir: str, file: str) -> str:
    p = Path(file)
    return str(p) if p.is_absolute() else str(Path(out_dir) / p)


def write_xyz_frame(os_: TextIO, f: E.FlatConfig, step: int) -> None:
    """write_xyz_frame (io.hpp:17-29)."""
    n = f.size()
    os_.write(f"{n}\nstep={step} box={_f17(f.box[0])} {_f17(f.box[1])} {_f17(f.box[2])}\n")
    types = f.type if f.type is not None else np.zeros(n, np.int32)
    os_.write("".join(f"{int(t)} {format(p[0], '.10g')} {format(p[1], '.10g')} "
                      f"{format(p[2], '.10g')}\n" for t, p in zip(types, f.pos)))


class TimingWriter:
    """TimingWriter (io.hpp:54-91): step_range,section,seconds."""

    def __init__(self, path: str, per_step: bool):
        try:
            self.out = open(path, "w")
        except OSError:
            raise E.ConfigError(f"cannot open timing file: {path}") from None
        self.per_step = per_step
        self.out.write("step_range,section,seconds\n")

    def record_step(self, step: int, delta) -> None:
        if not self.per_step:
            return
        rng = f"{step - 1}-{step}"
        for name, v in zip(E.SECTION_NAMES, delta):
            self.out.write(f"{rng},{name},{format(v, '.9g')}\n")

    def finish(self, steps: int, t: E.SectionTimers) -> None:
        rng = f"0-{steps}"
        for name, v in zip(E.SECTION_NAMES, t.seconds):
            self.out.write(f"{rng},{name},{format(v, '.9g')}\n")
        self.out.write(f"{rng},Elapsed,{format(t.elapsed, '.9g')}\n")
        self.out.close()


def _print_obs(o: E.StepObservables) -> None:
    sys.stdout.write(f"{o.step},{_f17(o.kinetic)},{_f17(o.potential)},"
                     f"{_f17(o.temperature)}\n")


def _device(cfg: RunConfig) -> int:
    return cfg.gpu.device


def run_engine(cfg: RunConfig, flat: E.FlatConfig, out_dir: str) -> None:
    """run_engine (md_cli.cpp:89-137) on one GPU."""
    ecfg = E.EngineConfig(dt=cfg.engine.dt, steps=cfg.engine.steps,
                          thermostat=cfg.engine.thermostat, n_sub=cfg.engine.n_sub,
                          worker_threads=cfg.engine.worker_threads,
                          observable_stride=cfg.engine.observable_stride,
                          section_timers=True, device=_device(cfg))
    eng = E.Engine(flat, cfg.inter, cfg.r_skin, ecfg)
    traj = None
    if cfg.output.trajectory_path:
        p = out_path(out_dir, cfg.output.trajectory_path)
        try:
            traj = open(p, "w")
        except OSError:
            raise E.ConfigError(f"cannot open trajectory file: {p}") from None
    timing = None
    per_step = cfg.output.timing_mode == "per_step"
    if cfg.output.timing_path:
        timing = TimingWriter(out_path(out_dir, cfg.output.timing_path), per_step)
    sys.stdout.write("step,kinetic,potential,temperature\n")
    _print_obs(eng.observe())
    if traj:
        write_xyz_frame(traj, eng.flatten(), 0)
    steps = cfg.engine.steps
    ostride, tstride = cfg.engine.observable_stride, cfg.output.trajectory_stride
    if not traj and not (timing and per_step) and steps > 0:
        # only observable rows: recorded on the device, no host round trip per row
        for r in eng.run_observed(steps, ostride):
            sys.stdout.write(f"{int(r[0])},{_f17(r[1])},{_f17(r[2])},{_f17(r[3])}\n")
    s = steps if (not traj and not (timing and per_step)) else 0
    while s < steps:
        # advance to the next step that needs the host (observable row,
        # trajectory frame, per-step timing record), in one device run
        nxt = min(steps, (s // ostride + 1) * ostride)
        if traj:
            nxt = min(nxt, (s // tstride + 1) * tstride)
        if timing and per_step:
            nxt = s + 1
        before = eng.timers().seconds.copy()
        eng.run(nxt - s)
        s = nxt
        if timing and per_step:
            timing.record_step(s, eng.timers().seconds - before)
        if traj and s % tstride == 0:
            write_xyz_frame(traj, eng.flatten(), s)
        if s % ostride == 0:
            _print_obs(eng.observe())
    sys.stdout.flush()
    t = eng.timers()
    if timing:
        timing.finish(steps, t)
    if traj:
        traj.close()
    secs = ", ".join(f"{n} {format(v, '.6g')}" for n, v in zip(E.SECTION_NAMES, t.seconds))
    sys.stderr.write(f"completed {eng.step_count()} steps in {format(t.elapsed, '.6g')} s "
                     f"({secs}); {eng.rebuild_count()} list rebuilds, "
                     f"{eng.steal_count()} steals\n")
    eng.close()


def run_decomposed(cfg: RunConfig, flat: E.FlatConfig) -> None:
    """engine.gpus > 1: one process per GPU (torchrun), z-slab decomposition."""
    import torch
    import torch.distributed as dist
    from .decomp import DecomposedEngine, TorchDistComm
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != cfg.gpu.gpus:
        raise E.ConfigError(f"engine.gpus = {cfg.gpu.gpus} needs torchrun with that many "
                            f"processes (WORLD_SIZE = {world})")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ecfg = E.EngineConfig(dt=cfg.engine.dt, thermostat=cfg.engine.thermostat,
                          section_timers=False, device=local)
    eng = DecomposedEngine(flat, cfg.inter, cfg.r_skin, ecfg, comm=TorchDistComm(),
                           device_of=lambda r: local, balance=cfg.gpu.balance)
    rank0 = dist.get_rank() == 0
    if rank0:
        sys.stdout.write("step,kinetic,potential,temperature\n")
    o = eng.observe()
    if rank0:
        _print_obs(o)
    t0 = time.perf_counter()
    s, steps, ostride = 0, cfg.engine.steps, cfg.engine.observable_stride
    while s < steps:
        nxt = min(steps, (s // ostride + 1) * ostride)
        eng.run(nxt - s)
        s = nxt
        o = eng.observe()
        if rank0 and s % ostride == 0:
            _print_obs(o)
    if rank0:
        sys.stderr.write(f"completed {steps} steps in {format(time.perf_counter() - t0, '.6g')}"
                         f" s on {world} GPUs; {eng.rebuild_count()} list rebuilds, "
                         f"{eng.recuts} re-cuts\n")
    eng.close()


def cmd_run(a) -> int:
    cfg = load_config(a.config, a.threads, a.seed)
    Path(a.out).mkdir(parents=True, exist_ok=True)
    flat = generate_system(cfg, device=_device(cfg))
    if cfg.gpu.gpus > 1:
        run_decomposed(cfg, flat)
    else:
        run_engine(cfg, flat, a.out)
    return EXIT_OK


def cmd_autotune(a) -> int:
    """The GPU engine has no subnodes to tune: probe the single configuration,
    report it in autotune.csv's format (io.hpp:94-101), then run."""
    cfg = load_config(a.config, a.threads, a.seed)
    Path(a.out).mkdir(parents=True, exist_ok=True)
    flat = generate_system(cfg, device=_device(cfg))
    ecfg = E.EngineConfig(dt=cfg.engine.dt, thermostat=cfg.engine.thermostat,
                          section_timers=False, device=_device(cfg))
    eng = E.Engine(flat, cfg.inter, cfg.r_skin, ecfg)
    t0 = time.perf_counter()
    eng.run(cfg.probe_steps)
    secs = time.perf_counter() - t0
    eng.close()
    p = out_path(a.out, "autotune.csv")
    with open(p, "w") as f:
        f.write(f"n_sub,seconds,selected\n1,{format(secs, '.9g')},1\n")
    sys.stderr.write(f"n_sub        1  {format(secs, '.6g')} s  <- selected "
                     f"(one GPU context, no subnodes)\nwrote {p}\n")
    if cfg.engine.steps > 0:
        run_engine(cfg, flat, a.out)
    return EXIT_OK


def cmd_generate(a) -> int:
    cfg = load_config(a.config, a.threads, a.seed)
    Path(a.out).mkdir(parents=True, exist_ok=True)
    flat = generate_system(cfg, device=_device(cfg))
    xyz = out_path(a.out, "system.xyz")
    with open(xyz, "w") as f:
        write_xyz_frame(f, flat, 0)
    rc = out_path(a.out, "resolved.cfg")
    Path(rc).write_text(serialize_run_config(cfg))
    nb = 0 if flat.bonds is None else len(flat.bonds)
    sys.stderr.write(f"generated {flat.size()} particles, {nb} bonds, 0 angles in box "
                     f"({format(flat.box[0], '.6g')}, {format(flat.box[1], '.6g')}, "
                     f"{format(flat.box[2], '.6g')}); wrote {xyz} and {rc}\n")
    return EXIT_OK


def cmd_verify(a) -> int:
    """cmd_verify (md_cli.cpp:205-306): one force evaluation of the engine vs
    the all-pairs evaluation; forces to 1e-10 and identical pair sets."""
    cfg = load_config(a.config, a.threads, a.seed)
    if cfg.engine.thermostat is not None:
        sys.stderr.write("verify compares conservative forces; ignoring the configured "
                         "thermostat\n")
        cfg.engine.thermostat = None
    flat = generate_system(cfg, device=_device(cfg))
    if flat.size() > VERIFY_CAP:
        raise E.ConfigError(f"verify runs an O(N^2) reference and is capped at {VERIFY_CAP} "
                            f"particles; this config generates {flat.size()}")
    if cfg.inter.fene is not None and flat.bonds is not None and len(flat.bonds):
        raise E.ConfigError("verify compares the pair (LJ) forces; bonded systems are checked "
                            "by the parity tests")
    n_sub = cfg.engine.n_sub
    if cfg.n_sub_auto:
        n_sub = 1
        sys.stderr.write("engine.n_sub = auto resolves to 1 for verification\n")
    eng = E.Engine(flat, cfg.inter, cfg.r_skin,
                   E.EngineConfig(dt=cfg.engine.dt, device=_device(cfg)))
    ids, got = eng.forces()
    pairs = eng.pairs()
    pe = eng.potential_energy()
    eng.close()
    want_f, want_pe, want_pairs = E.brute_force(flat, cfg.inter,
                                                cfg.inter.lj.r_cut + cfg.r_skin,
                                                device=_device(cfg))
    order = np.argsort(flat.id, kind="stable")
    max_diff = float(np.abs(got - want_f[order]).max()) if len(order) else 0.0
    eng_set = {tuple(p) for p in pairs.tolist()}
    ref_set = {tuple(p) for p in want_pairs.tolist()}
    engine_only = sorted(eng_set - ref_set)
    oracle_only = sorted(ref_set - eng_set)
    out = sys.stdout
    out.write(f"N = {flat.size()}, n_sub = {n_sub}, {len(pairs)} listed pairs\n")
    out.write(f"max |dF| = {format(max_diff, '.3g')} (tolerance "
              f"{format(VERIFY_TOLERANCE, '.3g')})\n")
    if not engine_only and not oracle_only:
        out.write("pair sets equal\n")
    else:
        out.write(f"pair sets differ: {len(engine_only)} listed only by the engine, "
                  f"{len(oracle_only)} only by the reference\n")
        for label, ps in (("engine", engine_only), ("reference", oracle_only)):
            for p in ps[:5]:
                out.write(f"  {label} ({p[0]}, {p[1]})\n")
    out.write(f"engine potential = {_f17(pe)}, reference potential = {_f17(want_pe)}\n")
    out.flush()
    if max_diff > VERIFY_TOLERANCE:
        raise E.VerifyError(f"force mismatch: max |dF| = {max_diff:f}")
    if engine_only or oracle_only:
        raise E.VerifyError("pair set mismatch")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(
        prog="md", description="short-range molecular dynamics on B200 (taskmd drop-in)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, helptext in (("run", "simulate a configured system"),
                           ("autotune", "probe, then run (no subnodes on the GPU)"),
                           ("generate", "write the initial system and the resolved config"),
                           ("verify", "check one force evaluation against an all-pairs one")):
        p = sub.add_parser(name, help=helptext)
        p.add_argument("--config", required=True, help="run configuration file")
        p.add_argument("--threads", type=int, default=0,
                       help="worker thread count (accepted; no GPU meaning)")
        p.add_argument("--seed", type=int, default=None, help="random seed (overrides config)")
        p.add_argument("--out", default=".", help="output directory")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_CONFIG
    cmds = {"run": cmd_run, "autotune": cmd_autotune, "generate": cmd_generate,
            "verify": cmd_verify}
    try:
        return cmds[a.cmd](a)
    except E.ConfigError as e:
        sys.stderr.write(f"config error: {e}\n")
        return EXIT_CONFIG
    except E.PhysicsError as e:
        sys.stderr.write(f"physics error: {e}\n")
        return EXIT_PHYSICS
    except E.VerifyError as e:
        sys.stderr.write(f"verification failed: {e}\n")
        return EXIT_VERIFY


if __name__ == "__main__":
    sys.exit(main())
