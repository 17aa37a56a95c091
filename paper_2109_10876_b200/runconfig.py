"""Run-configuration files for the GPU engine.

A restatement of the reference's run_config.hpp (parse_run_config,
serialize_run_config, generate_system; run_config.hpp:15-423): flat
"key = value" lines with dotted section prefixes, full-line # comments, blank
lines; unknown keys rejected; parse and type errors cite the line and key;
the same required / paired keys, defaults and validation messages, and a
canonical serialisation that parses back to the same values.

GPU additions (all optional; absent keys keep reference configs valid and
their serialisation unchanged):

  system.generator = fcc | fcc_slab | kg_melt   the BASELINE.json inputs
  system.cells = <int>                          fcc / fcc_slab lattice cells
  system.warmup = true|false                    kg_melt: force-capped warm-up
  engine.backend = gpu                          the only backend here
  engine.gpus = <int>                           z-slab decomposition (torchrun)
  engine.balance = static | count               slab cut planes (row f3)
  engine.device = <int>                         CUDA ordinal for one GPU
"""
from __future__ import annotations

import copy
import math
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from . import engine as E
from .engine import ConfigError

_DOUBLE = re.compile(r"^-?(?:\d+\.?\d*(?:[eE][-+]?\d+)?|\.\d+(?:[eE][-+]?\d+)?|"
                     r"(?:inf|infinity|nan)(?:\([A-Za-z0-9_]*\))?)$", re.IGNORECASE)
_INT = re.compile(r"^-?\d+$")
_UINT = re.compile(r"^\d+$")


@dataclass
class SystemSpec:
    generator: str = ""
    n: int = 0
    rho: float = 0.0
    temperature: float = 0.0
    box_length: float = 0.0
    diameter_fraction: float = 0.0
    rho_in: float = 0.0
    alpha: float = 0.0
    chains: int = 0
    chain_length: int = 0
    bond_length: float = 0.97
    min_distance: float = 0.8
    cells: int = 0          # GPU addition: fcc / fcc_slab
    warmup: bool = True     # GPU addition: kg_melt


@dataclass
class OutputSpec:
    timing_path: str = ""
    timing_mode: str = "summary"
    trajectory_path: str = ""
    trajectory_stride: int = 100
    observable_stride: int = 100


@dataclass
class GpuSpec:
    backend: str = "gpu"
    gpus: int = 1
    balance: str = "static"
    device: int = -1
    given: set = field(default_factory=set)  # GPU keys present in the file


@dataclass
class RunConfig:
    seed: int = 0
    system: SystemSpec = field(default_factory=SystemSpec)
    inter: E.Interactions = field(default_factory=E.Interactions)
    r_skin: float = 0.3
    engine: E.EngineConfig = field(default_factory=E.EngineConfig)
    n_sub_auto: bool = False
    output: OutputSpec = field(default_factory=OutputSpec)
    probe_steps: int = 20
    full_sweep: bool = False
    gpu: GpuSpec = field(default_factory=GpuSpec)


@dataclass
class _Entry:
    key: str
    value: str
    line: int


def _parse_kv_lines(text: str) -> List[_Entry]:
    """config_detail::parse_kv_lines (run_config.hpp:66-100)."""
    entries, seen = [], set()
    for line, raw in enumerate(text.split("\n"), start=1):
        stripped = raw.strip(" \t\r")
        if not stripped or stripped[0] == "#":
            continue
        eq = stripped.find("=")
        if eq < 0:
            raise ConfigError(f"config line {line}: expected 'key = value'")
        key = stripped[:eq].strip(" \t\r")
        value = stripped[eq + 1:].strip(" \t\r")
        if not key:
            raise ConfigError(f"config line {line}: empty key")
        if key in seen:
            raise ConfigError(f"config line {line}: duplicate key '{key}'")
        seen.add(key)
        entries.append(_Entry(key, value, line))
    return entries


def _bad(e: _Entry, want: str) -> ConfigError:
    return ConfigError(f"config line {e.line}, key '{e.key}': expected {want}, got '{e.value}'")


def _double(e: _Entry) -> float:
    if not _DOUBLE.match(e.value):
        raise _bad(e, "a number")
    v = e.value.lower()
    if v.lstrip("-").startswith("nan"):
        return float("nan")
    return float(v)


def _int(e: _Entry) -> int:
    if not _INT.match(e.value):
        raise _bad(e, "an integer")
    v = int(e.value)
    if not -(2 ** 63) <= v < 2 ** 63:
        raise _bad(e, "an integer")
    return v


def _uint(e: _Entry) -> int:
    if not _UINT.match(e.value) or int(e.value) >= 2 ** 64:
        raise _bad(e, "a non-negative integer")
    return int(e.value)


def _bool(e: _Entry) -> bool:
    if e.value == "true":
        return True
    if e.value == "false":
        return False
    raise _bad(e, "true or false")


def _validate_lj(lj: E.LjParams) -> None:
    """validate_lj (potentials.hpp:28-38)."""
    for name, v in (("epsilon", lj.epsilon), ("sigma", lj.sigma), ("r_cut", lj.r_cut)):
        if not (v > 0.0) or not math.isfinite(v):
            raise ConfigError(f"lj {name} must be finite and positive")


def _validate_fene(p: E.FeneParams) -> None:
    """validate_fene (potentials.hpp:84-91)."""
    if not (p.k > 0.0) or not math.isfinite(p.k):
        raise ConfigError("fene k must be finite and positive")
    if not (p.r_max > 0.0) or not math.isfinite(p.r_max):
        raise ConfigError("fene r_max must be finite and positive")


def _validate_angle(p: E.AngleParams) -> None:
    """validate_angle (potentials.hpp:115-124)."""
    if not (p.k >= 0.0) or not math.isfinite(p.k):
        raise ConfigError("angle k must be finite and >= 0")
    if not (0.0 <= p.theta0 <= 3.14159265358979323846):
        raise ConfigError("angle theta0 must lie in [0, pi]")


_SCALAR_KEYS = {
    "system.n": ("system", "n", _int), "system.rho": ("system", "rho", _double),
    "system.temperature": ("system", "temperature", _double),
    "system.box_length": ("system", "box_length", _double),
    "system.diameter_fraction": ("system", "diameter_fraction", _double),
    "system.rho_in": ("system", "rho_in", _double), "system.alpha": ("system", "alpha", _double),
    "system.chains": ("system", "chains", _int),
    "system.chain_length": ("system", "chain_length", _int),
    "system.bond_length": ("system", "bond_length", _double),
    "system.min_distance": ("system", "min_distance", _double),
    "system.cells": ("system", "cells", _int), "system.warmup": ("system", "warmup", _bool),
    "output.trajectory_stride": ("output", "trajectory_stride", _int),
    "output.observable_stride": ("output", "observable_stride", _int),
}


def parse_run_config(text: str) -> RunConfig:
    """parse_run_config (run_config.hpp:146-315) + the GPU keys."""
    c = RunConfig()
    present = set()
    fene = [0.0, 0.0]
    angle = [0.0, 0.0]
    bath = [0.0, 0.0]
    for e in _parse_kv_lines(text):
        present.add(e.key)
        k = e.key
        if k == "seed":
            c.seed = _uint(e)
        elif k == "system.generator":
            c.system.generator = e.value
        elif k in _SCALAR_KEYS:
            part, attr, conv = _SCALAR_KEYS[k]
            setattr(getattr(c, part), attr, conv(e))
        elif k == "interaction.epsilon":
            c.inter.lj.epsilon = _double(e)
        elif k == "interaction.sigma":
            c.inter.lj.sigma = _double(e)
        elif k == "interaction.r_cut":
            c.inter.lj.r_cut = _double(e)
        elif k == "interaction.energy_shifted":
            c.inter.lj.energy_shifted = _bool(e)
        elif k == "interaction.r_skin":
            c.r_skin = _double(e)
        elif k == "interaction.fene.k":
            fene[0] = _double(e)
        elif k == "interaction.fene.r_max":
            fene[1] = _double(e)
        elif k == "interaction.angle.k":
            angle[0] = _double(e)
        elif k == "interaction.angle.theta0":
            angle[1] = _double(e)
        elif k == "engine.dt":
            c.engine.dt = _double(e)
        elif k == "engine.steps":
            c.engine.steps = _int(e)
        elif k == "engine.n_sub":
            if e.value == "auto":
                c.n_sub_auto = True
            else:
                c.engine.n_sub = _int(e)
        elif k == "engine.worker_threads":
            c.engine.worker_threads = _int(e)
        elif k == "engine.thermostat.gamma":
            bath[0] = _double(e)
        elif k == "engine.thermostat.temperature":
            bath[1] = _double(e)
        elif k == "output.timing_path":
            c.output.timing_path = e.value
        elif k == "output.timing_mode":
            if e.value not in ("summary", "per_step"):
                raise _bad(e, "summary or per_step")
            c.output.timing_mode = e.value
        elif k == "output.trajectory_path":
            c.output.trajectory_path = e.value
        elif k == "autotune.probe_steps":
            c.probe_steps = _int(e)
        elif k == "autotune.full_sweep":
            c.full_sweep = _bool(e)
        elif k == "engine.backend":
            if e.value != "gpu":
                raise _bad(e, "gpu (the only backend of this build)")
            c.gpu.backend = e.value
            c.gpu.given.add(k)
        elif k == "engine.gpus":
            c.gpu.gpus = _int(e)
            c.gpu.given.add(k)
        elif k == "engine.balance":
            if e.value not in ("static", "count"):
                raise _bad(e, "static or count")
            c.gpu.balance = e.value
            c.gpu.given.add(k)
        elif k == "engine.device":
            c.gpu.device = _int(e)
            c.gpu.given.add(k)
        else:
            raise ConfigError(f"config line {e.line}: unknown key '{k}'")

    def require(key):
        if key not in present:
            raise ConfigError(f"config is missing required key '{key}'")

    def together(a, b):
        if (a in present) != (b in present):
            raise ConfigError(f"keys '{a}' and '{b}' must be given together")

    require("system.generator")
    g = c.system.generator
    if g in ("lattice", "random"):
        for key in ("system.n", "system.rho", "system.temperature"):
            require(key)
    elif g == "spherical":
        for key in ("system.box_length", "system.diameter_fraction", "system.rho_in",
                    "system.alpha", "system.temperature"):
            require(key)
    elif g in ("melt", "kg_melt"):
        for key in ("system.chains", "system.chain_length", "system.rho"):
            require(key)
    elif g in ("fcc", "fcc_slab"):
        for key in ("system.cells", "system.rho", "system.temperature"):
            require(key)
    else:
        raise ConfigError(f"unknown generator '{g}' (expected lattice, spherical, melt, or "
                          "random; this build adds fcc, fcc_slab, and kg_melt)")

    together("interaction.fene.k", "interaction.fene.r_max")
    together("interaction.angle.k", "interaction.angle.theta0")
    together("engine.thermostat.gamma", "engine.thermostat.temperature")
    if "interaction.fene.k" in present:
        c.inter.fene = E.FeneParams(fene[0], fene[1])
    elif g in ("melt", "kg_melt"):
        c.inter.fene = E.FeneParams()
    if "interaction.angle.k" in present:
        c.inter.angle = E.AngleParams(angle[0], angle[1])
    elif g == "melt":
        c.inter.angle = E.AngleParams()
    if "engine.thermostat.gamma" in present:
        c.engine.thermostat = E.LangevinParams(bath[0], bath[1], c.seed)
    c.engine.observable_stride = c.output.observable_stride

    if c.output.trajectory_stride < 1:
        raise ConfigError("trajectory stride must be at least 1")
    if c.output.observable_stride < 1:
        raise ConfigError("observable stride must be at least 1")
    if c.probe_steps < 10:
        raise ConfigError("autotune probe_steps must be at least 10")
    if c.engine.dt <= 0.0 or not math.isfinite(c.engine.dt):
        raise ConfigError("engine.dt must be positive and finite")
    E.validate_engine_config(c.engine)
    _validate_lj(c.inter.lj)
    if c.inter.fene is not None:
        _validate_fene(c.inter.fene)
    if c.inter.angle is not None:
        _validate_angle(c.inter.angle)
    if not math.isfinite(c.r_skin) or c.r_skin < 0.0:
        raise ConfigError("interaction.r_skin must be finite and non-negative")
    if c.gpu.gpus < 1:
        raise ConfigError("engine.gpus must be at least 1")
    return c


def _g(v: float) -> str:
    """std::ostream << double at precision 17 (the reference's serialisation)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return format(v, ".17g")


def serialize_run_config(c: RunConfig) -> str:
    """serialize_run_config (run_config.hpp:318-395) + the GPU keys given."""
    o: List[str] = [f"seed = {c.seed}\n\n", f"system.generator = {c.system.generator}\n"]
    s, g = c.system, c.system.generator
    if g in ("lattice", "random"):
        o += [f"system.n = {s.n}\n", f"system.rho = {_g(s.rho)}\n",
              f"system.temperature = {_g(s.temperature)}\n"]
    if g == "random":
        o.append(f"system.min_distance = {_g(s.min_distance)}\n")
    if g == "spherical":
        o += [f"system.box_length = {_g(s.box_length)}\n",
              f"system.diameter_fraction = {_g(s.diameter_fraction)}\n",
              f"system.rho_in = {_g(s.rho_in)}\n", f"system.alpha = {_g(s.alpha)}\n",
              f"system.temperature = {_g(s.temperature)}\n"]
    if g in ("melt", "kg_melt"):
        o += [f"system.chains = {s.chains}\n", f"system.chain_length = {s.chain_length}\n",
              f"system.rho = {_g(s.rho)}\n", f"system.bond_length = {_g(s.bond_length)}\n"]
    if g == "kg_melt":
        o.append(f"system.warmup = {'true' if s.warmup else 'false'}\n")
    if g in ("fcc", "fcc_slab"):
        o += [f"system.cells = {s.cells}\n", f"system.rho = {_g(s.rho)}\n",
              f"system.temperature = {_g(s.temperature)}\n"]
        if g == "fcc_slab" and s.n:
            o.append(f"system.n = {s.n}\n")
    o.append("\n")
    lj = c.inter.lj
    o += [f"interaction.epsilon = {_g(lj.epsilon)}\n", f"interaction.sigma = {_g(lj.sigma)}\n",
          f"interaction.r_cut = {_g(lj.r_cut)}\n",
          f"interaction.energy_shifted = {'true' if lj.energy_shifted else 'false'}\n",
          f"interaction.r_skin = {_g(c.r_skin)}\n"]
    if c.inter.fene is not None:
        o += [f"interaction.fene.k = {_g(c.inter.fene.k)}\n",
              f"interaction.fene.r_max = {_g(c.inter.fene.r_max)}\n"]
    if c.inter.angle is not None:
        o += [f"interaction.angle.k = {_g(c.inter.angle.k)}\n",
              f"interaction.angle.theta0 = {_g(c.inter.angle.theta0)}\n"]
    o.append("\n")
    o += [f"engine.dt = {_g(c.engine.dt)}\n", f"engine.steps = {c.engine.steps}\n",
          "engine.n_sub = auto\n" if c.n_sub_auto else f"engine.n_sub = {c.engine.n_sub}\n",
          f"engine.worker_threads = {c.engine.worker_threads}\n"]
    if c.engine.thermostat is not None:
        o += [f"engine.thermostat.gamma = {_g(c.engine.thermostat.gamma)}\n",
              f"engine.thermostat.temperature = {_g(c.engine.thermostat.temperature)}\n"]
    for key, val in (("engine.backend", c.gpu.backend), ("engine.gpus", c.gpu.gpus),
                     ("engine.balance", c.gpu.balance), ("engine.device", c.gpu.device)):
        if key in c.gpu.given:
            o.append(f"{key} = {val}\n")
    o.append("\n")
    if c.output.timing_path:
        o.append(f"output.timing_path = {c.output.timing_path}\n")
    o.append(f"output.timing_mode = {c.output.timing_mode}\n")
    if c.output.trajectory_path:
        o.append(f"output.trajectory_path = {c.output.trajectory_path}\n")
    o += [f"output.trajectory_stride = {c.output.trajectory_stride}\n",
          f"output.observable_stride = {c.output.observable_stride}\n",
          f"autotune.probe_steps = {c.probe_steps}\n",
          f"autotune.full_sweep = {'true' if c.full_sweep else 'false'}\n"]
    return "".join(o)


def generate_system(c: RunConfig, device: int = -1) -> E.FlatConfig:
    """generate_system (run_config.hpp:398-421) + the GPU generators."""
    s = c.system
    if s.generator == "lattice":
        if s.n < 1:
            raise ConfigError("system.n must be at least 1")
        return E.gen_lattice(s.n, s.rho, s.temperature, c.seed)
    if s.generator == "spherical":
        return E.gen_spherical(s.box_length, s.diameter_fraction, s.rho_in, s.alpha,
                               s.temperature, c.seed)
    if s.generator == "melt":
        raise ConfigError("the ring melt carries angle terms, which are not on the GPU "
                          "path; use system.generator = kg_melt (linear Kremer-Grest chains)")
    if s.generator == "random":
        if s.n < 1:
            raise ConfigError("system.n must be at least 1")
        return E.gen_random(s.n, s.rho, s.min_distance, s.temperature, c.seed)
    if s.generator == "fcc":
        if s.cells < 1:
            raise ConfigError("system.cells must be at least 1")
        return E.gen_fcc(s.cells, s.rho, s.temperature, c.seed)
    if s.generator == "fcc_slab":
        if s.cells < 1:
            raise ConfigError("system.cells must be at least 1")
        return E.gen_fcc_slab(s.cells, s.rho, s.temperature, c.seed, n=s.n or None)
    if s.generator == "kg_melt":
        if s.chains < 1:
            raise ConfigError("system.chains must be at least 1")
        if s.chain_length < 2:
            raise ConfigError("system.chain_length must be at least 2")
        f = E.gen_chains(s.chains, s.chain_length, s.rho, s.bond_length, seed=c.seed)
        if s.warmup:
            f = E.kg_warmup(f, r_skin=c.r_skin, seed=c.seed, device=device)
        return f
    raise ConfigError(f"unknown generator '{s.generator}'")


def with_overrides(c: RunConfig, threads: int = 0, seed: Optional[int] = None) -> RunConfig:
    """md_cli.cpp:46-61: --threads and --seed override the file."""
    c = copy.deepcopy(c)
    if threads > 0:
        c.engine.worker_threads = threads
    if seed is not None:
        c.seed = seed
        if c.engine.thermostat is not None:
            c.engine.thermostat.seed = seed
    return c
