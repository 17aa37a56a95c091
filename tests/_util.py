"""Shared helpers for the parity tests (tolerances are the north star's)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

SYSTEMS = ["jit6_s101", "jit6_s41_T08", "random500_s1", "random500_s2", "random500_s3",
           "fcc8_jit", "aniso", "thin"]

# Tolerances (BASELINE.json north_star): forces 1e-10 relative, energies and
# virial 1e-12 relative, neighbour sets and cells bit-exact. "Relative" for
# forces is against max(max|F_ref|, rms(F_ref)) because near-lattice forces
# vanish by symmetry (SURVEY §7 "Relative force tolerance near zero").
F_RTOL = 1e-10
E_RTOL = 1e-12


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def load_json(name: str):
    return json.loads((GOLDEN / name).read_text())


def force_scale(f_ref: np.ndarray) -> float:
    return max(float(np.abs(f_ref).max()), float(np.sqrt((f_ref ** 2).mean())))


def assert_forces_close(f, f_ref, rtol=F_RTOL, what="forces"):
    scale = force_scale(f_ref)
    err = float(np.abs(np.asarray(f) - f_ref).max())
    assert err <= rtol * max(scale, 1e-300), (
        f"{what}: max |dF| = {err:.3e} > {rtol:g} * {scale:.3e}")


def assert_rel(x, ref, rtol, what):
    err = abs(x - ref) / max(abs(ref), 1e-300)
    assert err <= rtol, f"{what}: {x!r} vs {ref!r} (rel {err:.2e} > {rtol:g})"
