"""The C-ABI library: loads, exports every symbol include/tmd_gpu.h declares,
its host-side helpers are bit-exact with the reference, and input validation
matches the reference's ConfigError cases — all without a GPU."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2109_10876_b200 import _abi
from paper_2109_10876_b200 import engine as E
from tests._util import load

HEADER = Path(__file__).resolve().parents[1] / "include" / "tmd_gpu.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(tmd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(_abi.EXPORTS) == names
    assert L.tmd_gpu_abi_version() == 4


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS and nothing else (no PTX/JIT fallback)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", str(_abi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
    ptx = subprocess.run([exe, "--list-ptx", str(_abi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert ".ptx" not in ptx


def test_host_rng_and_velocities_match_reference():
    g = load("rng")
    for k, n3, u3 in zip(g["keys"], g["normal3"], g["uniform3"]):
        k = [int(x) for x in k]
        assert np.array_equal(E.counter_normal3(*k), n3)
        assert np.array_equal(E.counter_uniform3(*k), u3)
    f = E.FlatConfig(np.ones(3), g["tv_ids"], np.zeros((len(g["tv_ids"]), 3)), None)
    E.thermal_velocities(f, 1.0, 12345)
    np.testing.assert_array_equal(f.vel, g["tv"])


def test_fcc_generator_matches_oracle_port():
    from oracle import port
    for cells in (2, 8, 20):
        f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
        box, ids, pos = port.gen_fcc(cells, 0.8442)
        np.testing.assert_array_equal(f.box, box)
        np.testing.assert_array_equal(f.id, ids)
        np.testing.assert_array_equal(f.pos, pos)
        np.testing.assert_array_equal(f.vel, port.thermal_velocities(ids, 1.0, 12345))


def _flat(n=8, box=10.0):
    rng = np.random.default_rng(0)
    return E.FlatConfig(np.full(3, box), np.arange(n), rng.uniform(0, box, (n, 3)), None)


@pytest.mark.parametrize("mutate,match", [
    (lambda f, i, c: setattr(f, "box", np.array([2.0, 10.0, 10.0])), "smaller than one cell"),
    (lambda f, i, c: setattr(f, "box", np.array([-1.0, 10.0, 10.0])), "finite and positive"),
    (lambda f, i, c: setattr(i.lj, "epsilon", 0.0), "epsilon"),
    (lambda f, i, c: setattr(i.lj, "sigma", float("nan")), "sigma"),
    (lambda f, i, c: setattr(i.lj, "r_cut", -2.5), "r_cut"),
    (lambda f, i, c: setattr(f, "id", np.array([0, 1, 2, 3, 4, 5, 6, 6])), "duplicate particle id"),
    (lambda f, i, c: setattr(f, "mass", np.array([1, 1, 1, 0.0, 1, 1, 1, 1])), "non-positive mass"),
    (lambda f, i, c: setattr(c, "dt", 0.0), "time step"),
    (lambda f, i, c: setattr(c, "thermostat", E.LangevinParams(gamma=-1.0)), "gamma"),
    (lambda f, i, c: setattr(c, "thermostat", E.LangevinParams(temperature=float("inf"))),
     "temperature"),
    (lambda f, i, c: setattr(f, "bonds", np.array([[0, 1]])), "no bond parameters"),
    (lambda f, i, c: (setattr(f, "bonds", np.array([[0, 1]])),
                      setattr(i, "fene", E.FeneParams(30.0, 3.1))), "ghost shell"),
    (lambda f, i, c: (setattr(f, "bonds", np.array([[0, 999]])),
                      setattr(i, "fene", E.FeneParams())), "unknown particle id 999"),
    (lambda f, i, c: (setattr(f, "bonds", np.array([[2, 2]])),
                      setattr(i, "fene", E.FeneParams())), "to itself"),
    (lambda f, i, c: setattr(i, "fene", E.FeneParams(k=0.0)), "fene k"),
    (lambda f, i, c: setattr(c, "force_cap", -1.0), "force cap"),
    (lambda f, i, c: setattr(i, "angle", E.AngleParams()), "angle"),
])
def test_config_errors_raise_before_touching_the_device(mutate, match):
    """validate_flat / validate_lj / build_cell_grid / validate_engine_config
    (flat_config.hpp:42-61, potentials.hpp:28-38, cell_grid.hpp:54-78,
    engine.hpp:28-41) map to ConfigError on the GPU path too."""
    f, inter, cfg = _flat(), E.Interactions(), E.EngineConfig()
    mutate(f, inter, cfg)
    with pytest.raises(E.ConfigError, match=match):
        E.Engine(f, inter, 0.3, cfg)


def test_negative_skin_rejected():
    with pytest.raises(E.ConfigError, match="skin"):
        E.Engine(_flat(), E.Interactions(), -0.1)


def test_no_cpu_fallback_without_a_device():
    """On a machine without a CUDA device a valid system fails loudly with
    CudaError instead of silently computing on the CPU."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present; covered by the -m gpu suite")
    with pytest.raises(E.CudaError):
        E.Engine(_flat(), E.Interactions(), 0.3)


def test_error_string_is_exposed_through_the_abi():
    L = _abi.lib()
    sysd = _abi.TmdSystem()
    sysd.box[:] = [1.0, 10.0, 10.0]
    ids = np.arange(2, dtype=np.int64)
    pos = np.zeros((2, 3))
    sysd.n = 2
    sysd.id = ids.ctypes.data_as(C.c_void_p)
    sysd.pos = pos.ctypes.data_as(C.c_void_p)
    lj = _abi.TmdLjParams(1.0, 1.0, 2.5, 1)
    p = _abi.TmdEngineParams()
    p.dt = 0.005
    p.r_skin = 0.3
    h = C.c_void_p()
    rc = L.tmd_gpu_create(C.byref(sysd), C.byref(lj), None, C.byref(p), C.byref(h))
    assert rc == _abi.TMD_ERR_CONFIG
    assert not h.value
    assert b"smaller than one cell" in L.tmd_gpu_last_error(None)


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors have the C structs' sizes and field offsets."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {
        "tmd_system": _abi.TmdSystem, "tmd_lj_params": _abi.TmdLjParams,
        "tmd_fene_params": _abi.TmdFeneParams,
        "tmd_engine_params": _abi.TmdEngineParams, "tmd_observables": _abi.TmdObservables,
        "tmd_list_stats": _abi.TmdListStats,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             'int main(void) {']
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ['  return 0;', '}']
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, str(src), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    import ctypes
    for line in got.splitlines():
        cname, field, val = line.split()
        cls = structs[cname]
        want = ctypes.sizeof(cls) if field == "size" else getattr(cls, field).offset
        assert int(val) == want, (cname, field, int(val), want)


def test_fcc_box_generator():
    """gen_fcc_box: a cube is gen_fcc bit for bit; an elongated box continues
    the same lattice (its first half is the cube's) at 4 particles per cell."""
    cube = E.gen_fcc(5, 0.8442, 1.0, 7)
    same = E.gen_fcc_box(5, 5, 5, 0.8442, 1.0, 7)
    np.testing.assert_array_equal(cube.pos, same.pos)
    np.testing.assert_array_equal(cube.vel, same.vel)
    long = E.gen_fcc_box(5, 5, 10, 0.8442, 1.0, 7)
    assert long.size() == 2 * cube.size()
    np.testing.assert_allclose(long.pos[: cube.size()], cube.pos, rtol=1e-15, atol=1e-14)
    np.testing.assert_allclose(long.box, [cube.box[0], cube.box[1], 2 * cube.box[2]],
                               rtol=1e-15)
    rho = long.size() / np.prod(long.box)
    assert abs(rho - 0.8442) < 1e-12
    assert abs(long.vel.sum(axis=0)).max() < 1e-9  # zero net momentum


def test_local_group_handle_lifecycle():
    """tmd_local_group_create / _destroy (the in-process transport of the
    native slab loop) need no device."""
    import ctypes as C
    L = _abi.lib()
    g = C.c_void_p()
    assert L.tmd_local_group_create(0, C.byref(g)) == _abi.TMD_ERR_CONFIG
    assert L.tmd_local_group_create(4, C.byref(g)) == _abi.TMD_OK and g.value
    L.tmd_local_group_destroy(g)


@pytest.mark.parametrize("mutate,match", [
    # build_domain runs validate_flat before validate_lj (domain.hpp:137-141)
    (lambda f, i: (setattr(f, "id", np.array([0, 1, 2, 3, 4, 5, 6, 6])),
                   setattr(i.lj, "epsilon", 0.0)), "duplicate particle id 6"),
    # the first failing particle in input order: a mass at index 3 before a
    # duplicate at index 7 (flat_config.hpp:50-58)
    (lambda f, i: (setattr(f, "id", np.array([0, 1, 2, 3, 4, 5, 6, 6])),
                   setattr(f, "mass", np.array([1, 1, 1, 0.0, 1, 1, 1, 1.0]))),
     "id 3 has non-positive mass"),
    (lambda f, i: (setattr(f, "id", np.array([0, 1, 2, 2, 4, 5, 6, 7])),
                   setattr(f, "mass", np.array([1, 1, 1, 1, 1, 1, 1, 0.0]))),
     "duplicate particle id 2"),
    # sparse ids take the hash-set path
    (lambda f, i: setattr(f, "id", np.array([10, 900, 7, 55, 3, 900, 1, 2])),
     "duplicate particle id 900"),
    # the box comes first of all (validate_box inside validate_flat)
    (lambda f, i: (setattr(f, "box", np.array([-1.0, 10.0, 10.0])),
                   setattr(f, "id", np.array([0, 1, 2, 3, 4, 5, 6, 6]))), "finite and positive"),
])
def test_config_error_order_follows_build_domain(mutate, match):
    f, inter = _flat(), E.Interactions()
    mutate(f, inter)
    with pytest.raises(E.ConfigError, match=match):
        E.Engine(f, inter, 0.3, E.EngineConfig())


def test_parallel_validation_names_the_first_duplicate():
    """Large systems validate on host threads; the reported id is still the
    reference's (the first repeated id in input order)."""
    n = 3 << 20
    ids = np.arange(n, dtype=np.int64)
    ids[2_000_000] = 1_500_000
    ids[2_500_000] = 700
    f = E.FlatConfig(np.full(3, 200.0), ids, np.zeros((n, 3)), None)
    with pytest.raises(E.ConfigError, match="duplicate particle id 1500000"):
        E.Engine(f, E.Interactions(), 0.3, E.EngineConfig())
