"""ctypes binding of include/tmd_gpu.h (libtmd_gpu.so).

This is the only place the package touches the shared library. Loading fails
loudly when the library is missing — there is no CPU fallback anywhere in the
product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtmd_gpu.so"
if os.environ.get("TMD_LIB"):  # A/B experiments against another build of the library
    LIB_PATH = Path(os.environ["TMD_LIB"]).resolve()

TMD_OK = 0
TMD_ERR_CONFIG = 1
TMD_ERR_PHYSICS = 2
TMD_ERR_VERIFY = 3
TMD_ERR_STATE = 4
TMD_ERR_CUDA = 5

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = [
    "tmd_gpu_create", "tmd_gpu_last_error", "tmd_gpu_compute_forces",
    "tmd_gpu_step", "tmd_gpu_observe", "tmd_gpu_download",
    "tmd_gpu_set_velocities", "tmd_gpu_cell_of", "tmd_gpu_pairs",
    "tmd_gpu_timers", "tmd_gpu_rebuild_count", "tmd_gpu_step_count",
    "tmd_gpu_size", "tmd_gpu_list_stats", "tmd_gpu_time_force_kernel",
    "tmd_gpu_stream", "tmd_gpu_destroy", "tmd_gen_fcc",
    "tmd_thermal_velocities", "tmd_counter_uniform3", "tmd_counter_normal3",
    "tmd_gpu_abi_version", "tmd_gpu_launch_count", "tmd_gpu_fp64_peak",
    "tmd_gpu_kernel_config", "tmd_gpu_slab_run_observed",
    "tmd_gpu_time_list_build",
    "tmd_gpu_create_slab", "tmd_gpu_slab_info", "tmd_gpu_slab_max_d2",
    "tmd_gpu_slab_decide", "tmd_gpu_slab_migrate_out", "tmd_gpu_slab_migrate_in",
    "tmd_gpu_slab_commit", "tmd_gpu_slab_border", "tmd_gpu_slab_ghost_in",
    "tmd_gpu_slab_ghosts_ready", "tmd_gpu_slab_kick_drift", "tmd_gpu_slab_forces",
    "tmd_gpu_slab_halo", "tmd_gpu_slab_sums", "tmd_gpu_slab_layer_counts",
    "tmd_gpu_slab_recut", "tmd_gen_chains", "tmd_gpu_brute_force", "tmd_gen_lattice",
    "tmd_gen_spherical", "tmd_gen_random", "tmd_gpu_run_observed", "tmd_nccl_unique_id",
    "tmd_gpu_slab_attach_nccl", "tmd_gpu_slab_setup", "tmd_gpu_slab_run",
    "tmd_gpu_slab_observe", "tmd_balanced_cuts", "tmd_gpu_release_cache",
    "tmd_gpu_time_step_kernel", "tmd_gpu_prepare_graphs",
    "tmd_local_group_create", "tmd_local_group_destroy", "tmd_gpu_slab_attach_local",
    "tmd_gpu_slab_attach_host",
    "tmd_gpu_build_pair_index_list", "tmd_gpu_pair_index_list", "tmd_gpu_compute_forces_pairs",
    "tmd_gpu_time_pair_traversal",
]


class TmdSystem(C.Structure):
    _fields_ = [
        ("box", C.c_double * 3),
        ("n", C.c_int64),
        ("id", C.c_void_p),
        ("type", C.c_void_p),
        ("mass", C.c_void_p),
        ("pos", C.c_void_p),
        ("vel", C.c_void_p),
        ("n_bonds", C.c_int64),
        ("bonds", C.c_void_p),
    ]


class TmdLjParams(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("sigma", C.c_double),
                ("r_cut", C.c_double), ("energy_shifted", C.c_int)]


class TmdFeneParams(C.Structure):
    _fields_ = [("k", C.c_double), ("r_max", C.c_double)]


class TmdEngineParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("r_skin", C.c_double),
                ("device", C.c_int), ("section_timers", C.c_int),
                ("nbr_capacity", C.c_int), ("reserved", C.c_int * 5),
                ("thermostat", C.c_int), ("gamma", C.c_double),
                ("temperature", C.c_double), ("seed", C.c_uint64),
                ("force_cap", C.c_double)]


class TmdObservables(C.Structure):
    _fields_ = [("step", C.c_int64), ("kinetic", C.c_double),
                ("potential", C.c_double), ("virial", C.c_double),
                ("temperature", C.c_double)]


class TmdListStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("entries", C.c_int64), ("in_cut", C.c_int64),
                ("max_count", C.c_int32), ("capacity", C.c_int32),
                ("dims", C.c_int32 * 3), ("cell_len", C.c_double * 3)]


_lib = None


def lib() -> C.CDLL:
    """Load libtmd_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2109_10876_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    L.tmd_gpu_create.argtypes = [C.POINTER(TmdSystem), C.POINTER(TmdLjParams),
                                 C.POINTER(TmdFeneParams), C.POINTER(TmdEngineParams),
                                 C.POINTER(P)]
    L.tmd_gpu_create.restype = C.c_int
    L.tmd_gpu_create_slab.argtypes = [C.POINTER(TmdSystem), C.POINTER(TmdLjParams),
                                      C.POINTER(TmdFeneParams), C.POINTER(TmdEngineParams),
                                      C.c_int, C.c_int, C.POINTER(P)]
    PP = C.POINTER(P)
    L.tmd_gpu_slab_info.argtypes = [P, P]
    L.tmd_gpu_slab_max_d2.argtypes = [P, C.POINTER(C.c_double)]
    L.tmd_gpu_slab_decide.argtypes = [P, C.c_int, C.c_int]
    L.tmd_gpu_slab_migrate_out.argtypes = [P, P, PP]
    L.tmd_gpu_slab_migrate_in.argtypes = [P, C.c_int64, PP]
    L.tmd_gpu_slab_commit.argtypes = [P, P]
    L.tmd_gpu_slab_border.argtypes = [P, C.c_int, PP, PP, PP]
    L.tmd_gpu_slab_ghost_in.argtypes = [P, C.c_int64, C.c_int64, PP, PP]
    L.tmd_gpu_slab_ghosts_ready.argtypes = [P]
    L.tmd_gpu_slab_kick_drift.argtypes = [P]
    L.tmd_gpu_slab_forces.argtypes = [P, C.c_int]
    L.tmd_gpu_slab_halo.argtypes = [P, PP, PP]
    L.tmd_gpu_slab_sums.argtypes = [P, P]
    L.tmd_gpu_slab_layer_counts.argtypes = [P, P]
    L.tmd_nccl_unique_id.argtypes = [P]
    L.tmd_balanced_cuts.argtypes = [P, C.c_int, C.c_int, P]
    L.tmd_gpu_slab_attach_nccl.argtypes = [P, P, C.c_int]
    L.tmd_local_group_create.argtypes = [C.c_int, PP]
    L.tmd_local_group_destroy.argtypes = [P]
    L.tmd_local_group_destroy.restype = None
    L.tmd_gpu_slab_attach_local.argtypes = [P, P, C.c_int]
    L.tmd_gpu_slab_attach_host.argtypes = [P, C.c_char_p, C.c_int]
    L.tmd_gpu_slab_setup.argtypes = [P]
    L.tmd_gpu_slab_run.argtypes = [P, C.c_int64]
    L.tmd_gpu_slab_observe.argtypes = [P, C.c_int64, C.POINTER(TmdObservables)]
    L.tmd_gpu_slab_run_observed.argtypes = [P, C.c_int64, C.c_int64,
                                            C.POINTER(TmdObservables), C.c_int64,
                                            C.POINTER(C.c_int64)]
    L.tmd_gpu_slab_recut.argtypes = [P, P]
    L.tmd_gpu_last_error.argtypes = [P]
    L.tmd_gpu_last_error.restype = C.c_char_p
    L.tmd_gpu_compute_forces.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.tmd_gpu_step.argtypes = [P, C.c_int64]
    L.tmd_gpu_observe.argtypes = [P, C.POINTER(TmdObservables)]
    L.tmd_gpu_run_observed.argtypes = [P, C.c_int64, C.c_int64, C.POINTER(TmdObservables),
                                       C.c_int64, C.POINTER(C.c_int64)]
    L.tmd_gpu_download.argtypes = [P, P, P, P, P, P, P]
    L.tmd_gpu_set_velocities.argtypes = [P, P, P]
    L.tmd_gpu_cell_of.argtypes = [P, P, P]
    L.tmd_gpu_pairs.argtypes = [P, P, C.c_size_t, C.POINTER(C.c_size_t)]
    L.tmd_gpu_timers.argtypes = [P, P, C.POINTER(C.c_double)]
    L.tmd_gpu_rebuild_count.argtypes = [P]
    L.tmd_gpu_rebuild_count.restype = C.c_uint64
    L.tmd_gpu_step_count.argtypes = [P]
    L.tmd_gpu_step_count.restype = C.c_int64
    L.tmd_gpu_size.argtypes = [P]
    L.tmd_gpu_size.restype = C.c_int64
    L.tmd_gpu_list_stats.argtypes = [P, C.POINTER(TmdListStats)]
    L.tmd_gpu_time_force_kernel.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    L.tmd_gpu_build_pair_index_list.argtypes = [P, C.POINTER(C.c_int64)]
    L.tmd_gpu_pair_index_list.argtypes = [P, P, C.c_size_t, C.POINTER(C.c_size_t)]
    L.tmd_gpu_compute_forces_pairs.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.tmd_gpu_time_pair_traversal.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    L.tmd_gpu_time_step_kernel.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    L.tmd_gpu_prepare_graphs.argtypes = [P, C.c_int64]
    L.tmd_gpu_time_list_build.argtypes = [P, C.c_int, C.POINTER(C.c_double)]
    L.tmd_gpu_stream.argtypes = [P]
    L.tmd_gpu_stream.restype = P
    L.tmd_gpu_kernel_config.argtypes = [P, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]
    L.tmd_gpu_kernel_config.restype = None
    L.tmd_gpu_launch_count.argtypes = [P]
    L.tmd_gpu_launch_count.restype = C.c_uint64
    L.tmd_gpu_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.tmd_gpu_destroy.argtypes = [P]
    L.tmd_gpu_destroy.restype = None
    L.tmd_gpu_release_cache.argtypes = []
    L.tmd_gpu_release_cache.restype = None
    L.tmd_gen_fcc.argtypes = [C.c_int, C.c_double, C.c_double, P, P, P]
    L.tmd_gpu_brute_force.argtypes = [C.POINTER(TmdSystem), C.POINTER(TmdLjParams), C.c_double,
                                      C.c_int, P, P, P, C.c_size_t, C.POINTER(C.c_size_t)]
    L.tmd_gen_lattice.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, P, P, P, P]
    L.tmd_gen_spherical.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_uint64, P, P, P, P, P]
    L.tmd_gen_random.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                 P, P, P, P]
    L.tmd_gen_chains.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                 P, P, P, P]
    L.tmd_thermal_velocities.argtypes = [C.c_int64, P, P, C.c_double, C.c_uint64, P]
    L.tmd_thermal_velocities.restype = None
    for name in ("tmd_counter_uniform3", "tmd_counter_normal3"):
        f = getattr(L, name)
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, P]
        f.restype = None
    _lib = L
    return L
