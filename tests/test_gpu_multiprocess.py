"""The native slab loop with one PROCESS per rank, several ranks on one GPU.

NCCL needs one GPU per rank, so the multi-process path of the production
loop — each rank a separate process, the fused halo's peer position buffers
opened by CUDA IPC (cudaIpcGetMemHandle / cudaIpcOpenMemHandle) and written
by the force kernel's epilogue across processes, the all-gathered row tables
and ghost offsets, migration between processes — is run here over the
host-staged transport (HostFileComm, tmd_gpu_slab_attach_host): every
collective synchronises the stream first, so no kernel ever waits on another
rank's kernel and the ranks can share one GPU. Parity: the reference's golden
vectors (pair sets bit-exact, forces 1e-10, PE 1e-12, 1e-9 trajectories with
equal rebuild counts) and bitwise equality with the same decomposition run
in one process (test_engine.cpp:242-260's decomposition invariance)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm
from tests._util import E_RTOL, assert_forces_close, assert_rel, load
from tests.test_gpu_native_slab import system

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

WORKER = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2109_10876_b200.decomp import DecomposedEngine, HostFileComm
from tests._util import load
from tests.test_gpu_native_slab import system
_, name, R, rank, path, out, halo, steps, balance = sys.argv[1:]
R, rank, steps = int(R), int(rank), int(steps)
g = load(name)
flat, inter, cfg = system(g)
eng = DecomposedEngine(flat, inter, float(g["r_skin"]), cfg, comm=HostFileComm(path, rank, R),
                       native=True, halo=halo, device_of=lambda r: 0, balance=balance)
pairs = eng.local_pairs()
ids0, pos0, vel0, f0 = eng.local_state()
o = eng.observe()
eng.run(steps)
ids, pos, vel, _ = eng.local_state()
np.savez(out, pairs=pairs, ids0=ids0, f0=f0, pe=o.potential, w=o.virial, ids=ids, pos=pos,
         vel=vel, rebuilds=eng.rebuild_count(), n_own=eng.slab_sizes()[rank]["n_own"])
eng.close()
"""


def run_ranks(tmp_path, name, R, halo, steps, balance="static"):
    shm = tmp_path / "transport.bin"
    if shm.exists():
        shm.unlink()
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    procs = []
    for r in range(R):
        out = tmp_path / f"rank{r}.npz"
        procs.append((out, subprocess.Popen(
            [sys.executable, "-c", WORKER, str(ROOT), name, str(R), str(r), str(shm),
             str(out), halo, str(steps), balance], env=env, stdout=subprocess.PIPE,
            stderr=subprocess.STDOUT, text=True)))
    res = []
    for out, p in procs:
        try:
            log, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for _, q in procs:
                q.kill()
            raise
        assert p.returncode == 0, log[-3000:]
        res.append(dict(np.load(out)))
    return res


@pytest.mark.parametrize("name,R,halo,balance", [
    ("fcc8_jit", 2, "fused", "static"), ("fcc8_jit", 3, "fused", "static"),
    ("kg_lattice10", 2, "fused", "static"), ("aniso", 2, "nccl", "static"),
    ("fcc8_jit", 3, "fused", "count")])
def test_native_loop_one_process_per_rank(tmp_path, name, R, halo, balance):
    g = load(name)
    steps = int(g["steps"])
    res = run_ranks(tmp_path, name, R, halo, steps, balance)
    cat = lambda k: np.concatenate([r[k] for r in res])  # noqa: E731
    pairs = cat("pairs")
    pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
    np.testing.assert_array_equal(pairs, g["pairs"])
    o0 = np.argsort(cat("ids0"))
    np.testing.assert_array_equal(cat("ids0")[o0], np.sort(g["ids"]))
    assert_forces_close(cat("f0")[o0], g["forces"])
    assert all(r["n_own"] > 0 for r in res)  # every rank really owned a slab
    for r in res:  # observe() is a collective: every rank got the global sums
        assert_rel(float(r["pe"]), float(g["pe_fsum"]), E_RTOL, "PE")
        assert_rel(float(r["w"]), float(g["w_fsum"]), E_RTOL, "virial")
    o = np.argsort(cat("ids"))
    pos, vel = cat("pos")[o], cat("vel")[o]
    assert np.abs(pos - g["final_pos"]).max() < 1e-9
    assert np.abs(vel - g["final_vel"]).max() < 1e-9
    assert {int(r["rebuilds"]) for r in res} == {int(g["rebuilds"])}
    # the same decomposition in one process (in-process transport): bitwise
    flat, inter, cfg = system(g)
    one = DecomposedEngine(flat, inter, float(g["r_skin"]), cfg, comm=InProcessComm(R),
                           native=True, halo=halo, balance=balance)
    try:
        one.run(steps)
        ids1, pos1, vel1, _ = one.local_state()
        np.testing.assert_array_equal(ids1, cat("ids")[o])
        np.testing.assert_array_equal(pos1, pos)
        np.testing.assert_array_equal(vel1, vel)
    finally:
        one.close()


def test_bench_launches_n_ranks_through_the_native_loop(tmp_path):
    """`bench.py --gpus 2` re-launches itself under torchrun; with
    --dist-backend hostfile both ranks share GPU 0 and run the production C++
    loop as separate processes (fused halo over CUDA IPC), so the N > 1 arm of
    the bench — launch, slab engines, device timing, the e2e leg — is
    exercised on a one-GPU box. The line must carry the rank count."""
    import json
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dist-backend",
                        "hostfile", "--cells", "20", "--steps", "30", "--warmup", "5"],
                       env=env, cwd=str(tmp_path), capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["steps"] == 30 and line["value"] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert "native C++ step loop" in line["details"]["parallelism"]
    assert line["details"]["rank0_slab"]["nranks"] == 2
    assert 0 < line["details"]["rank0_slab"]["n_own"] < 32000
