"""bench.py host logic (no GPU): the launch of N ranks, the config object both
arms print, and the reference arm's library-free inputs."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2109_10876_b200 import engine as E  # noqa: E402


def _env():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    return env


def test_gpus_flag_launches_that_many_ranks():
    # `--gpus 2` without a torchrun environment re-launches under
    # torch.distributed.run; rank 0 reports the world it joined
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, env=_env(), timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_flag"] == 2 and d["rank_sum"] == 3


def test_gpus_flag_must_match_the_launchers_world_size():
    env = _env()
    env.update(WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0
    assert "WORLD_SIZE=4" in r.stderr


def test_one_gpu_needs_no_launcher():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--launch-check"],
                       capture_output=True, text=True, env=_env(), timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 1
    assert d["config"]["n_particles"] == 16384000  # default: configs[4]
    assert "configs[4]" in d["config"]["workload"]


@pytest.mark.parametrize("kind,cells,weak,ranks", [
    ("lj", 160, False, 1), ("lj", 64, False, 2), ("lj", 20, False, 1), ("lj", 160, True, 8),
    ("kg", 64, False, 1), ("slab", 64, False, 4)])
def test_config_object_is_a_pure_function_of_the_command_line(kind, cells, weak, ranks):
    a = bench.workload_config(kind, cells, weak, ranks)
    b = bench.workload_config(kind, cells, weak, ranks)
    assert a == b
    assert json.loads(json.dumps(a)) == a
    assert "parallelism" not in a  # run-specific facts go to "details"


@pytest.mark.parametrize("cells", [1, 3, 6, 20])
def test_numpy_fcc_matches_the_engine_generator_bitwise(cells):
    box, ids, pos = bench.fcc_numpy(cells, cells, cells)
    f = E.gen_fcc(cells, bench.RHO, 1.0, bench.SEED)
    assert np.array_equal(box, f.box)
    assert np.array_equal(ids, f.id)
    assert np.array_equal(pos, f.pos)


def test_numpy_fcc_box_matches_the_engine_generator_bitwise():
    box, ids, pos = bench.fcc_numpy(4, 2, 2)
    f = E.gen_fcc_box(4, 2, 2, bench.RHO, 1.0, bench.SEED)
    assert np.array_equal(box, f.box)
    assert np.array_equal(ids, f.id)
    assert np.array_equal(pos, f.pos)


def test_reference_inputs_equal_our_inputs():
    pytest.importorskip("oracle.ref")
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = bench.make_inputs_reference("lj", 6, 0)
    f, _, _ = bench.make_inputs_ours("lj", 6, 0)
    assert np.array_equal(w.pos, f.pos) and np.array_equal(w.vel, f.vel)
    w = bench.make_inputs_reference("slab", 5, 0)
    f, _, _ = bench.make_inputs_ours("slab", 5, 0)
    assert np.array_equal(w.box, f.box)
    assert np.array_equal(w.id, f.id)
    assert np.array_equal(w.pos, f.pos) and np.array_equal(w.vel, f.vel)


def test_reference_arm_does_not_import_the_package():
    # the reference arm's process must never map libtmd_gpu.so
    code = ("import sys; sys.argv=['bench.py']; sys.path.insert(0, %r); import bench; "
            "bench.make_inputs_reference('lj', 4, 0); "
            "import sys; assert 'paper_2109_10876_b200' not in sys.modules, 'package imported'; "
            "maps = open('/proc/self/maps').read(); assert 'libtmd_gpu' not in maps; print('ok')"
            % str(ROOT))
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=_env(), timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok")


def test_cpu_reference_run_reports_sections_and_one_thread_rate():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    w = bench.make_inputs_reference("lj", 5, 0)
    c = bench.cpu_reference_run(w, 3, 1, 5.0, one_thread_budget_s=2.0)
    assert c["value"] > 0 and c["steps"] >= 1
    assert set(c["sections_s"]) == {"Forces", "Comm", "Integrate", "Neigh", "Resort"}
    assert c["sections_s"]["Forces"] > 0
    assert c["one_thread"]["value"] > 0
