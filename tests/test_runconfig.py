"""Run-config front end on CPU: the parser mirrors
run_config.hpp (the reference's test_config_io.cpp cases), the generators
match the reference's own output bit for bit (tests/golden/generators.npz,
made by oracle/make_golden.py from the reference headers), and the writers
keep io.hpp's formats."""
from __future__ import annotations

import io

import numpy as np
import pytest

from paper_2109_10876_b200 import cli, engine as E
from paper_2109_10876_b200.runconfig import (generate_system, parse_run_config,
                                             serialize_run_config)
from tests._util import load

FULL = """# bulk fluid benchmark
seed = 12345

system.generator = lattice
system.n = 4000
system.rho = 0.8442
system.temperature = 0.72

interaction.epsilon = 1.0
interaction.sigma = 1.0
interaction.r_cut = 2.5
interaction.energy_shifted = true
interaction.r_skin = 0.3

engine.dt = 0.005
engine.steps = 100
engine.n_sub = auto
engine.worker_threads = 4
engine.thermostat.gamma = 1.0
engine.thermostat.temperature = 0.72

output.timing_path = timings.csv
output.timing_mode = per_step
output.trajectory_path = traj.xyz
output.trajectory_stride = 50
output.observable_stride = 10

autotune.probe_steps = 12
autotune.full_sweep = true
"""


def test_full_configuration_parses_field_by_field():
    c = parse_run_config(FULL)
    assert c.seed == 12345 and c.system.generator == "lattice" and c.system.n == 4000
    assert c.system.rho == 0.8442 and c.system.temperature == 0.72
    assert (c.inter.lj.epsilon, c.inter.lj.sigma, c.inter.lj.r_cut) == (1.0, 1.0, 2.5)
    assert c.inter.lj.energy_shifted and c.r_skin == 0.3
    assert c.inter.fene is None and c.inter.angle is None
    assert c.engine.dt == 0.005 and c.engine.steps == 100 and c.n_sub_auto
    assert c.engine.worker_threads == 4
    th = c.engine.thermostat
    assert (th.gamma, th.temperature, th.seed) == (1.0, 0.72, 12345)
    assert c.output.timing_path == "timings.csv" and c.output.timing_mode == "per_step"
    assert c.output.trajectory_path == "traj.xyz" and c.output.trajectory_stride == 50
    assert c.output.observable_stride == 10 and c.engine.observable_stride == 10
    assert c.probe_steps == 12 and c.full_sweep


def test_serialize_round_trip_is_a_fixed_point():
    c = parse_run_config(FULL)
    text = serialize_run_config(c)
    back = parse_run_config(text)
    assert serialize_run_config(back) == text
    assert back.system == c.system and back.output == c.output


def test_melt_defaults_its_bonded_parameters():
    c = parse_run_config("seed = 7\nsystem.generator = melt\nsystem.chains = 5\n"
                         "system.chain_length = 20\nsystem.rho = 0.85\n")
    assert (c.inter.fene.k, c.inter.fene.r_max) == (30.0, 1.5)
    assert (c.inter.angle.k, c.inter.angle.theta0) == (1.0, 0.0)
    back = parse_run_config(serialize_run_config(c))
    assert back.system == c.system


def test_explicit_n_sub_stays_numeric():
    c = parse_run_config("seed = 1\nsystem.generator = random\nsystem.n = 100\n"
                         "system.rho = 0.5\nsystem.temperature = 0.5\nengine.n_sub = 8\n")
    assert not c.n_sub_auto and c.engine.n_sub == 8 and c.system.min_distance == 0.8
    assert parse_run_config(serialize_run_config(c)).engine.n_sub == 8


@pytest.mark.parametrize("text,needles", [
    ("seed = 1\nbogus.key = 3\n", ["line 2", "bogus.key"]),
    ("seed 1\n", ["line 1"]),
    ("seed = 1\nseed = 2\n", ["duplicate", "seed"]),
    ("seed = 1\nengine.dt = fast\n", ["engine.dt", "fast"]),
    ("output.timing_mode = sometimes\n", ["summary or per_step"]),
    ("system.generator = lattice\nsystem.n = 10\nsystem.rho = 0.5\n", ["system.temperature"]),
    ("system.generator = lattice\nsystem.n = 10\nsystem.rho = 0.5\nsystem.temperature = 1.0\n"
     "engine.thermostat.gamma = 1.0\n", ["together"]),
    ("system.generator = maxwell\n", ["maxwell"]),
    ("system.generator = lattice\nsystem.n = 10\nsystem.rho = 0.5\nsystem.temperature = 1.0\n"
     "engine.dt = 0.0\n", ["engine.dt"]),
    ("seed = -1\n", ["seed", "non-negative integer"]),
    ("seed = 1\nsystem.n = 1.5\n", ["system.n", "integer"]),
    ("seed = 1\nsystem.rho = +1\n", ["system.rho"]),
    ("seed = 1\ninteraction.energy_shifted = yes\n", ["true or false"]),
    ("seed = 1\nengine.backend = cpu\n", ["engine.backend"]),
    ("seed = 1\nengine.balance = magic\n", ["static or count"]),
])
def test_parse_errors_cite_the_line_and_the_key(text, needles):
    with pytest.raises(E.ConfigError) as ei:
        parse_run_config(text)
    for n in needles:
        assert n in str(ei.value)


def test_comments_blank_lines_and_spacing_are_tolerated():
    c = parse_run_config("# leading comment\n\n   seed   =   9   \nsystem.generator = lattice\n"
                         "system.n=10\nsystem.rho = 0.5\n\t system.temperature = 1.0\n"
                         "# trailing comment\n")
    assert c.seed == 9 and c.system.n == 10 and c.system.temperature == 1.0


def test_gpu_keys_round_trip_and_stay_absent_otherwise():
    base = "seed = 3\nsystem.generator = fcc\nsystem.cells = 4\nsystem.rho = 0.8442\n" \
           "system.temperature = 1.0\n"
    assert "engine.gpus" not in serialize_run_config(parse_run_config(base))
    c = parse_run_config(base + "engine.gpus = 4\nengine.balance = count\nengine.backend = gpu\n")
    assert (c.gpu.gpus, c.gpu.balance) == (4, "count")
    text = serialize_run_config(c)
    assert "engine.gpus = 4" in text and "engine.balance = count" in text
    assert serialize_run_config(parse_run_config(text)) == text


def test_generated_systems_follow_the_config():
    c = parse_run_config("seed = 3\nsystem.generator = random\nsystem.n = 40\n"
                         "system.rho = 0.4\nsystem.temperature = 0.5\n")
    assert generate_system(c).size() == 40
    c = parse_run_config("seed = 3\nsystem.generator = melt\nsystem.chains = 2\n"
                         "system.chain_length = 8\nsystem.rho = 0.6\n")
    with pytest.raises(E.ConfigError, match="kg_melt"):
        generate_system(c)  # ring melts carry angle terms: not on the GPU path
    c = parse_run_config("seed = 3\nsystem.generator = kg_melt\nsystem.chains = 2\n"
                         "system.chain_length = 8\nsystem.rho = 0.6\nsystem.warmup = false\n")
    m = generate_system(c)
    assert m.size() == 16 and len(m.bonds) == 14


GEN = [("lat100", lambda: E.gen_lattice(100, 0.8442, 0.72, 3)),
       ("lat1000", lambda: E.gen_lattice(1000, 0.5, 1.0, 12345)),
       ("lat9", lambda: E.gen_lattice(9, 0.1, 0.0, 1)),
       ("rnd200", lambda: E.gen_random(200, 0.8442, 0.8, 0.72, 1)),
       ("rnd50", lambda: E.gen_random(50, 0.3, 1.0, 0.0, 99)),
       ("sph", lambda: E.gen_spherical(14.0, 0.7, 0.8442, 0.1, 0.1, 7)),
       ("sph_full", lambda: E.gen_spherical(9.0, 1.0, 0.6, 1.0, 0.5, 2))]


@pytest.mark.parametrize("tag,make", GEN)
def test_generators_match_the_reference_bitwise(tag, make):
    g = load("generators")
    f = make()
    np.testing.assert_array_equal(f.box, g[f"{tag}_box"])
    np.testing.assert_array_equal(f.id, g[f"{tag}_ids"])
    np.testing.assert_array_equal(f.pos, g[f"{tag}_pos"])
    np.testing.assert_array_equal(f.vel, g[f"{tag}_vel"])


def test_generator_argument_errors():
    with pytest.raises(E.ConfigError, match="at least 1 particle"):
        E.gen_lattice(0, 0.8, 1.0, 1)
    with pytest.raises(E.ConfigError, match="diameter fraction"):
        E.gen_spherical(10.0, 1.5, 0.8, 0.1, 1.0, 1)
    with pytest.raises(E.ConfigError, match="density too high"):
        E.gen_random(30, 2.0, 1.2, 1.0, 1)


def test_xyz_frames_carry_step_box_and_rows():
    f = E.FlatConfig(np.full(3, 6.0), np.arange(3), np.array([[0.5 + k, 1.5, 2.25]
                                                              for k in range(3)]), None,
                     type=np.arange(3) % 2)
    s = io.StringIO()
    cli.write_xyz_frame(s, f, 42)
    lines = s.getvalue().splitlines()
    assert lines[0] == "3" and lines[1] == "step=42 box=6 6 6"
    assert lines[2:] == ["0 0.5 1.5 2.25", "1 1.5 1.5 2.25", "0 2.5 1.5 2.25"]


def test_per_step_timing_file(tmp_path):
    p = tmp_path / "t.csv"
    w = cli.TimingWriter(str(p), True)
    d = np.array([0.25, 0, 0, 0, 0])
    w.record_step(1, d)
    w.record_step(2, d)
    w.finish(2, E.SectionTimers(np.array([0.5, 0, 0, 0, 0]), 0.625))
    lines = p.read_text().splitlines()
    assert len(lines) == 1 + 2 * 5 + 5 + 1 and lines[0] == "step_range,section,seconds"
    assert lines[1] == "0-1,Forces,0.25" and lines[6].startswith("1-2,Forces")
    assert lines[11] == "0-2,Forces,0.5" and lines[-1] == "0-2,Elapsed,0.625"


def test_cli_config_errors_exit_1(tmp_path, capsys):
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("seed = 1\nbogus = 2\n")
    assert cli.main(["run", "--config", str(cfg)]) == cli.EXIT_CONFIG
    assert "config error" in capsys.readouterr().err
    assert cli.main(["run", "--config", str(tmp_path / "missing.cfg")]) == cli.EXIT_CONFIG
    assert cli.main(["run"]) == cli.EXIT_CONFIG


def test_cli_generate_writes_system_and_resolved_config(tmp_path):
    cfg = tmp_path / "lat.cfg"
    cfg.write_text("seed = 5\nsystem.generator = lattice\nsystem.n = 27\nsystem.rho = 0.5\n"
                   "system.temperature = 0.3\n")
    out = tmp_path / "out"
    assert cli.main(["generate", "--config", str(cfg), "--out", str(out)]) == 0
    lines = (out / "system.xyz").read_text().splitlines()
    assert lines[0] == "27" and len(lines) == 29
    back = parse_run_config((out / "resolved.cfg").read_text())
    assert back.system.n == 27 and back.seed == 5
