"""Native slab loop (one rank, in-process NCCL) against the single-context
engine on the same 1M-particle FCC system: wall ms per step (a) on a
T = 0 perfect lattice that never rebuilds and (b) on the T = 1 liquid, and
the time of one forced rebuild. What the decomposition costs per step and
per rebuild before any second GPU exists.
python scripts/slab_overhead_probe.py [cells]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_10876_b200 import engine as E  # noqa: E402
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64


def wall(run, steps):
    t0 = time.perf_counter()
    run(steps)
    return (time.perf_counter() - t0) / steps * 1e3


for T in (0.0, 1.0):
    f = E.gen_fcc(cells, 0.8442, T, 12345)
    if T == 0.0:
        f.vel[:] = 0.0
    cfg = E.EngineConfig(dt=0.005, section_timers=False)
    one = E.Engine(f, E.Interactions(), 0.3, cfg)
    one.run(50)
    one.observe()
    t_one = wall(one.run, 400)
    r_one = one.rebuild_count()
    one.close()
    dec = DecomposedEngine(f, E.Interactions(), 0.3, cfg, comm=InProcessComm(1), native=True)
    dec.run(50)
    r0 = dec.rebuild_count()
    t_dec = wall(dec.run, 400)
    r_dec = dec.rebuild_count() - r0
    dec.close()
    print(f"T={T} n={f.size()} single {t_one:.4f} ms/step, native slab (1 rank) "
          f"{t_dec:.4f} ms/step, rebuilds in 400 steps: {r_dec}", flush=True)

# where the native loop's time goes (CUDA-event section timers, liquid)
f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
cfg = E.EngineConfig(dt=0.005, section_timers=True)
dec = DecomposedEngine(f, E.Interactions(), 0.3, cfg, comm=InProcessComm(1), native=True)
dec.run(50)
t0 = dec.timers()
r0 = dec.rebuild_count()
dec.run(400)
t1 = dec.timers()
nreb = dec.rebuild_count() - r0
d = t1.seconds - t0.seconds
print("native loop sections (ms/step): " + ", ".join(
    f"{n} {1e3 * v / 400:.4f}" for n, v in zip(E.SECTION_NAMES, d)) +
    f"; elapsed {1e3 * (t1.elapsed - t0.elapsed) / 400:.4f}; {nreb} rebuilds", flush=True)
dec.close()
one = E.Engine(f, E.Interactions(), 0.3, cfg)
one.run(50)
t0 = one.timers()
one.run(400)
t1 = one.timers()
d = t1.seconds - t0.seconds
print("single context sections (ms/step): " + ", ".join(
    f"{n} {1e3 * v / 400:.4f}" for n, v in zip(E.SECTION_NAMES, d)) +
    f"; elapsed {1e3 * (t1.elapsed - t0.elapsed) / 400:.4f}", flush=True)
