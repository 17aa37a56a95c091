"""The native slab loop at R = 1, 2, 4, 8 ranks on ONE GPU (in-process
transport: every rank's context here, one host thread per rank) against the
single-context engine on the same system: ms per step over the same steps.
On one GPU the R slabs share its SMs, so R x (work per slab) = the whole
system's work: the gap to the single context is the decomposition's own
cost (per-step MAX all-reduce, halo, per-rebuild migration/ghost protocol
and host round trips, R x smaller kernels).
python scripts/slab_ranks_probe.py [cells=160] [steps=60] [ranks=1,2,4,8]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_10876_b200 import engine as E  # noqa: E402
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 160
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
ranks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4,8").split(",")]
f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
cfg = E.EngineConfig(dt=0.005, section_timers=False)
one = E.Engine(f, E.Interactions(), 0.3, cfg)
one.run(20)
r0 = one.rebuild_count()
t0 = time.perf_counter()
one.run(steps)
one.observe()
t1 = (time.perf_counter() - t0) / steps * 1e3
print(f"n={f.size()} single context: {t1:.4f} ms/step ({one.rebuild_count() - r0} rebuilds)",
      flush=True)
one.close()
E.release_cache() if hasattr(E, "release_cache") else None
for R in ranks:
    dec = DecomposedEngine(f, E.Interactions(), 0.3, cfg, comm=InProcessComm(R), native=True)
    dec.run(20)
    r0 = dec.rebuild_count()
    t0 = time.perf_counter()
    dec.run(steps)
    dec.observe()
    t = (time.perf_counter() - t0) / steps * 1e3
    print(f"R={R}: {t:.4f} ms/step ({dec.rebuild_count() - r0} rebuilds), "
          f"{t1 / t * 100:.1f} % of the single context's throughput", flush=True)
    dec.close()
