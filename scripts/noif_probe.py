"""Graph step overhead by system size: a T = 0 perfect lattice (no rebuilds)
and the liquid (rebuild every ~9 steps), with IF nodes vs early-returning
rebuild kernel nodes (TMD_IF_NODES=1/0). python scripts/noif_probe.py"""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E


def steady(eng, k):
    eng.run(300)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        eng.run(k)
        best = min(best, (time.perf_counter() - t0) / k * 1e3)
    return best


for cells in [int(c) for c in (sys.argv[1:] or ["20", "32", "40", "64"])]:
    k = max(200, int(3e7 / (4 * cells ** 3)))
    f = E.gen_fcc(cells, 0.8442, 0.0, 12345)
    f.vel[:] = 0.0
    cold = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005, section_timers=False))
    liq = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3,
                   E.EngineConfig(dt=0.005, section_timers=False))
    print(f"N={4 * cells ** 3}: cold step {steady(cold, k):.5f} ms, liquid step "
          f"{steady(liq, k):.5f} ms, step kernel {cold.time_step_kernel(50):.5f} ms", flush=True)
    cold.close()
    liq.close()
