"""Where a configs[0] (32K) step goes: the graph step without rebuilds (T = 0
perfect lattice), the liquid step (rebuild every ~9 steps), the fused step
kernel, the list build, and the per-rebuild surcharge.
python scripts/small_probe.py [cells=20]"""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E


def steady(eng, k=2000, reps=3):
    eng.run(300)
    best = 1e9
    for _ in range(reps):
        r0 = eng.rebuild_count()
        t0 = time.perf_counter()
        eng.run(k)
        dt = (time.perf_counter() - t0) / k * 1e3
        if dt < best:
            best, nreb = dt, eng.rebuild_count() - r0
    return best, nreb


cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for lanes in (0, 1, 2, 4):
    f = E.gen_fcc(cells, 0.8442, 0.0, 12345)
    f.vel[:] = 0.0
    cfg = E.EngineConfig(dt=0.005, section_timers=False, lanes=lanes)
    cold = E.Engine(f, E.Interactions(), 0.3, cfg)
    t_cold, _ = steady(cold)
    liq = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3, cfg)
    t_liq, nreb = steady(liq)
    kc = liq.kernel_config()
    t_force = liq.time_force_kernel(50)
    t_step = liq.time_step_kernel(50)
    t_build = liq.time_list_build(20)
    per_rebuild = (t_liq - t_cold) * 2000 / max(nreb, 1)
    print(f"N={f.size()} lanes={kc['lanes']} build_kind={kc['build_kind']}: step no-rebuild "
          f"{t_cold:.4f} ms, liquid {t_liq:.4f} ms ({nreb} rebuilds/2000), step kernel "
          f"{t_step:.4f}, forces-only {t_force:.4f}, build {t_build:.4f}, surcharge per rebuild "
          f"{per_rebuild:.4f} ms", flush=True)
    cold.close()
    liq.close()
