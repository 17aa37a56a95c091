"""configs[0] (32K) step split per list-build kind (graph mode, spec blocks):
python scripts/small_probe2.py [cells=20]"""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for build in (6, 3, 5):
    cfg = E.EngineConfig(dt=0.005, section_timers=False, build=build)
    liq = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3, cfg)
    liq.run(300)
    best = 1e9
    for _ in range(3):
        r0 = liq.rebuild_count()
        t0 = time.perf_counter()
        liq.run(2000)
        dt = (time.perf_counter() - t0) / 2000 * 1e3
        if dt < best:
            best, nreb = dt, liq.rebuild_count() - r0
    kc = liq.kernel_config()
    print(f"N={liq.flatten().pos.shape[0]} {kc}: liquid {best:.4f} ms/step ({nreb} rebuilds/2000), "
          f"step kernel {liq.time_step_kernel(50):.4f}, build {liq.time_list_build(20):.4f} ms",
          flush=True)
    liq.close()
cfg = E.EngineConfig(dt=0.005, section_timers=True)
liq = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3, cfg)
liq.run(300)
s0 = liq.timers()
t0 = time.perf_counter()
liq.run(2000)
el = time.perf_counter() - t0
s1 = liq.timers()
names = ["Forces", "Comm", "Integrate", "Neigh", "Resort"]
print("timers (graph mode, ms/step):",
      {k: round((s1.seconds[i] - s0.seconds[i]) / 2000 * 1e3, 5) for i, k in enumerate(names)},
      f"elapsed {(s1.elapsed - s0.elapsed) / 2000 * 1e3:.4f}, wall {el / 2000 * 1e3:.4f} ms/step")
