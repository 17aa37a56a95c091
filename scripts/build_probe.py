"""List build and step kernel at the BASELINE LJ sizes (equilibrated 100
steps): ms per build (time_list_build), step kernel, steady step.
python scripts/build_probe.py [cells...]"""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

for cells in [int(c) for c in (sys.argv[1:] or ["20", "64", "160"])]:
    eng = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3,
                   E.EngineConfig(dt=0.005, section_timers=False))
    eng.run(100)
    k = max(50, int(2e7 / (4 * cells ** 3)))
    r0 = eng.rebuild_count()
    t0 = time.perf_counter()
    eng.run(k)
    step = (time.perf_counter() - t0) / k * 1e3
    nreb = eng.rebuild_count() - r0
    print(f"N={4 * cells ** 3}: build {eng.time_list_build(5):.4f} ms, step kernel "
          f"{eng.time_step_kernel(10):.4f} ms, step {step:.4f} ms ({nreb} rebuilds / {k})",
          flush=True)
    eng.close()
