"""Where the Kremer-Grest (configs[2]) end-to-end time goes: create phases
(TMD_DEBUG_TIMING), run_observed, flatten. python scripts/kg_e2e_probe.py [cells]"""
import os
import sys
import time
sys.path.insert(0, "/root/repo")
os.environ.setdefault("TMD_DEBUG_TIMING", "1")
import bench  # noqa: E402
from paper_2109_10876_b200 import engine as E  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = bench.Workload("kg", cells)
cfg = E.EngineConfig(dt=w.dt, section_timers=False)
E.Engine(w.flat, w.inter, w.r_skin, cfg).close()  # warm the process
for _ in range(2):
    t0 = time.perf_counter()
    e = E.Engine(w.flat, w.inter, w.r_skin, cfg)
    t1 = time.perf_counter()
    e.run_observed(200, stride=1)
    t2 = time.perf_counter()
    e.flatten()
    t3 = time.perf_counter()
    print(f"n={w.n} create {1e3*(t1-t0):.1f} ms, run_observed(200) {1e3*(t2-t1):.1f} ms, "
          f"flatten {1e3*(t3-t2):.1f} ms", flush=True)
    e.close()
