"""Per-step cost without rebuilds: a perfect FCC lattice at T = 0 never moves
(forces cancel by symmetry), so run(K) on it times the graph's step (decide +
conditional + fused force/integrate kernel) with no list build; compared with
the forces-only kernel. python scripts/step_probe.py [cells]"""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
f = E.gen_fcc(cells, 0.8442, 0.0, 12345)
f.vel[:] = 0.0
eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005, section_timers=False))
eng.run(300)
import ctypes as C
t = []
for _ in range(3):
    t0 = time.perf_counter()
    eng.run(1000)
    t.append((time.perf_counter() - t0) / 1000 * 1e3)
print(f"N={f.size()} rebuilds={eng.rebuild_count()} step ms (graph, no rebuild) "
      f"{min(t):.4f}; forces-only kernel {eng.time_force_kernel(20):.4f} ms; "
      f"build {eng.time_list_build(5):.4f} ms")
