"""Eager (timed sections, no graphs) run of a bench workload for ncu launch
lists: python scripts/prof_config.py <lj|kg|slab> <cells> [steps] [build kind]."""
import sys
sys.path.insert(0, "/root/repo")
import bench
from paper_2109_10876_b200 import engine as E

kind, cells = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
build = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = bench.Workload(kind, cells)
eng = E.Engine(w.flat, w.inter, w.r_skin, E.EngineConfig(dt=w.dt, section_timers=True, build=build))
eng.run(steps)
t = eng.timers()
print("sections", dict(zip(E.SECTION_NAMES, t.seconds.round(5).tolist())), "elapsed", t.elapsed)
print("rebuilds", eng.rebuild_count(), "force ms", eng.time_force_kernel(3),
      "build ms", eng.time_list_build(2))
print(eng.list_stats())
