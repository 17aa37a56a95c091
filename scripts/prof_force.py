"""Eager (no CUDA graphs) run of the 1M config for ncu captures: 50 steps,
then 3 timed force launches and 2 list builds (the kernels ncu should see).
python scripts/prof_force.py [cells] [build kind]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
build = int(sys.argv[2]) if len(sys.argv) > 2 else 0
f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005, section_timers=True,
                                                        build=build))
eng.run(50)
print("force ms", eng.time_force_kernel(3))
print("build ms", eng.time_list_build(2))
print(eng.list_stats())
