"""Eager (graphs=False: ncu cannot profile the kernel nodes of graphs with
conditional nodes; section timers on) run of an FCC LJ config for ncu
captures: 30 steps (every step's force launch but the last is the fused
production kernel k_forces_l1<*, kFused>), then the step-kernel and list-build
timing hooks. python scripts/prof_step.py [cells=160] [steps=30]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 160
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005, section_timers=True,
                                                        graphs=False))
eng.run(steps)
print("timers", eng.timers())
print("step kernel ms", eng.time_step_kernel(3))
print("build ms", eng.time_list_build(2))
print(eng.list_stats(), eng.kernel_config())
