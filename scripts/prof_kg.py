"""Eager KG run for ncu captures of its step kernel: python scripts/prof_kg.py [cells=64]"""
import sys
sys.path.insert(0, "/root/repo")
import bench
from paper_2109_10876_b200 import engine as E
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
flat, inter, w = bench.make_inputs_ours("kg", cells, 0)
eng = E.Engine(flat, inter, w.r_skin, E.EngineConfig(dt=w.dt, graphs=False, section_timers=False))
eng.run(30)
print(eng.kernel_config(), eng.list_stats())
