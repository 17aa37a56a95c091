"""Step-kernel time (fused force + integrator) of the KG melt and the LJ fluid
at 1M / 16.4M: python scripts/force_prefetch_probe.py  (A/B via TMD_LIB)."""
import sys
sys.path.insert(0, "/root/repo")
import bench
from paper_2109_10876_b200 import engine as E

flat, inter, w = bench.make_inputs_ours("kg", 64, 0)
eng = E.Engine(flat, inter, w.r_skin, E.EngineConfig(dt=w.dt, section_timers=False))
eng.run(50)
print(f"kg 4M step kernel {eng.time_step_kernel(20):.4f} ms", flush=True)
eng.close()
for cells in (64, 160):
    eng = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3,
                   E.EngineConfig(dt=0.005, section_timers=False))
    eng.run(50)
    print(f"lj {4 * cells ** 3} step kernel {eng.time_step_kernel(10):.4f} ms", flush=True)
    eng.close()
