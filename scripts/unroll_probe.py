"""Step kernel (k_forces_l1<unroll, kFused>) by gathers in flight per thread."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E
for cells in (64, 160):
    for unroll in (1, 2, 4):
        eng = E.Engine(E.gen_fcc(cells, 0.8442, 1.0, 12345), E.Interactions(), 0.3,
                       E.EngineConfig(dt=0.005, section_timers=False, unroll=unroll))
        eng.run(50)
        print(f"lj {4 * cells ** 3} unroll {unroll} step kernel {eng.time_step_kernel(10):.4f} ms", flush=True)
        eng.close()
