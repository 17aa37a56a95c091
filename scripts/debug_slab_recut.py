"""Debug driver: liquid-slab system through the load-aware decomposition."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E
from paper_2109_10876_b200.decomp import DecomposedEngine, InProcessComm

R = int(sys.argv[1]) if len(sys.argv) > 1 else 3
flat = E.gen_fcc_slab(8, 0.8442, 0.7, 5)
cfg = E.EngineConfig(dt=0.005, section_timers=False)
print("single", flush=True)
one = E.Engine(flat, E.Interactions(), 0.3, cfg)
print("single ok", one.list_stats(), flush=True)
one.run(20)
print("single run ok", flush=True)
dec = DecomposedEngine(flat, E.Interactions(), 0.3, cfg, comm=InProcessComm(R), balance="count")
print("dec ok", dec.recuts, dec.cuts, dec.slab_sizes(), flush=True)
try:
    dec.run(20)
    print("dec run ok", flush=True)
finally:
    dec.close()
print("dec closed", flush=True)
one.close()
print("one closed", flush=True)
