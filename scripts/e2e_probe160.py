"""The bench's e2e sequence at configs[4] (16.4M), split into phases, with the
create() phase marks (TMD_DEBUG_TIMING). python scripts/e2e_probe160.py [cells]"""
import os
import sys
import time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 160
steps = 20
t0 = time.perf_counter()
f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
print(f"gen {time.perf_counter() - t0:.2f} s", flush=True)
cfg = E.EngineConfig(dt=0.005, section_timers=False)
e = E.Engine(f, E.Interactions(), 0.3, cfg)   # the bench's device-timed engine
e.run(5)
e.close()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
fp = E.FlatConfig(f.box, pin(f.id), pin(f.pos), pin(f.vel))
n = f.size()
out = E.FlatConfig(f.box, torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(),
                   torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy(),
                   torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy())
torch.cuda.synchronize()
os.environ["TMD_DEBUG_TIMING"] = "1"
for rep in range(2):
    t0 = time.perf_counter()
    e3 = E.Engine(fp, E.Interactions(), 0.3, cfg)
    t1 = time.perf_counter()
    e3.run_observed(steps, stride=1)
    t2 = time.perf_counter()
    e3.flatten(out=out)
    t3 = time.perf_counter()
    e3.close()
    print(f"e2e split #{rep}: create {1e3*(t1-t0):.1f} ms, run_observed({steps}) "
          f"{1e3*(t2-t1):.1f} ms, flatten {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms",
          flush=True)
