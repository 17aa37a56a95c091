"""Engine create/close cycles at 1M (TMD_DEBUG_TIMING=1 prints create's
phases): how much of create is device-memory mapping."""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E
import torch

f = E.gen_fcc(64, 0.8442, 1.0, 12345)
cfg = E.EngineConfig(dt=0.005, section_timers=False)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    t0 = time.perf_counter()
    e = E.Engine(f, E.Interactions(), 0.3, cfg)
    t1 = time.perf_counter()
    e.run(10)
    e.close()
    t2 = time.perf_counter()
    free, total = torch.cuda.mem_get_info()
    print(f"cycle {k}: create {1e3*(t1-t0):.1f} ms, run(10)+close {1e3*(t2-t1):.1f} ms, "
          f"free {free / 2**30:.2f} GiB", flush=True)
