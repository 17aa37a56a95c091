"""Threads per particle of the variant-3 force kernel (k_forces_lanes) across
system sizes (one GPU).

    python scripts/lanes_probe.py [--cells 20,32,40,64] [--lanes 1,2,4,8]

For each FCC size and lane count: an engine from the same state, 100 warm-up
steps, the force kernel timed with CUDA events (mean of 50 launches), then
the wall time of 500 steps (run() returns after the device finished). PE and
forces are compared with the one-lane engine (summation-order differences)."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_10876_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", default="20,32,40,64")
ap.add_argument("--lanes", default="1,2,4,8")
ap.add_argument("--steps", type=int, default=500)
args = ap.parse_args()
for cells in [int(x) for x in args.cells.split(",")]:
    f = E.gen_fcc(cells, 0.8442, 1.0, 12345)
    n = f.size()
    base = None
    for lanes in [int(x) for x in args.lanes.split(",")]:
        eng = E.Engine(f, E.Interactions(), 0.3,
                       E.EngineConfig(section_timers=False, lanes=lanes))
        ids, f0 = eng.forces()
        pe0 = eng.potential_energy()
        eng.run(100)
        ms_force = eng.time_force_kernel(50)
        eng.run(10)
        t0 = time.perf_counter()
        eng.run(args.steps)
        eng.observe()
        dt = time.perf_counter() - t0
        row = {"n": n, "lanes": lanes, "force_ms": ms_force,
               "ms_per_step": dt / args.steps * 1e3, "psps": n * args.steps / dt}
        if base is None:
            base = (f0, pe0)
        else:
            row["f_maxrel"] = float(np.abs(f0 - base[0]).max() / np.abs(base[0]).max())
            row["pe_rel"] = abs(pe0 - base[1]) / abs(base[1])
        print(json.dumps(row), flush=True)
        eng.close()
