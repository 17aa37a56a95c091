"""List-build kernels compared (k_build_brick3 = warp per cell, brick-staged;
k_build_thread = thread per particle; k_build_cull = warp per cell over the
culled candidate stream): build ms, identical pair sets and bit-identical
forces (same entry order).
python scripts/build_variants.py <lj|kg|slab> <cells>"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import bench
from paper_2109_10876_b200 import engine as E

kind, cells = sys.argv[1], int(sys.argv[2])
w = bench.Workload(kind, cells)
res = {}
builds = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [3, 5, 6]
for b in builds:
    eng = E.Engine(w.flat, w.inter, w.r_skin, E.EngineConfig(dt=w.dt, build=b,
                                                               section_timers=False))
    eng.run(20)
    ms = eng.time_list_build(5)
    res[b] = (ms, eng.pairs() if w.n <= 1_100_000 else None, eng.list_stats()["entries"],
              eng.forces()[1])
    eng.close()
    print(f"{kind} cells={cells} n={w.n} build {b}: {ms:.3f} ms, entries {res[b][2]}", flush=True)
b0 = builds[0]
if res[b0][1] is not None:
    print("pair sets identical:", [np.array_equal(res[b0][1], res[b][1]) for b in builds[1:]])
print("forces bit-identical:", [np.array_equal(res[b0][3], res[b][3]) for b in builds[1:]])
