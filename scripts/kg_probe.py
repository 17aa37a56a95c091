"""Kremer-Grest melt (BASELINE configs[2]) kernel probe on one GPU: force
kernel at 1/2/4 threads per particle, list build kinds, and the step time.
python scripts/kg_probe.py [cells=64] [lanes=1,2,4] [builds=5] [unrolls=4]"""
import itertools
import sys
import time
sys.path.insert(0, "/root/repo")
import bench
from paper_2109_10876_b200 import engine as E

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
lanes_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4").split(",")]
builds = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "5").split(",")]
unrolls = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "4").split(",")]
flat, inter, w = bench.make_inputs_ours("kg", cells, 0)
for build, unroll, lanes in itertools.product(builds, unrolls, lanes_list):
    eng = E.Engine(flat, inter, w.r_skin,
                   E.EngineConfig(dt=w.dt, build=build, lanes=lanes, unroll=unroll,
                                  section_timers=False))
    eng.run(50)
    fms = eng.time_force_kernel(20)
    bms = eng.time_list_build(5)
    r0 = eng.rebuild_count()
    t0 = time.perf_counter()
    eng.run(400)
    eng.observe()
    dt = (time.perf_counter() - t0) / 400
    print(f"kg n={w.n} build={build} lanes={lanes} unroll={unroll} force {fms:.4f} ms "
          f"build {bms:.4f} ms step {dt * 1e3:.4f} ms "
          f"rebuilds/step {(eng.rebuild_count() - r0) / 400:.3f}", flush=True)
    eng.close()
