"""Probe the KG warm-up: minimum non-bonded distance, bond lengths, max force,
energy drift of NVE at several dt after the capped Langevin warm-up."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

nc, cl = int(sys.argv[1]), int(sys.argv[2])
spc = int(sys.argv[3]) if len(sys.argv) > 3 else 100


def stats(f, tag):
    eng = E.Engine(f, E.kg_interactions(), 0.4, E.EngineConfig(dt=0.01))
    ids, F = eng.forces()
    pairs = eng.pairs()
    pos = f.pos[np.argsort(f.id)]
    d = pos[pairs[:, 0]] - pos[pairs[:, 1]]
    d -= f.box * np.round(d / f.box)
    r = np.sqrt((d * d).sum(1))
    bd = pos[f.bonds[:, 0]] - pos[f.bonds[:, 1]]
    bd -= f.box * np.round(bd / f.box)
    br = np.sqrt((bd * bd).sum(1))
    o = eng.observe()
    print(f"{tag}: min pair r {r.min():.3f}, bonds [{br.min():.3f}, {br.max():.3f}], "
          f"max|F| {np.abs(F).max():.1f}, PE/N {o.potential / f.size():.3f}, T {o.temperature:.3f}",
          flush=True)
    eng.close()


f = E.gen_chains(nc, cl, 0.85, 0.97, seed=3)
print("N", f.size(), "L", f.box[0])
cur = f
caps = (5.0, 10.0, 20.0, 50.0, 100.0, 300.0, 1000.0)
for k, cap in enumerate(list(caps) + [0.0]):
    cfg = E.EngineConfig(dt=0.002 if cap else 0.005, section_timers=False, force_cap=float(cap),
                         thermostat=E.LangevinParams(1.0, 1.0, 7 + k))
    try:
        with E.Engine(cur, E.kg_interactions(), 0.4, cfg) as eng:
            eng.run(spc if cap else 1500)
            cur = eng.flatten()
    except Exception as e:
        print("cap", cap, "failed:", e)
        break
    stats(cur, f"after cap {cap}")
for dt in (0.005, 0.01):
    eng = E.Engine(cur, E.kg_interactions(), 0.4, E.EngineConfig(dt=dt, section_timers=False))
    o0 = eng.observe()
    e0 = o0.kinetic + o0.potential
    try:
        for c in range(10):
            eng.run(50)
            o = eng.observe()
            print(f"  dt {dt} step {o.step}: dE/E {(o.kinetic + o.potential - e0) / e0:.2e} T {o.temperature:.3f}", flush=True)
    except Exception as e:
        print("  dt", dt, "failed:", e)
    eng.close()
