"""Times the LJ force kernel variants on the same 1M-particle state (one GPU).

    python scripts/force_variants.py [--cells 64] [--steps 100] [--reps 20]

Each variant is a separate engine (own list layout) started from the same
FCC state and run for --steps steps; the force kernel is then timed with CUDA
events on the engine's stream (mean over --reps back-to-back launches)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_10876_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=64)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--variants", default="1,2,3:1,3:2,3:4,3:8")
args = ap.parse_args()
f = E.gen_fcc(args.cells, 0.8442, 1.0, 12345)
n = f.size()
res = []
for spec in args.variants.split(","):
    v, _, u = spec.partition(":")
    cfg = E.EngineConfig(section_timers=False, variant=int(v))
    eng = E.Engine(f, E.Interactions(), 0.3, cfg)
    if u:
        # unroll lives in tmd_engine_params.reserved[1]: rebuild with it
        eng.close()
        from paper_2109_10876_b200 import _abi
        import ctypes as C
        sysd = _abi.TmdSystem()
        sysd.box[:] = list(f.box)
        sysd.n = n
        sysd.id = f.id.ctypes.data_as(C.c_void_p)
        sysd.pos = f.pos.ctypes.data_as(C.c_void_p)
        sysd.vel = f.vel.ctypes.data_as(C.c_void_p)
        lj = _abi.TmdLjParams(1.0, 1.0, 2.5, 1)
        p = _abi.TmdEngineParams()
        p.dt, p.r_skin, p.device, p.section_timers = 0.005, 0.3, -1, 0
        p.reserved[0], p.reserved[1] = int(v), int(u)
        h = C.c_void_p()
        assert _abi.lib().tmd_gpu_create(C.byref(sysd), C.byref(lj), None, C.byref(p), C.byref(h)) == 0
        eng = E.Engine.__new__(E.Engine)
        eng._h, eng._n, eng._cfg, eng.box = h, n, cfg, f.box.copy()
    eng.run(args.steps)
    ms = eng.time_force_kernel(args.reps)
    ms_build = eng.time_list_build(max(2, args.reps // 4))
    st = eng.list_stats()
    o = eng.observe()
    B = n * 52 + st["entries"] * 28
    res.append({"variant": spec, "force_ms": ms, "build_ms": ms_build, "frac_hbm_roofline": B / 6552.6e9 / (ms * 1e-3),
                "entries": st["entries"], "pe": o.potential})
    print(json.dumps(res[-1]), flush=True)
    eng.close()
