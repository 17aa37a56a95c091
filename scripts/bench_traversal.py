"""The reference's traversal microbenchmark (tools/bench_traversal.cpp,
acceptance criterion 11) on the GPU: the full (sorted) list force kernel vs
the explicit pair list (PairIndexList) traversal, same state, best of reps.
python scripts/bench_traversal.py"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2109_10876_b200 import engine as E

cases = [("SC lattice N=4096, rho 0.8442, T 0.72, 50 NVE steps (bench_traversal defaults)",
          lambda: E.gen_lattice(4096, 0.8442, 0.72, 7), 50),
         ("FCC 64^3 x 4 = 1,048,576 (configs[1]), 50 NVE steps",
          lambda: E.gen_fcc(64, 0.8442, 1.0, 12345), 50)]
for what, make, warm in cases:
    f = make()
    with E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005)) as w:
        w.run(warm)
        f = w.flatten()
    eng = E.Engine(f, E.Interactions(), 0.3, E.EngineConfig(dt=0.005))
    m = eng.build_pair_index_list()
    t_runs = min(eng.time_force_kernel(20) for _ in range(3))
    t_pairs = min(eng.time_pair_traversal(20) for _ in range(3))
    st = eng.list_stats()
    print(f"{what}: {st['entries']} full-list entries, {m} explicit pairs; "
          f"full list {t_runs * 1e3:.1f} us, pair list {t_pairs * 1e3:.1f} us, "
          f"ratio (pair list / full list) {t_pairs / t_runs:.2f}", flush=True)
    eng.close()
