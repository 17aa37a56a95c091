"""TEST INFRASTRUCTURE ONLY — generates tests/golden/* from the UNMODIFIED
reference engine (oracle/_ref/libtaskmd_ref.so, built from
/root/reference/proj/include by oracle/Makefile).

Every array in a fixture is an output of the reference's own code path
(build_domain / Engine / lj_eval / build_cell_grid / wrap_position /
counter RNG / gen_random / gen_lattice / oracle_forces_energy), except the
`*_fsum` energies, which are exactly-rounded sums (math.fsum) of the
reference's own per-pair terms over the reference's own pair set — the
compensated anchor SURVEY §7 asks for (the reference's running double sum is
only good to ~1e-12 relative).

    python oracle/make_golden.py            # writes tests/golden/
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402

OUT = ROOT / "tests" / "golden"
K_PLACEMENT = 3


def jittered_lattice(side, edge, seed, jitter, temperature=0.0):
    """test_neighbor.cpp:16-37 / test_engine.cpp:15-42 fixture, via the
    reference's counter RNG (ix-major id order)."""
    n = side ** 3
    ids = np.arange(n, dtype=np.int64)
    pos = np.empty((n, 3))
    vel = np.zeros((n, 3))
    spacing = edge / side
    k = 0
    for ix in range(side):
        for iy in range(side):
            for iz in range(side):
                u = ref.counter_uniform3(seed, K_PLACEMENT, 0, k)
                pos[k] = [(ix + 0.5) * spacing + jitter * (2.0 * u[0] - 1.0),
                          (iy + 0.5) * spacing + jitter * (2.0 * u[1] - 1.0),
                          (iz + 0.5) * spacing + jitter * (2.0 * u[2] - 1.0)]
                if temperature > 0.0:
                    g = ref.counter_normal3(seed, 2, 0, k)
                    s = math.sqrt(temperature)
                    vel[k] = [s * g[0], s * g[1], s * g[2]]
                k += 1
    return np.array([edge, edge, edge]), ids, pos, vel


def fcc(cells, rho, offset=0.25):
    """FCC of SURVEY §8(d) (absent from the reference): L = cbrt(n/rho),
    a = L/cells, ids in z, y, x, basis order. Uses the C port's generator so
    that libm's cbrt is the one the product generator (tmd_gen_fcc) uses."""
    from oracle import port
    return port.gen_fcc(cells, rho, offset)


def exact_energies(box, pos_by_id, pairs, lj=(1.0, 1.0, 2.5, True)):
    """fsum of the reference's per-pair LJ terms over its own pair set, with the
    reference's displacement rounding (plain differences of images)."""
    q = ref.lj_prepare(*lj)
    sigma2, rc2, eps4, eps24, shift = q
    ids_sorted, pos_sorted = pos_by_id
    up = np.unique(pairs, axis=0)        # boxes < 2 r_v list a pair once per image
    ia = np.searchsorted(ids_sorted, up[:, 0])
    ib = np.searchsorted(ids_sorted, up[:, 1])
    d0 = pos_sorted[ia] - pos_sorted[ib]
    r2s = []
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            for sz in (-1, 0, 1):
                d = d0 + box * np.array([sx, sy, sz])
                r2s.append((d * d).sum(axis=1))
    r2 = np.concatenate(r2s)
    m = r2 < rc2
    inv = sigma2 / r2[m]
    i6 = inv * inv * inv
    e = eps4 * (i6 * i6 - i6) - shift
    ff = eps24 * (2.0 * i6 * i6 - i6) / r2[m]
    return math.fsum(e.tolist()), math.fsum((ff * r2[m]).tolist()), int(m.sum())


def bond_energies(box, pos_by_id, bonds, fene):
    """fsum of the reference's FENE terms (fene_eval, potentials.hpp:95-104)
    over the minimum-image bond vectors, and their virial ff r^2."""
    k, r_max = fene
    ids_sorted, pos_sorted = pos_by_id
    ia = np.searchsorted(ids_sorted, bonds[:, 0])
    ib = np.searchsorted(ids_sorted, bonds[:, 1])
    d = pos_sorted[ia] - pos_sorted[ib]
    d -= box * np.round(d / box)
    r2 = (d * d).sum(axis=1)
    rmax2 = r_max * r_max
    g = 1.0 - r2 / rmax2
    e = -0.5 * k * rmax2 * np.log(g)
    ff = -k / g
    return math.fsum(e.tolist()), math.fsum((ff * r2).tolist())


def system_fixture(name, box, ids, pos, vel, *, r_skin=0.3, n_subs=(1, 8), steps=0,
                   trace_every=0, dt=0.005, oracle=False, thermostat=None, lj=None,
                   bonds=None, fene=None):
    out = dict(box=box, ids=ids, pos=pos, vel=vel, r_skin=np.float64(r_skin),
               dt=np.float64(dt))
    if thermostat is not None:
        out["thermostat"] = np.array(thermostat, dtype=np.float64)  # gamma, T, seed
    lj = lj or (1.0, 1.0, 2.5, True)
    if lj != (1.0, 1.0, 2.5, True):
        out["lj"] = np.array([lj[0], lj[1], lj[2], 1.0 if lj[3] else 0.0])
    if bonds is not None:
        out["bonds"] = np.asarray(bonds, np.int64)
        out["fene"] = np.array(fene, dtype=np.float64)
    pairs0 = None
    for ns in n_subs:
        e = ref.RefEngine(box, ids, pos, vel, r_skin=r_skin, n_sub=ns, dt=dt,
                          thermostat=thermostat, eps=lj[0], sigma=lj[1], r_cut=lj[2],
                          shifted=lj[3], bonds=bonds, fene=fene)
        p = e.pairs()
        if pairs0 is None:
            pairs0 = p
            ci, cell = e.cell_of()
            fi, f = e.forces()
            o = e.observe()
            fl_ids, fl_pos, fl_vel = e.flatten()
            out.update(pairs=p.astype(np.int64), cell=cell, forces=f,
                       pe_ref=np.float64(o["potential"]), ke_ref=np.float64(o["kinetic"]),
                       wrapped=fl_pos)
            dims, cl = e.grid()
            out.update(dims=dims, cell_len=cl)
            pe_f, w_f, ncut = exact_energies(box, (fl_ids, fl_pos), p, lj)
            if bonds is not None:
                be, bw = bond_energies(box, (fl_ids, fl_pos), np.asarray(bonds), fene)
                pe_f, w_f = math.fsum([pe_f, be]), math.fsum([w_f, bw])
            out.update(pe_fsum=np.float64(pe_f), w_fsum=np.float64(w_f),
                       n_incut=np.int64(ncut))
            if steps:
                trace = []
                done = 0
                while done < steps:
                    k = min(trace_every or steps, steps - done)
                    e.run(k)
                    done += k
                    ob = e.observe()
                    trace.append([ob["step"], ob["kinetic"], ob["potential"]])
                ti, tp, tv = e.flatten()
                out.update(steps=np.int64(steps), trace=np.array(trace),
                           final_pos=tp, final_vel=tv,
                           rebuilds=np.int64(e.rebuild_count()))
        else:
            assert np.array_equal(p, pairs0), f"{name}: n_sub={ns} pair set differs"
        e.close()
    if oracle:
        f_or, pe_or = ref.oracle_forces(box, ids, pos)
        out.update(oracle_forces=f_or, oracle_pe=np.float64(pe_or),
                   oracle_pairs=ref.oracle_pairs(box, ids, pos, 2.5 + r_skin))
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"  {name}: n={len(ids)} pairs={len(pairs0)} dims={out['dims'].tolist()}")


def thermostat_fixtures():
    """Langevin runs (thermostat_and_half_kick, engine.hpp:209-239): the
    reference's worker-independence system (test_engine.cpp:214-240) and a
    jittered FCC melt."""
    b, i, p, v = jittered_lattice(6, 7.2, 29, 0.05, 0.0)
    system_fixture("langevin_jit6", b, i, p, v, n_subs=(1, 8), steps=30, trace_every=5,
                   thermostat=(1.0, 0.8, 99))
    b, i, p = fcc(8, 0.8442)
    for k in range(len(i)):
        u = ref.counter_uniform3(777, K_PLACEMENT, 0, k)
        p[k] += 0.15 * (2.0 * u - 1.0)
    v = ref.thermal_velocities(i, 0.7, 4242)
    system_fixture("langevin_fcc8", b, i, p, v, n_subs=(1, 8), steps=100, trace_every=20,
                   thermostat=(0.5, 1.4, 2021))


def lattice_chains(side, rho, seed, jitter=0.05, temperature=1.0):
    """Kremer-Grest test melt without overlaps: side^3 beads on a simple cubic
    lattice at bead density rho, one chain per z plane running boustrophedon
    through it (every bond one lattice spacing, about 1.056 at rho = 0.85),
    positions jittered with the reference's counter RNG, thermal velocities."""
    a = (1.0 / rho) ** (1.0 / 3.0)
    n = side ** 3
    ids = np.arange(n, dtype=np.int64)
    pos = np.empty((n, 3))
    bonds = []
    k = 0
    for z in range(side):
        for y in range(side):
            xs = range(side) if y % 2 == 0 else range(side - 1, -1, -1)
            for x in xs:
                u = ref.counter_uniform3(seed, K_PLACEMENT, 0, k)
                pos[k] = [(x + 0.5) * a + jitter * (2.0 * u[0] - 1.0),
                          (y + 0.5) * a + jitter * (2.0 * u[1] - 1.0),
                          (z + 0.5) * a + jitter * (2.0 * u[2] - 1.0)]
                k += 1
        base = z * side * side
        bonds += [[base + j, base + j + 1] for j in range(side * side - 1)]
    vel = ref.thermal_velocities(ids, temperature, seed)
    return np.full(3, side * a), ids, pos, vel, np.array(bonds, dtype=np.int64)


def bonded_fixtures():
    """FENE + WCA (Kremer-Grest) runs of the reference (row f1)."""
    wca = (1.0, 1.0, 2.0 ** (1.0 / 6.0), True)
    kg_fene = (30.0, 1.5)
    b, i, p, v, bonds = lattice_chains(10, 0.85, 17)
    system_fixture("kg_lattice10", b, i, p, v, r_skin=0.4, n_subs=(1, 8), steps=200,
                   trace_every=20, dt=0.005, lj=wca, bonds=bonds, fene=kg_fene)
    # bonded LJ liquid: FENE chains inside the standard LJ fluid (r_cut 2.5)
    b, i, p, v, bonds = lattice_chains(8, 0.8, 23, jitter=0.08, temperature=0.8)
    system_fixture("fene_lj8", b, i, p, v, r_skin=0.3, n_subs=(1, 8), steps=100,
                   trace_every=20, dt=0.004, bonds=bonds, fene=kg_fene)


def generator_fixtures():
    """The reference's generators (generators.hpp) on a few parameter sets:
    pins the product's restatements used by the run-config front end."""
    out = {}
    for tag, (n, rho, t, seed) in {"lat100": (100, 0.8442, 0.72, 3),
                                   "lat1000": (1000, 0.5, 1.0, 12345),
                                   "lat9": (9, 0.1, 0.0, 1)}.items():
        b, i, p, v = ref.gen_lattice(n, rho, t, seed)
        out.update({f"{tag}_box": b, f"{tag}_ids": i, f"{tag}_pos": p, f"{tag}_vel": v})
    for tag, (n, rho, dmin, t, seed) in {"rnd200": (200, 0.8442, 0.8, 0.72, 1),
                                         "rnd50": (50, 0.3, 1.0, 0.0, 99)}.items():
        b, i, p, v = ref.gen_random(n, rho, dmin, t, seed)
        out.update({f"{tag}_box": b, f"{tag}_ids": i, f"{tag}_pos": p, f"{tag}_vel": v})
    for tag, args in {"sph": (14.0, 0.7, 0.8442, 0.1, 0.1, 7),
                      "sph_full": (9.0, 1.0, 0.6, 1.0, 0.5, 2)}.items():
        b, i, p, v = ref.gen_spherical(*args)
        out.update({f"{tag}_box": b, f"{tag}_ids": i, f"{tag}_pos": p, f"{tag}_vel": v})
    np.savez_compressed(OUT / "generators.npz", **out)
    print("  generators:", sorted({k.split("_")[0] for k in out}))


def main():
    if not ref.available():
        ref.build()
    OUT.mkdir(parents=True, exist_ok=True)
    if "--only-generators" in sys.argv:
        generator_fixtures()
        return
    if "--only-thermostat" in sys.argv:
        thermostat_fixtures()
        return
    if "--only-bonded" in sys.argv:
        bonded_fixtures()
        return

    # -- scalar LJ: lj_eval over a grid of r2 (test_potentials.cpp:33-89)
    r2 = np.concatenate([np.linspace(0.64, 7.0, 257), [2 ** (1 / 3), 1.0, 6.25,
                                                      6.25 * (1 - 1e-14), 9.0]])
    rows = []
    for x in r2:
        for sh in (True, False):
            e, ff = ref.lj_eval(float(x), 1.0, 1.0, 2.5, sh)
            rows.append([x, 1.0 if sh else 0.0, e, ff])
    np.savez_compressed(OUT / "lj_scalar.npz", table=np.array(rows),
                        prep_shifted=ref.lj_prepare(1.0, 1.0, 2.5, True),
                        prep_unshifted=ref.lj_prepare(1.0, 1.0, 2.5, False))

    # -- grids + binning (test_grid.cpp:8-95)
    grids = []
    for box, rc, sk in [((67.7177,) * 3, 2.5, 0.3), ((12.0, 6.0, 30.0), 2.5, 0.5),
                        ((12.0, 9.0, 15.0), 2.5, 0.5), ((12.0,) * 3, 2.5, 0.5),
                        ((33.591923828, ) * 3, 2.5, 0.3), ((107.49415, ) * 3, 2.5, 0.3),
                        ((268.7354, ) * 3, 2.5, 0.3), ((135.434, 135.434, 406.30), 2.5, 0.3),
                        ((4.0, 7.0, 7.0), 2.5, 0.3)]:
        dims, cl = ref.build_cell_grid(np.array(box), rc, sk)
        grids.append(dict(box=list(box), r_cut=rc, r_skin=sk, dims=dims.tolist(),
                          cell_len=cl.tolist()))
    (OUT / "grids.json").write_text(json.dumps(grids, indent=1))
    # tricky positions: upper face, tiny negatives, far outside both ways
    rng = np.random.default_rng(7)
    L = 12.0
    pts = [[L - 1e-13, 0.0, 6.0], [0.0, 0.0, 0.0], [-1e-17, -1e-300, L],
           [L, 2 * L, -L], [-5e-16, L - 5e-16, 3.0]]
    pts += [[-5.0 + 0.7 * k, 25.0 - 0.9 * k, 0.31 * k] for k in range(50)]
    pts += (rng.uniform(-3 * L, 4 * L, size=(400, 3))).tolist()
    pts += (np.repeat(np.arange(0, 5) * 3.0, 3).reshape(5, 3) + np.array([[-1e-16, 0, 1e-16]])).tolist()
    pts = np.array(pts)
    w, cell = ref.wrap_and_bin(pts, np.array([L, L, L]), 2.5, 0.5)
    np.savez_compressed(OUT / "binning.npz", pos=pts, box=np.array([L, L, L]), r_cut=2.5,
                        r_skin=0.5, wrapped=w, cell=cell)

    # -- counter RNG + thermal velocities (random.hpp, generators.hpp:19-39)
    keys = np.array([[s, c, st, i] for s in (0, 1, 12345, 2 ** 63 + 5) for c in (1, 2, 3)
                     for st in (0, 7) for i in (0, 1, 999, 2 ** 40)], dtype=np.uint64)
    nrm = np.array([ref.counter_normal3(*map(int, k)) for k in keys])
    uni = np.array([ref.counter_uniform3(*map(int, k)) for k in keys])
    tv_ids = np.arange(1000, dtype=np.int64) * 3 + 11
    tv = ref.thermal_velocities(tv_ids, 1.0, 12345)
    np.savez_compressed(OUT / "rng.npz", keys=keys, normal3=nrm, uniform3=uni,
                        tv_ids=tv_ids, tv=tv)

    # -- systems
    print("systems:")
    b, i, p, v = jittered_lattice(6, 7.0, 101, 0.1)
    system_fixture("jit6_s101", b, i, p, v, oracle=True)
    b, i, p, v = jittered_lattice(6, 7.2, 41, 0.05, 0.8)
    system_fixture("jit6_s41_T08", b, i, p, v, steps=1, n_subs=(1, 8))
    for seed in (1, 2, 3):
        b, i, p, v = ref.gen_random(500, 0.8442, 0.8, 0.72, seed)
        system_fixture(f"random500_s{seed}", b, i, p, v, n_subs=(1, 8), oracle=True)
    # FCC 8^3 x 4, jittered (SURVEY §8c jitter rule), T = 1.0 seed 12345
    b, i, p = fcc(8, 0.8442)
    for k in range(len(i)):
        u = ref.counter_uniform3(777, K_PLACEMENT, 0, k)
        p[k] += 0.15 * (2.0 * u - 1.0)
    v = ref.thermal_velocities(i, 1.0, 12345)
    system_fixture("fcc8_jit", b, i, p, v, n_subs=(1, 8), steps=200, trace_every=20)
    # anisotropic box, and one axis a single cell wide (periodic self-images)
    rng = np.random.default_rng(11)
    for name, box, n in (("aniso", (12.0, 9.5, 30.0), 260), ("thin", (4.0, 7.0, 7.0), 120)):
        box = np.array(box)
        pts = []
        while len(pts) < n:
            q = rng.uniform(0, 1, 3) * box
            ok = True
            for r in pts:
                d = q - r
                d -= box * np.round(d / box)
                if (d * d).sum() < 0.85 ** 2:
                    ok = False
                    break
            if ok:
                pts.append(q)
        pos = np.array(pts)
        ids = (np.arange(n, dtype=np.int64) * 7919) % 100003  # non-contiguous ids
        vel = ref.thermal_velocities(ids, 0.5, 99)
        system_fixture(name, box, ids, pos, vel, n_subs=(1,), steps=50, trace_every=10)
    thermostat_fixtures()
    bonded_fixtures()
    generator_fixtures()
    # SC lattice 4000 (acceptance criterion 3): energy traces at dt 0.005, 0.001
    b, i, p, v = ref.gen_lattice(4000, 0.8442, 0.6, 3)
    traces = {}
    for dt in (0.005, 0.001):
        e = ref.RefEngine(b, i, p, v, r_skin=0.3, n_sub=8, dt=dt)
        o = e.observe()
        e0 = o["kinetic"] + o["potential"]
        tr = []
        for _ in range(100):
            e.run(10)
            ob = e.observe()
            tr.append(ob["kinetic"] + ob["potential"])
        tr = np.array(tr)
        traces[f"dt{dt}"] = tr
        traces[f"e0_dt{dt}"] = np.float64(e0)
        traces[f"worst_dt{dt}"] = np.float64(np.abs(tr - e0).max() / abs(e0))
        traces[f"rebuilds_dt{dt}"] = np.int64(e.rebuild_count())
    np.savez_compressed(OUT / "lattice4000_s3.npz", box=b, ids=i, pos=p, vel=v, **traces)
    print("  lattice4000_s3: worst drift", traces["worst_dt0.005"], traces["worst_dt0.001"])

    # -- config 1 (32K FCC, seed 12345) summary known answers
    b, i, p = fcc(20, 0.8442)
    v = ref.thermal_velocities(i, 1.0, 12345)
    e = ref.RefEngine(b, i, p, v, r_skin=0.3)
    pr = e.pairs()
    fl_ids, fl_pos, _ = e.flatten()
    pe_f, w_f, ncut = exact_energies(b, (fl_ids, fl_pos), pr)
    o = e.observe()
    _, cell = e.cell_of()
    summary = dict(n=len(i), L=float(b[0]), pairs=int(len(pr)), in_cut=ncut,
                   pe_ref=o["potential"], ke_ref=o["kinetic"], pe_fsum=pe_f, w_fsum=w_f,
                   cell_checksum=int((cell.astype(np.int64) * (np.arange(len(i)) % 9973 + 1)).sum()),
                   pair_checksum=int(((pr[:, 0] * 1000003 + pr[:, 1]) % 2147483647).sum()))
    (OUT / "fcc20_summary.json").write_text(json.dumps(summary, indent=1))
    print("  fcc20:", summary)


if __name__ == "__main__":
    main()
