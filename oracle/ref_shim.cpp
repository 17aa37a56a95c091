// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" shim over the UNMODIFIED reference engine (`taskmd`, header-only
// C++20 under /root/reference/proj/include). This file contains no reference
// source: it only #includes the reference headers at build time
// (oracle/Makefile, -I$(REF_INCLUDE)) and exposes the reference's own public
// API through plain C entry points so that the parity tests (tests/), the
// golden-vector generator (oracle/make_golden.py) and the CPU baseline arm of
// bench.py can drive it through ctypes. The built library lands in
// oracle/_ref/libtaskmd_ref.so (git-ignored, travels to the GPU box).
//
// Every entry point names the reference symbol it forwards to.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "taskmd/domain.hpp"      // build_domain, flatten_domain (domain.hpp:134-207)
#include "taskmd/engine.hpp"      // Engine, EngineConfig, autotune_subnodes (engine.hpp:19-373)
#include "taskmd/generators.hpp"  // gen_lattice, gen_random, thermal_velocities (generators.hpp)
#include "taskmd/oracle.hpp"      // oracle_forces_energy, oracle_pair_set (oracle.hpp:34-191)
#include "taskmd/random.hpp"      // counter_uniform3, counter_normal3 (random.hpp:53-81)

using namespace taskmd;

namespace {

// Status codes shared with include/tmd_gpu.h.
constexpr int kOk = 0, kConfig = 1, kPhysics = 2, kVerify = 3, kState = 4,
              kOther = 9;

void put_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
  }
}

template <class F>
int guarded(char* err, int errlen, F&& fn) {
  try {
    fn();
    return kOk;
  } catch (const ConfigError& e) {
    put_err(err, errlen, e.what());
    return kConfig;
  } catch (const PhysicsError& e) {
    put_err(err, errlen, e.what());
    return kPhysics;
  } catch (const VerifyError& e) {
    put_err(err, errlen, e.what());
    return kVerify;
  } catch (const StateError& e) {
    put_err(err, errlen, e.what());
    return kState;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return kOther;
  }
}

FlatConfig make_flat(std::int64_t n, const std::int64_t* id,
                     const double* mass, const double* pos, const double* vel,
                     const double box[3]) {
  FlatConfig f;
  f.box = BoxSpec{{box[0], box[1], box[2]}};
  for (std::int64_t k = 0; k < n; ++k) {
    ParticleRec r;
    r.id = id[k];
    r.type = 0;
    r.mass = mass ? mass[k] : 1.0;
    r.pos = {pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]};
    if (vel) r.vel = {vel[3 * k], vel[3 * k + 1], vel[3 * k + 2]};
    f.push(r);
  }
  return f;
}

Interactions make_inter(double eps, double sigma, double rc, int shifted) {
  Interactions inter;
  inter.lj = LjParams{eps, sigma, rc, shifted != 0};
  return inter;
}

void copy_out_flat(const FlatConfig& f, std::int64_t* id, double* pos,
                   double* vel) {
  for (std::size_t k = 0; k < f.size(); ++k) {
    if (id) id[k] = f.id[k];
    if (pos) {
      pos[3 * k] = f.pos[k].x;
      pos[3 * k + 1] = f.pos[k].y;
      pos[3 * k + 2] = f.pos[k].z;
    }
    if (vel) {
      vel[3 * k] = f.vel[k].x;
      vel[3 * k + 1] = f.vel[k].y;
      vel[3 * k + 2] = f.vel[k].z;
    }
  }
}

}  // namespace

struct ref_engine {
  std::unique_ptr<Engine> eng;
};

extern "C" {

// build_domain (domain.hpp:134) + Engine::Engine (engine.hpp:68): the initial
// (untimed) force evaluation runs here.
int ref_create(std::int64_t n, const std::int64_t* id, const double* mass,
               const double* pos, const double* vel, const double box[3],
               double eps, double sigma, double rc, int shifted, double r_skin,
               int n_sub, int workers, double dt, ref_engine** out, char* err,
               int errlen) {
  *out = nullptr;
  return guarded(err, errlen, [&] {
    FlatConfig f = make_flat(n, id, mass, pos, vel, box);
    EngineConfig cfg;
    cfg.dt = dt;
    cfg.n_sub = n_sub;
    cfg.worker_threads = workers;
    auto h = std::make_unique<ref_engine>();
    h->eng = std::make_unique<Engine>(
        build_domain(f, make_inter(eps, sigma, rc, shifted), r_skin, n_sub),
        cfg);
    *out = h.release();
  });
}

// The same with the optional parts of the configuration: a Langevin bath
// (EngineConfig::thermostat, engine.hpp:19-26) and FENE bonds
// (Topology::bonds + Interactions::fene, topology.hpp:14-31, domain.hpp:19-23).
struct ref_opts {
  int thermostat;
  double gamma, temperature;
  std::uint64_t seed;
  std::int64_t n_bonds;
  const std::int64_t* bonds;
  int fene;
  double fene_k, fene_rmax;
};

int ref_create_ex(std::int64_t n, const std::int64_t* id, const double* mass,
                  const double* pos, const double* vel, const double box[3], double eps,
                  double sigma, double rc, int shifted, double r_skin, int n_sub, int workers,
                  double dt, const ref_opts* o, ref_engine** out, char* err, int errlen) {
  *out = nullptr;
  return guarded(err, errlen, [&] {
    FlatConfig f = make_flat(n, id, mass, pos, vel, box);
    for (std::int64_t k = 0; k < o->n_bonds; ++k) {
      f.topo.bonds.push_back({o->bonds[2 * k], o->bonds[2 * k + 1]});
    }
    Interactions inter = make_inter(eps, sigma, rc, shifted);
    if (o->fene) inter.fene = FeneParams{o->fene_k, o->fene_rmax};
    EngineConfig cfg;
    cfg.dt = dt;
    cfg.n_sub = n_sub;
    cfg.worker_threads = workers;
    if (o->thermostat) {
      LangevinParams bath;
      bath.gamma = o->gamma;
      bath.temperature = o->temperature;
      bath.seed = o->seed;
      cfg.thermostat = bath;
    }
    auto h = std::make_unique<ref_engine>();
    h->eng = std::make_unique<Engine>(build_domain(f, inter, r_skin, n_sub), cfg);
    *out = h.release();
  });
}

void ref_destroy(ref_engine* h) { delete h; }

// Engine::Engine(Domain, EngineConfig) (engine.hpp:68-77) over a copy of h's
// Domain with another worker count (the same subnode layout): the CPU
// baseline's 1-thread rate without a second build_domain.
int ref_clone(ref_engine* h, int workers, ref_engine** out, char* err, int errlen) {
  *out = nullptr;
  return guarded(err, errlen, [&] {
    EngineConfig cfg = h->eng->config();
    cfg.worker_threads = workers;
    auto c = std::make_unique<ref_engine>();
    c->eng = std::make_unique<Engine>(Domain(h->eng->domain()), cfg);
    *out = c.release();
  });
}

// Engine::run (engine.hpp:128).
int ref_step(ref_engine* h, std::int64_t nsteps, char* err, int errlen) {
  return guarded(err, errlen, [&] { h->eng->run(nsteps); });
}

// Engine::observe (engine.hpp:132): {step, kinetic, potential, temperature}.
void ref_observe(ref_engine* h, double out[4]) {
  const StepObservables o = h->eng->observe();
  out[0] = static_cast<double>(o.step);
  out[1] = o.kinetic;
  out[2] = o.potential;
  out[3] = o.temperature;
}

std::int64_t ref_size(ref_engine* h) {
  return static_cast<std::int64_t>(h->eng->domain().n_particles);
}

// flatten_domain (domain.hpp:193): sorted by id, positions wrapped.
void ref_flatten(ref_engine* h, std::int64_t* id, double* pos, double* vel) {
  copy_out_flat(flatten_domain(h->eng->domain()), id, pos, vel);
}

// Interior forces by id, read from the stores like acceptance.cpp:53-64.
// Output sorted by id.
void ref_forces(ref_engine* h, std::int64_t* id, double* f) {
  const Domain& d = h->eng->domain();
  std::vector<std::pair<std::int64_t, Vec3>> rows;
  for (const Subnode& sn : d.subs) {
    for (std::int32_t c : sn.interior) {
      const CellSpan& span = sn.store.cells[c];
      for (std::size_t k = span.begin; k < span.begin + span.real; ++k) {
        rows.emplace_back(sn.store.id[k], sn.store.force(k));
      }
    }
  }
  std::sort(rows.begin(), rows.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  for (std::size_t k = 0; k < rows.size(); ++k) {
    id[k] = rows[k].first;
    f[3 * k] = rows[k].second.x;
    f[3 * k + 1] = rows[k].second.y;
    f[3 * k + 2] = rows[k].second.z;
  }
}

// Global cell each owned particle is stored in (local_to_global of its store
// cell, subnode.hpp:31), sorted by id: the reference's binning result
// (distribute_records, domain.hpp:54-65).
void ref_cell_of(ref_engine* h, std::int64_t* id, std::int32_t* cell) {
  const Domain& d = h->eng->domain();
  std::vector<std::pair<std::int64_t, std::int32_t>> rows;
  for (const Subnode& sn : d.subs) {
    for (std::int32_t c : sn.interior) {
      const CellSpan& span = sn.store.cells[c];
      for (std::size_t k = span.begin; k < span.begin + span.real; ++k) {
        rows.emplace_back(sn.store.id[k], sn.local_to_global[c]);
      }
    }
  }
  std::sort(rows.begin(), rows.end());
  for (std::size_t k = 0; k < rows.size(); ++k) {
    id[k] = rows[k].first;
    cell[k] = rows[k].second;
  }
}

// Every (min id, max id) pair held in the sorted neighbour lists, sentinel
// padding skipped, sorted (the listed_pairs helper of test_neighbor.cpp:49-65
// restated over the public Domain fields). Returns the count; writes at most
// cap pairs.
std::int64_t ref_pairs(ref_engine* h, std::int64_t* out, std::int64_t cap) {
  const Domain& d = h->eng->domain();
  std::vector<std::pair<std::int64_t, std::int64_t>> pairs;
  for (int s = 0; s < d.n_sub(); ++s) {
    const SoaStore& st = d.subs[s].store;
    const SortedNeighborList& nl = d.nlists[s];
    for (std::size_t n = 0; n < nl.ilist.size(); ++n) {
      const std::int64_t a = st.id[nl.ilist[n]];
      for (std::int32_t j = nl.irange[n].first; j < nl.irange[n].second; ++j) {
        const std::int64_t b = st.id[nl.jlist[j]];
        if (b == SoaStore::kSentinelId) continue;
        pairs.emplace_back(std::min(a, b), std::max(a, b));
      }
    }
  }
  std::sort(pairs.begin(), pairs.end());
  const std::int64_t n = static_cast<std::int64_t>(pairs.size());
  for (std::int64_t k = 0; k < std::min(n, cap); ++k) {
    out[2 * k] = pairs[k].first;
    out[2 * k + 1] = pairs[k].second;
  }
  return n;
}

// Engine::timers (engine.hpp:145), SectionTimers order Forces, Comm,
// Integrate, Neigh, Resort (timers.hpp:11-17).
void ref_timers(ref_engine* h, double sec[5], double* elapsed) {
  const SectionTimers& t = h->eng->timers();
  for (int k = 0; k < 5; ++k) sec[k] = t.seconds[k];
  *elapsed = t.elapsed;
}

std::uint64_t ref_rebuild_count(ref_engine* h) {
  return h->eng->rebuild_count();
}

void ref_grid(ref_engine* h, int dims[3], double cell_len[3]) {
  const CellGrid& g = h->eng->domain().grid;
  for (int k = 0; k < 3; ++k) dims[k] = g.dims[k];
  cell_len[0] = g.cell_len.x;
  cell_len[1] = g.cell_len.y;
  cell_len[2] = g.cell_len.z;
}

// ---- standalone reference functions -------------------------------------

// lj_prepare (potentials.hpp:49): {sigma2, rc2, eps4, eps24, shift}.
void ref_lj_prepare(double eps, double sigma, double rc, int shifted,
                    double out[5]) {
  const LjPrepared q = lj_prepare(LjParams{eps, sigma, rc, shifted != 0});
  out[0] = q.sigma2;
  out[1] = q.rc2;
  out[2] = q.eps4;
  out[3] = q.eps24;
  out[4] = q.shift;
}

// lj_eval (potentials.hpp:65): {energy, force_factor}.
void ref_lj_eval(double r2, double eps, double sigma, double rc, int shifted,
                 double out[2]) {
  const PairTerm t = lj_eval(r2, LjParams{eps, sigma, rc, shifted != 0});
  out[0] = t.energy;
  out[1] = t.force_factor;
}

// build_cell_grid (cell_grid.hpp:54).
int ref_build_cell_grid(const double box[3], double rc, double skin,
                        int dims[3], double cell_len[3], char* err,
                        int errlen) {
  return guarded(err, errlen, [&] {
    const CellGrid g =
        build_cell_grid(BoxSpec{{box[0], box[1], box[2]}}, rc, skin);
    for (int k = 0; k < 3; ++k) dims[k] = g.dims[k];
    cell_len[0] = g.cell_len.x;
    cell_len[1] = g.cell_len.y;
    cell_len[2] = g.cell_len.z;
  });
}

// wrap_position (box.hpp:53) + CellGrid::cell_of (cell_grid.hpp:48) for a
// batch of raw positions: the binning map the GPU must reproduce bit-exactly.
int ref_wrap_and_bin(std::int64_t n, const double* pos, const double box[3],
                     double rc, double skin, double* wrapped,
                     std::int32_t* cell, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const BoxSpec b{{box[0], box[1], box[2]}};
    const CellGrid g = build_cell_grid(b, rc, skin);
    for (std::int64_t k = 0; k < n; ++k) {
      const Vec3 w =
          wrap_position({pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]}, b);
      wrapped[3 * k] = w.x;
      wrapped[3 * k + 1] = w.y;
      wrapped[3 * k + 2] = w.z;
      cell[k] = g.cell_of(w);
    }
  });
}

// CellGrid::cell_coords (cell_grid.hpp:36) on an already-wrapped position.
void ref_cell_coords(const double box[3], double rc, double skin,
                     const double p[3], int out[3]) {
  const CellGrid g = build_cell_grid(BoxSpec{{box[0], box[1], box[2]}}, rc, skin);
  const auto c = g.cell_coords({p[0], p[1], p[2]});
  for (int k = 0; k < 3; ++k) out[k] = c[k];
}

double ref_wrap1(double p, double length) { return wrap1(p, length); }

// counter_uniform3 / counter_normal3 (random.hpp:53-81).
void ref_counter_uniform3(std::uint64_t seed, std::uint64_t ctx,
                          std::uint64_t step, std::uint64_t id, double out[3]) {
  const Vec3 u = counter_uniform3(seed, static_cast<RngContext>(ctx), step, id);
  out[0] = u.x;
  out[1] = u.y;
  out[2] = u.z;
}

void ref_counter_normal3(std::uint64_t seed, std::uint64_t ctx,
                         std::uint64_t step, std::uint64_t id, double out[3]) {
  const Vec3 u = counter_normal3(seed, static_cast<RngContext>(ctx), step, id);
  out[0] = u.x;
  out[1] = u.y;
  out[2] = u.z;
}

// gen_detail::thermal_velocities + zero_net_momentum (generators.hpp:19-39),
// applied to caller-provided ids/masses.
void ref_thermal_velocities(std::int64_t n, const std::int64_t* id,
                            const double* mass, double temperature,
                            std::uint64_t seed, double* vel) {
  FlatConfig f;
  f.box = BoxSpec::cubic(1.0);
  for (std::int64_t k = 0; k < n; ++k) {
    ParticleRec r;
    r.id = id[k];
    r.mass = mass ? mass[k] : 1.0;
    f.push(r);
  }
  gen_detail::thermal_velocities(f, temperature, seed);
  gen_detail::zero_net_momentum(f);
  copy_out_flat(f, nullptr, nullptr, vel);
}

// gen_lattice (generators.hpp:50) — simple cubic; arrays sized n.
int ref_gen_lattice(std::int64_t n, double rho, double temperature,
                    std::uint64_t seed, std::int64_t* id, double* pos,
                    double* vel, double box[3], char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const FlatConfig f =
        gen_lattice(static_cast<std::size_t>(n), rho, temperature, seed);
    copy_out_flat(f, id, pos, vel);
    box[0] = f.box.length.x;
    box[1] = f.box.length.y;
    box[2] = f.box.length.z;
  });
}

// gen_random (generators.hpp:216).
int ref_gen_random(std::int64_t n, double rho, double min_d,
                   double temperature, std::uint64_t seed, std::int64_t* id,
                   double* pos, double* vel, double box[3], char* err,
                   int errlen) {
  return guarded(err, errlen, [&] {
    const FlatConfig f = gen_random(static_cast<std::size_t>(n), rho, min_d,
                                    temperature, seed);
    copy_out_flat(f, id, pos, vel);
    box[0] = f.box.length.x;
    box[1] = f.box.length.y;
    box[2] = f.box.length.z;
  });
}

// gen_spherical (generators.hpp:87). Arrays sized cap; *n_out = count.
int ref_gen_spherical(double box_length, double frac, double rho_in, double alpha,
                      double temperature, std::uint64_t seed, std::int64_t cap,
                      std::int64_t* id, double* pos, double* vel, std::int64_t* n_out,
                      char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const FlatConfig f = gen_spherical(box_length, frac, rho_in, alpha, temperature, seed);
    *n_out = static_cast<std::int64_t>(f.size());
    if (*n_out <= cap) copy_out_flat(f, id, pos, vel);
  });
}

// oracle_forces_energy (oracle.hpp:112): brute-force minimum-image forces in
// input order and the pair energy.
int ref_oracle_forces(std::int64_t n, const std::int64_t* id, const double* pos,
                      const double box[3], double eps, double sigma, double rc,
                      int shifted, double* f, double* pe, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    const FlatConfig fc = make_flat(n, id, nullptr, pos, nullptr, box);
    const OracleResult r =
        oracle_forces_energy(fc, make_inter(eps, sigma, rc, shifted));
    for (std::int64_t k = 0; k < n; ++k) {
      f[3 * k] = r.force[k].x;
      f[3 * k + 1] = r.force[k].y;
      f[3 * k + 2] = r.force[k].z;
    }
    *pe = r.pair_energy;
  });
}

// oracle_pair_set (oracle.hpp:34). Returns the count; writes at most cap.
std::int64_t ref_oracle_pairs(std::int64_t n, const std::int64_t* id,
                              const double* pos, const double box[3],
                              double r_verlet, std::int64_t* out,
                              std::int64_t cap) {
  const FlatConfig fc = make_flat(n, id, nullptr, pos, nullptr, box);
  const auto pairs = oracle_pair_set(fc, r_verlet);
  const std::int64_t m = static_cast<std::int64_t>(pairs.size());
  for (std::int64_t k = 0; k < std::min(m, cap); ++k) {
    out[2 * k] = pairs[k].first;
    out[2 * k + 1] = pairs[k].second;
  }
  return m;
}

// autotune_subnodes (engine.hpp:316): returns the selected n_sub.
int ref_autotune(std::int64_t n, const std::int64_t* id, const double* mass,
                 const double* pos, const double* vel, const double box[3],
                 double eps, double sigma, double rc, int shifted,
                 double r_skin, int workers, double dt, int probe_steps,
                 int* selected, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const FlatConfig f = make_flat(n, id, mass, pos, vel, box);
    EngineConfig cfg;
    cfg.dt = dt;
    cfg.worker_threads = workers;
    const AutotuneReport rep = autotune_subnodes(
        f, make_inter(eps, sigma, rc, shifted), r_skin, cfg, probe_steps);
    *selected = rep.selected;
  });
}

}  // extern "C"
