// TEST PROGRAM — the drop-in check of include/taskmd_gpu/engine.hpp.
//
// Runs the UNMODIFIED reference engine (taskmd::build_domain + taskmd::Engine,
// compiled from /root/reference/proj/include) and taskmd_gpu::Engine side by
// side through the reference's own types, mirroring acceptance.cpp's
// criteria 1-3 and the reference's engine tests. One verdict line per check;
// exit 0 only if all hold. Built by tests/cpp/Makefile into tests/cpp/_bin/.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "taskmd/domain.hpp"
#include "taskmd/engine.hpp"
#include "taskmd/generators.hpp"
#include "taskmd/oracle.hpp"
#include "taskmd_gpu/engine.hpp"

using namespace taskmd;

static int g_fail = 0;

static void verdict(const char* name, bool ok, const std::string& detail) {
  std::printf("%-44s %s  %s\n", name, ok ? "PASS" : "FAIL", detail.c_str());
  if (!ok) ++g_fail;
}

static Interactions lj_only() {
  Interactions inter;
  inter.lj = LjParams{1.0, 1.0, 2.5, true};
  return inter;
}

static std::vector<std::pair<std::int64_t, std::int64_t>> ref_pairs(const Domain& d) {
  std::vector<std::pair<std::int64_t, std::int64_t>> p;
  for (int s = 0; s < d.n_sub(); ++s) {
    const SoaStore& st = d.subs[s].store;
    const SortedNeighborList& nl = d.nlists[s];
    for (std::size_t n = 0; n < nl.ilist.size(); ++n) {
      const std::int64_t a = st.id[nl.ilist[n]];
      for (std::int32_t j = nl.irange[n].first; j < nl.irange[n].second; ++j) {
        const std::int64_t b = st.id[nl.jlist[j]];
        if (b != SoaStore::kSentinelId) p.emplace_back(std::min(a, b), std::max(a, b));
      }
    }
  }
  std::sort(p.begin(), p.end());
  return p;
}

int main() {
  // criterion 1: 10 random configs, forces vs oracle <= 1e-10, pair sets equal
  {
    double worst = 0.0;
    int equal = 0;
    for (std::uint64_t seed = 1; seed <= 10; ++seed) {
      const FlatConfig flat = gen_random(500, 0.8442, 0.8, 0.72, seed);
      EngineConfig cfg;
      taskmd_gpu::Engine g(flat, lj_only(), 0.3, cfg);
      const OracleResult want = oracle_forces_energy(flat, lj_only());
      std::map<std::int64_t, std::size_t> row;
      for (std::size_t k = 0; k < flat.size(); ++k) row[flat.id[k]] = k;
      for (const auto& [id, f] : g.forces()) {
        const Vec3& w = want.force[row[id]];
        worst = std::max({worst, std::abs(f.x - w.x), std::abs(f.y - w.y), std::abs(f.z - w.z)});
      }
      if (g.listed_pairs() == oracle_pair_set(flat, 2.8)) ++equal;
    }
    verdict("criterion 1 (random N=500 x10)", worst <= 1e-10 && equal == 10,
            "worst |dF| " + std::to_string(worst) + ", pair sets equal " +
                std::to_string(equal) + "/10");
  }
  // same pair multiset as the reference engine's own lists
  {
    const FlatConfig flat = gen_lattice(4096, 0.8442, 0.72, 11);
    Domain d = build_domain(flat, lj_only(), 0.3, 8);
    const auto want = ref_pairs(d);
    EngineConfig cfg;
    taskmd_gpu::Engine g(flat, lj_only(), 0.3, cfg);
    verdict("listed pairs == reference lists (n_sub 8)", g.listed_pairs() == want,
            std::to_string(want.size()) + " pairs");
  }
  // criterion 2: one NVE step within 1e-10 of the reference
  {
    const FlatConfig flat = gen_lattice(4096, 0.8442, 0.72, 11);
    EngineConfig cfg;
    cfg.dt = 0.005;
    cfg.n_sub = 8;
    Engine ref(build_domain(flat, lj_only(), 0.3, 8), cfg);
    ref.run(1);
    const FlatConfig a = flatten_domain(ref.domain());
    taskmd_gpu::Engine g(flat, lj_only(), 0.3, cfg);
    g.run(1);
    const FlatConfig b = g.flatten();
    double worst = 0.0;
    bool ids = a.id == b.id;
    for (std::size_t k = 0; ids && k < a.size(); ++k) {
      worst = std::max({worst, std::abs(a.pos[k].x - b.pos[k].x),
                        std::abs(a.pos[k].y - b.pos[k].y), std::abs(a.pos[k].z - b.pos[k].z)});
    }
    verdict("criterion 2 (one step vs reference)", ids && worst <= 1e-10,
            "max position spread " + std::to_string(worst));
  }
  // thermostat: the same EngineConfig (with a Langevin bath) through both
  // engines, 30 steps (test_engine.cpp:214-240's system and bath)
  {
    const FlatConfig flat = gen_lattice(4096, 0.8442, 0.0, 29);
    EngineConfig cfg;
    cfg.dt = 0.005;
    cfg.n_sub = 8;
    LangevinParams bath;
    bath.gamma = 1.0;
    bath.temperature = 0.8;
    bath.seed = 99;
    cfg.thermostat = bath;
    Engine ref(build_domain(flat, lj_only(), 0.3, 8), cfg);
    ref.run(30);
    const FlatConfig a = flatten_domain(ref.domain());
    taskmd_gpu::Engine g(flat, lj_only(), 0.3, cfg);
    g.run(30);
    const FlatConfig b = g.flatten();
    double worst = 0.0;
    bool ids = a.id == b.id;
    for (std::size_t k = 0; ids && k < a.size(); ++k) {
      worst = std::max({worst, std::abs(a.pos[k].x - b.pos[k].x),
                        std::abs(a.pos[k].y - b.pos[k].y), std::abs(a.pos[k].z - b.pos[k].z),
                        std::abs(a.vel[k].x - b.vel[k].x), std::abs(a.vel[k].y - b.vel[k].y),
                        std::abs(a.vel[k].z - b.vel[k].z)});
    }
    verdict("Langevin bath, 30 steps vs reference", ids && worst <= 1e-9,
            "max state spread " + std::to_string(worst));
  }
  // FENE chains (Kremer-Grest interactions): boustrophedon chains on a
  // jittered lattice, the reference's Topology + FeneParams through both
  // engines, 50 steps
  {
    FlatConfig flat = gen_lattice(1000, 0.85, 1.0, 5);
    // one chain per z plane of the 10^3 lattice (ids x-fastest), snaking in y
    for (int z = 0; z < 10; ++z) {
      for (int j = 0; j + 1 < 100; ++j) {
        auto at = [z](int k) {
          const int y = k / 10, xi = k % 10, x = (y % 2 == 0) ? xi : 9 - xi;
          return static_cast<std::int64_t>(x + 10 * (y + 10 * z));
        };
        flat.topo.bonds.push_back({at(j), at(j + 1)});
      }
    }
    Interactions inter = lj_only();
    inter.lj.r_cut = std::pow(2.0, 1.0 / 6.0);
    inter.fene = FeneParams{30.0, 1.5};
    EngineConfig cfg;
    cfg.dt = 0.004;
    cfg.n_sub = 8;
    Engine ref(build_domain(flat, inter, 0.4, 8), cfg);
    ref.run(50);
    const FlatConfig a = flatten_domain(ref.domain());
    taskmd_gpu::Engine g(flat, inter, 0.4, cfg);
    g.run(50);
    const FlatConfig b = g.flatten();
    double worst = 0.0;
    bool ids = a.id == b.id && b.topo.bonds.size() == flat.topo.bonds.size();
    for (std::size_t k = 0; ids && k < a.size(); ++k) {
      worst = std::max({worst, std::abs(a.pos[k].x - b.pos[k].x),
                        std::abs(a.pos[k].y - b.pos[k].y), std::abs(a.pos[k].z - b.pos[k].z)});
    }
    const double pe_a = ref.potential_energy(), pe_b = g.potential_energy();
    verdict("FENE chains (KG), 50 steps vs reference",
            ids && worst <= 1e-9 && std::abs(pe_a - pe_b) <= 1e-10 * std::abs(pe_a),
            "max position spread " + std::to_string(worst) + ", PE " + std::to_string(pe_a) +
                " / " + std::to_string(pe_b));
  }
  // taskmd_gpu::SlabEngine (one process per GPU; here one slab exchanging
  // its halo with itself through NCCL and the fused peer-store halo) against
  // the reference engine, 40 steps
  {
    const FlatConfig flat = gen_lattice(8000, 0.8442, 0.9, 17);
    EngineConfig cfg;
    cfg.dt = 0.005;
    cfg.n_sub = 8;
    Engine ref(build_domain(flat, lj_only(), 0.3, 8), cfg);
    ref.run(40);
    const FlatConfig a = flatten_domain(ref.domain());
    taskmd_gpu::SlabEngine g(flat, lj_only(), 0.3, cfg, 0, 1, taskmd_gpu::nccl_unique_id());
    g.run(40);
    const FlatConfig b = g.local();
    double worst = 0.0;
    bool ids = a.id == b.id;
    for (std::size_t k = 0; ids && k < a.size(); ++k) {
      worst = std::max({worst, std::abs(a.pos[k].x - b.pos[k].x),
                        std::abs(a.pos[k].y - b.pos[k].y), std::abs(a.pos[k].z - b.pos[k].z)});
    }
    const double pe_a = ref.potential_energy(), pe_b = g.observe().potential;
    verdict("SlabEngine (NCCL, fused halo), 40 steps", ids && worst <= 1e-9 &&
                std::abs(pe_a - pe_b) <= 1e-10 * std::abs(pe_a),
            "max position spread " + std::to_string(worst) + ", rebuilds " +
                std::to_string(g.rebuild_count()) + " / " + std::to_string(ref.rebuild_count()));
  }
  // Engine(Domain, EngineConfig) + domain() + flatten() with mixed types and
  // masses: the class-name-only switch of a reference caller
  {
    FlatConfig flat = gen_lattice(4096, 0.8442, 0.72, 11);
    for (std::size_t k = 0; k < flat.size(); ++k) {
      flat.type[k] = static_cast<std::int32_t>(k % 4);
      flat.mass[k] = 1.0 + 0.5 * static_cast<double>(k % 3);
    }
    EngineConfig cfg;
    cfg.dt = 0.005;
    cfg.n_sub = 8;
    Engine ref(build_domain(flat, lj_only(), 0.3, 8), cfg);
    taskmd_gpu::Engine g(build_domain(flat, lj_only(), 0.3, 8), cfg);
    ref.run(25);
    g.run(25);
    const FlatConfig a = flatten_domain(ref.domain());
    const FlatConfig b = g.flatten();
    const FlatConfig c = flatten_domain(g.domain());
    bool same = a.id == b.id && a.type == b.type && a.mass == b.mass && c.id == a.id &&
                c.type == a.type && c.mass == a.mass;
    double worst = 0.0;
    for (std::size_t k = 0; k < a.size() && same; ++k) {
      worst = std::max({worst, std::abs(a.pos[k].x - b.pos[k].x), std::abs(a.vel[k].y - b.vel[k].y),
                        std::abs(c.pos[k].z - b.pos[k].z)});
    }
    // forces read from the stores, as md_cli.cpp:230-240 does
    std::map<std::int64_t, Vec3> fr, fg;
    const Domain* doms[2] = {&ref.domain(), &g.domain()};
    for (const Domain* d : doms) {
      auto& dst = d == doms[0] ? fr : fg;
      for (const Subnode& sn : d->subs) {
        for (std::int32_t cidx : sn.interior) {
          const CellSpan& span = sn.store.cells[cidx];
          for (std::size_t k = span.begin; k < span.begin + span.real; ++k) {
            dst[sn.store.id[k]] = sn.store.force(k);
          }
        }
      }
    }
    double fworst = 0.0, fscale = 0.0;
    for (const auto& [id, f] : fr) {
      const Vec3& h = fg.at(id);
      fscale = std::max({fscale, std::abs(f.x), std::abs(f.y), std::abs(f.z)});
      fworst = std::max({fworst, std::abs(f.x - h.x), std::abs(f.y - h.y), std::abs(f.z - h.z)});
    }
    verdict("Engine(Domain) + domain() + flatten (types, masses)",
            same && worst <= 1e-9 && fr.size() == flat.size() && fworst <= 1e-8 * fscale,
            "ids/types/masses equal " + std::to_string(same) + ", max |dx| " +
                std::to_string(worst) + ", max |dF| " + std::to_string(fworst));
  }
  // criterion 3: NVE drift, N=4000 SC lattice, seed 3, T=0.6
  {
    const FlatConfig flat = gen_lattice(4000, 0.8442, 0.6, 3);
    double drift[2];
    const double dts[2] = {0.005, 0.001};
    for (int v = 0; v < 2; ++v) {
      EngineConfig cfg;
      cfg.dt = dts[v];
      taskmd_gpu::Engine g(flat, lj_only(), 0.3, cfg);
      const StepObservables o0 = g.observe();
      const double e0 = o0.kinetic + o0.potential;
      double worst = 0.0;
      for (int c = 0; c < 100; ++c) {
        g.run(10);
        const StepObservables o = g.observe();
        worst = std::max(worst, std::abs(o.kinetic + o.potential - e0) / std::abs(e0));
      }
      drift[v] = worst;
    }
    verdict("criterion 3 (NVE drift, 2nd order)", drift[0] <= 1e-3 && drift[0] / drift[1] >= 10,
            "drift " + std::to_string(drift[0]) + " / " + std::to_string(drift[1]));
  }
  // error mapping: coincident particles -> taskmd::PhysicsError
  {
    FlatConfig f;
    f.box = BoxSpec::cubic(8.5);
    ParticleRec a, b;
    a.id = 0;
    a.pos = {4.0, 4.0, 4.0};
    b.id = 1;
    b.pos = {4.0, 4.0, 4.0};
    f.push(a);
    f.push(b);
    bool caught = false;
    try {
      EngineConfig cfg;
      taskmd_gpu::Engine g(f, lj_only(), 0.3, cfg);
    } catch (const PhysicsError&) {
      caught = true;
    }
    verdict("overlap -> taskmd::PhysicsError", caught, "");
  }
  // error mapping: bad box -> taskmd::ConfigError
  {
    FlatConfig f;
    f.box = BoxSpec{{2.0, 10.0, 10.0}};
    ParticleRec a;
    a.id = 0;
    f.push(a);
    bool caught = false;
    try {
      EngineConfig cfg;
      taskmd_gpu::Engine g(f, lj_only(), 0.3, cfg);
    } catch (const ConfigError&) {
      caught = true;
    }
    verdict("thin box -> taskmd::ConfigError", caught, "");
  }
  std::printf(g_fail == 0 ? "all drop-in checks hold\n" : "%d drop-in checks failed\n", g_fail);
  return g_fail == 0 ? 0 : 1;
}
