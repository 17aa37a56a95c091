// taskmd_gpu::Engine — header-only C++ drop-in for taskmd::Engine
// (/root/reference/proj/include/taskmd/engine.hpp:66-290) backed by the B200
// engine through the C ABI in include/tmd_gpu.h (libtmd_gpu.so).
//
// Reference users switch by replacing the class name only:
//     taskmd::Engine     eng(taskmd::build_domain(flat, inter, r_skin, n_sub), cfg);
//     taskmd_gpu::Engine eng(taskmd::build_domain(flat, inter, r_skin, n_sub), cfg);
// (or skip the CPU build_domain: taskmd_gpu::Engine eng(flat, inter, r_skin,
// cfg)) and keep calling step() / run() / observe() / potential_energy() /
// timers() / step_count() / rebuild_count() / steal_count() / domain(). Errors come back as the
// reference's own exception types (taskmd::ConfigError / PhysicsError /
// StateError, errors.hpp:19-43), so the CLI's exit-code mapping
// (md_cli.cpp:333-352) holds unchanged.
//
// The reference's value types (FlatConfig, Interactions, EngineConfig,
// StepObservables, SectionTimers) are used as-is when this header is
// compiled with the reference headers on the include path (the default, and
// what a reference user has). Define TASKMD_GPU_STANDALONE to use the
// minimal look-alike types below instead (no reference headers needed).
#ifndef TASKMD_GPU_ENGINE_HPP_
#define TASKMD_GPU_ENGINE_HPP_

#include <algorithm>
#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "../tmd_gpu.h"

#ifndef TASKMD_GPU_STANDALONE
#include "taskmd/domain.hpp"
#include "taskmd/engine.hpp"
#include "taskmd/errors.hpp"
#include "taskmd/flat_config.hpp"
#include "taskmd/timers.hpp"
#else
#include <array>
#include <optional>
#include <stdexcept>
namespace taskmd {
struct Vec3 { double x = 0, y = 0, z = 0; };
struct BoxSpec { Vec3 length; };
struct Bond { std::int64_t a = 0, b = 0; };
struct Angle { std::int64_t i = 0, j = 0, k = 0; };
struct Topology { std::vector<Bond> bonds; std::vector<Angle> angles; };
struct FlatConfig {
  BoxSpec box;
  std::vector<std::int64_t> id;
  std::vector<std::int32_t> type;
  std::vector<double> mass;
  std::vector<Vec3> pos, vel;
  Topology topo;
  std::size_t size() const { return id.size(); }
};
struct LjParams { double epsilon = 1.0, sigma = 1.0, r_cut = 2.5; bool energy_shifted = true; };
struct FeneParams { double k = 30.0, r_max = 1.5; };
struct AngleParams { double k = 1.0, theta0 = 0.0; };
struct LangevinParams { double gamma = 1.0, temperature = 1.0; std::uint64_t seed = 0; };
struct Interactions { LjParams lj; std::optional<FeneParams> fene; std::optional<AngleParams> angle; };
struct EngineConfig {
  double dt = 0.005;
  std::int64_t steps = 0;
  std::optional<LangevinParams> thermostat;
  int n_sub = 1, worker_threads = 1;
  std::int64_t observable_stride = 100;
};
struct StepObservables { std::int64_t step = 0; double kinetic = 0, potential = 0, temperature = 0; };
enum class Section : std::size_t { kForces = 0, kComm = 1, kIntegrate = 2, kNeigh = 3, kResort = 4 };
struct SectionTimers {
  std::array<double, 5> seconds{};
  double elapsed = 0.0;
  double operator[](Section s) const { return seconds[static_cast<std::size_t>(s)]; }
  double section_sum() const { double t = 0; for (double s : seconds) t += s; return t; }
};
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PhysicsError : std::runtime_error { using std::runtime_error::runtime_error; };
struct VerifyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StateError : std::logic_error { using std::logic_error::logic_error; };
}  // namespace taskmd
#endif

namespace taskmd_gpu {

// GPU-only knobs (everything else comes from taskmd::EngineConfig).
struct GpuOptions {
  int device = -1;             // CUDA ordinal, -1 = current
  bool section_timers = true;  // per-phase CUDA-event timers (off: CUDA graphs)
  int nbr_capacity = 0;        // 0 = auto
  int variant = 0;             // 0 = default kernels
};

[[noreturn]] inline void throw_status(int rc, const std::string& msg) {
  switch (rc) {
    case TMD_ERR_CONFIG: throw taskmd::ConfigError(msg);
    case TMD_ERR_PHYSICS: throw taskmd::PhysicsError(msg);
    case TMD_ERR_VERIFY: throw taskmd::VerifyError(msg);
    case TMD_ERR_STATE: throw taskmd::StateError(msg);
    default: throw std::runtime_error("CUDA: " + msg);
  }
}

// The C-ABI view of a FlatConfig + Interactions + EngineConfig (arrays owned
// here; tmd_gpu_create* copies them).
struct CSystem {
  std::vector<double> pos, vel;
  std::vector<int64_t> bonds;  // Topology::bonds as (a, b) id pairs
  tmd_system sys{};
  tmd_lj_params lj{};
  tmd_fene_params fene{};
  bool has_fene = false;
  tmd_engine_params p{};

  CSystem(const taskmd::FlatConfig& flat, const taskmd::Interactions& inter, double r_skin,
          const taskmd::EngineConfig& cfg, const GpuOptions& opt) {
    if (inter.angle || !flat.topo.angles.empty()) {
      throw taskmd::ConfigError("angle terms are not on the GPU LJ path");
    }
    const std::size_t n = flat.size();
    pos.resize(3 * n);
    vel.resize(3 * n);
    for (std::size_t k = 0; k < n; ++k) {
      pos[3 * k] = flat.pos[k].x;
      pos[3 * k + 1] = flat.pos[k].y;
      pos[3 * k + 2] = flat.pos[k].z;
      vel[3 * k] = flat.vel[k].x;
      vel[3 * k + 1] = flat.vel[k].y;
      vel[3 * k + 2] = flat.vel[k].z;
    }
    sys.box[0] = flat.box.length.x;
    sys.box[1] = flat.box.length.y;
    sys.box[2] = flat.box.length.z;
    sys.n = static_cast<int64_t>(n);
    sys.id = flat.id.data();
    sys.type = flat.type.empty() ? nullptr : flat.type.data();
    sys.mass = flat.mass.empty() ? nullptr : flat.mass.data();
    sys.pos = pos.data();
    sys.vel = vel.data();
    bonds.reserve(2 * flat.topo.bonds.size());
    for (const auto& b : flat.topo.bonds) {
      bonds.push_back(b.a);
      bonds.push_back(b.b);
    }
    sys.n_bonds = static_cast<int64_t>(flat.topo.bonds.size());
    sys.bonds = bonds.empty() ? nullptr : bonds.data();
    if (inter.fene) {
      fene = tmd_fene_params{inter.fene->k, inter.fene->r_max};
      has_fene = true;
    }
    lj = tmd_lj_params{inter.lj.epsilon, inter.lj.sigma, inter.lj.r_cut,
                       inter.lj.energy_shifted ? 1 : 0};
    p.dt = cfg.dt;
    p.r_skin = r_skin;
    p.device = opt.device;
    p.section_timers = opt.section_timers ? 1 : 0;
    p.nbr_capacity = opt.nbr_capacity;
    p.reserved[0] = opt.variant;
    if (cfg.thermostat) {
      p.thermostat = 1;
      p.gamma = cfg.thermostat->gamma;
      p.temperature = cfg.thermostat->temperature;
      p.seed = cfg.thermostat->seed;
    }
  }
  const tmd_fene_params* fene_ptr() const { return has_fene ? &fene : nullptr; }
};

class Engine {
 public:
  // build_domain(flat, inter, r_skin, n_sub) + Engine(domain, cfg)
  // (domain.hpp:134-189, engine.hpp:68-77). n_sub / worker_threads have no
  // GPU meaning and are ignored; angle terms are rejected with ConfigError.
  // FENE bonds and a thermostat run on the device.
  Engine(const taskmd::FlatConfig& flat, const taskmd::Interactions& inter, double r_skin,
         const taskmd::EngineConfig& cfg, const GpuOptions& opt = {})
      : cfg_(cfg), inter_(inter), r_skin_(r_skin) {
    CSystem cs(flat, inter, r_skin, cfg, opt);
    const int rc = tmd_gpu_create(&cs.sys, &cs.lj, cs.fene_ptr(), &cs.p, &ctx_);
    if (rc != TMD_OK) throw_status(rc, tmd_gpu_last_error(nullptr));
    box_ = flat.box;
    topo_ = flat.topo;
  }

#ifndef TASKMD_GPU_STANDALONE
  // Engine(Domain, EngineConfig) (engine.hpp:68-77): the domain a caller
  // assembled with build_domain is flattened (flatten_domain, domain.hpp:
  // 193-207: ids, types, masses, wrapped positions, velocities, topology) and
  // rebuilt on the device with its own interactions and skin.
  Engine(taskmd::Domain domain, const taskmd::EngineConfig& cfg, const GpuOptions& opt = {})
      : Engine(taskmd::flatten_domain(domain), domain.inter, domain.r_skin, cfg, opt) {}

  // Engine::domain() (engine.hpp:142-143) for callers that read the stores
  // (md_cli.cpp:226-250, acceptance.cpp:53-64): a reference Domain rebuilt on
  // the host from the current device state (build_domain over flatten(), with
  // EngineConfig::n_sub subnodes), every owned slot's force set to the
  // device's last evaluation. Its neighbour lists are the reference's at the
  // current positions. Cached until the next step.
  const taskmd::Domain& domain() const {
    if (!dom_ || dom_step_ != step_count()) {
      const taskmd::FlatConfig f = flatten();
      auto d = std::make_unique<taskmd::Domain>(
          taskmd::build_domain(f, inter_, r_skin_, std::max(1, cfg_.n_sub)));
      const auto fr = forces();  // sorted by id
      for (taskmd::Subnode& sn : d->subs) {
        for (std::int32_t cidx : sn.interior) {
          const taskmd::CellSpan& span = sn.store.cells[static_cast<std::size_t>(cidx)];
          for (std::size_t k = span.begin; k < span.begin + span.real; ++k) {
            const auto it = std::lower_bound(
                fr.begin(), fr.end(), sn.store.id[k],
                [](const std::pair<std::int64_t, taskmd::Vec3>& a, std::int64_t v) {
                  return a.first < v;
                });
            sn.store.fx[k] = it->second.x;
            sn.store.fy[k] = it->second.y;
            sn.store.fz[k] = it->second.z;
          }
        }
      }
      dom_ = std::move(d);
      dom_step_ = step_count();
    }
    return *dom_;
  }
#endif

  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept
      : ctx_(std::exchange(o.ctx_, nullptr)), cfg_(o.cfg_), inter_(o.inter_),
        r_skin_(o.r_skin_), box_(o.box_), topo_(std::move(o.topo_)) {}
  ~Engine() { tmd_gpu_destroy(ctx_); }

  void step() { run(1); }
  void run(std::int64_t steps) { check(tmd_gpu_step(ctx_, steps)); }

  taskmd::StepObservables observe() const {
    tmd_observables o{};
    check(tmd_gpu_observe(ctx_, &o));
    taskmd::StepObservables r;
    r.step = o.step;
    r.kinetic = o.kinetic;
    r.potential = o.potential;
    r.temperature = o.temperature;
    return r;
  }
  double virial() const {
    tmd_observables o{};
    check(tmd_gpu_observe(ctx_, &o));
    return o.virial;
  }

  const taskmd::EngineConfig& config() const { return cfg_; }
  taskmd::SectionTimers timers() const {
    taskmd::SectionTimers t;
    double sec[5], el = 0.0;
    check(tmd_gpu_timers(ctx_, sec, &el));
    for (int k = 0; k < 5; ++k) t.seconds[k] = sec[k];
    t.elapsed = el;
    return t;
  }
  std::int64_t step_count() const { return tmd_gpu_step_count(ctx_); }
  double potential_energy() const { return observe().potential; }
  std::uint64_t rebuild_count() const { return tmd_gpu_rebuild_count(ctx_); }
  std::uint64_t steal_count() const { return 0; }  // no work-stealing pool on the GPU

  // flatten_domain (domain.hpp:193-207): sorted by id, positions wrapped,
  // each particle's type and mass as created.
  taskmd::FlatConfig flatten() const {
    const std::size_t n = static_cast<std::size_t>(tmd_gpu_size(ctx_));
    std::vector<std::int64_t> id(n);
    std::vector<double> pos(3 * n), vel(3 * n);
    taskmd::FlatConfig f;
    f.type.resize(n);
    f.mass.resize(n);
    check(tmd_gpu_download(ctx_, id.data(), pos.data(), vel.data(), nullptr, f.type.data(),
                           f.mass.data()));
    f.box = box_;
    f.topo = topo_;
    f.id.assign(id.begin(), id.end());
    f.pos.resize(n);
    f.vel.resize(n);
    for (std::size_t k = 0; k < n; ++k) {
      f.pos[k] = {pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]};
      f.vel[k] = {vel[3 * k], vel[3 * k + 1], vel[3 * k + 2]};
    }
    return f;
  }

  // Forces of the last evaluation, sorted by id (the interior_forces helper
  // of the reference tests, acceptance.cpp:53-64).
  std::vector<std::pair<std::int64_t, taskmd::Vec3>> forces() const {
    const std::size_t n = static_cast<std::size_t>(tmd_gpu_size(ctx_));
    std::vector<std::int64_t> id(n);
    std::vector<double> f(3 * n);
    check(tmd_gpu_download(ctx_, id.data(), nullptr, nullptr, f.data(), nullptr, nullptr));
    std::vector<std::pair<std::int64_t, taskmd::Vec3>> out(n);
    for (std::size_t k = 0; k < n; ++k) out[k] = {id[k], {f[3 * k], f[3 * k + 1], f[3 * k + 2]}};
    return out;
  }

  // Sorted (min id, max id) listed pairs (test_neighbor.cpp:49-65).
  std::vector<std::pair<std::int64_t, std::int64_t>> listed_pairs() const {
    size_t m = 0;
    check(tmd_gpu_pairs(ctx_, nullptr, 0, &m));
    std::vector<std::int64_t> raw(2 * m + 2);
    check(tmd_gpu_pairs(ctx_, raw.data(), m, &m));
    std::vector<std::pair<std::int64_t, std::int64_t>> out(m);
    for (size_t k = 0; k < m; ++k) out[k] = {raw[2 * k], raw[2 * k + 1]};
    return out;
  }

  tmd_gpu_ctx* handle() const { return ctx_; }

 private:
  void check(int rc) const {
    if (rc != TMD_OK) throw_status(rc, tmd_gpu_last_error(ctx_));
  }

  tmd_gpu_ctx* ctx_ = nullptr;
  taskmd::EngineConfig cfg_;
  taskmd::Interactions inter_;
  double r_skin_ = 0.0;
  taskmd::BoxSpec box_;
  taskmd::Topology topo_;
#ifndef TASKMD_GPU_STANDALONE
  mutable std::unique_ptr<taskmd::Domain> dom_;
  mutable std::int64_t dom_step_ = -1;
#endif
};

using NcclId = std::array<unsigned char, 128>;

// ncclGetUniqueId, on one rank; the caller broadcasts the bytes (MPI_Bcast,
// torch.distributed, a file...).
inline NcclId nccl_unique_id() {
  NcclId id{};
  const int rc = tmd_nccl_unique_id(id.data());
  if (rc != TMD_OK) throw_status(rc, tmd_gpu_last_error(nullptr));
  return id;
}

// One GPU's slab of an N-GPU run, one process per GPU: the
// native step loop with NCCL on the context stream and the fused halo
// (tmd_slab_nccl.cuh). Every rank passes the whole system and the same
// NcclId; run / observe are collective.
class SlabEngine {
 public:
  SlabEngine(const taskmd::FlatConfig& flat, const taskmd::Interactions& inter, double r_skin,
             const taskmd::EngineConfig& cfg, int rank, int nranks, const NcclId& id,
             const GpuOptions& opt = {}, bool load_balance = false)
      : n_total_(static_cast<int64_t>(flat.size())), box_(flat.box) {
    CSystem cs(flat, inter, r_skin, cfg, opt);
    int rc = tmd_gpu_create_slab(&cs.sys, &cs.lj, cs.fene_ptr(), &cs.p, rank, nranks, &ctx_);
    if (rc != TMD_OK) throw_status(rc, tmd_gpu_last_error(nullptr));
    check(tmd_gpu_slab_attach_nccl(ctx_, id.data(), (load_balance ? 1 : 0) | 2));
    check(tmd_gpu_slab_setup(ctx_));
  }
  SlabEngine(const SlabEngine&) = delete;
  SlabEngine& operator=(const SlabEngine&) = delete;
  ~SlabEngine() { tmd_gpu_destroy(ctx_); }

  void step() { run(1); }
  void run(std::int64_t steps) { check(tmd_gpu_slab_run(ctx_, steps)); }

  // Engine::observe over the whole system (an all-reduce: collective).
  taskmd::StepObservables observe() const {
    tmd_observables o{};
    check(tmd_gpu_slab_observe(ctx_, n_total_, &o));
    taskmd::StepObservables r;
    r.step = o.step;
    r.kinetic = o.kinetic;
    r.potential = o.potential;
    r.temperature = o.temperature;
    return r;
  }
  std::int64_t step_count() const { return tmd_gpu_step_count(ctx_); }
  std::uint64_t rebuild_count() const { return tmd_gpu_rebuild_count(ctx_); }
  // Engine::timers (engine.hpp:145) of this rank's stream (CUDA-event phases
  // of the native loop; GpuOptions::section_timers = false leaves only elapsed).
  taskmd::SectionTimers timers() const {
    taskmd::SectionTimers t;
    double sec[5], el = 0.0;
    check(tmd_gpu_timers(ctx_, sec, &el));
    for (int k = 0; k < 5; ++k) t.seconds[k] = sec[k];
    t.elapsed = el;
    return t;
  }

  // The particles this slab owns, sorted by id, positions wrapped, types and
  // masses as created.
  taskmd::FlatConfig local() const {
    const std::size_t n = static_cast<std::size_t>(tmd_gpu_size(ctx_));
    std::vector<std::int64_t> id(n);
    std::vector<double> pos(3 * n), vel(3 * n);
    taskmd::FlatConfig f;
    f.type.resize(n);
    f.mass.resize(n);
    check(tmd_gpu_download(ctx_, id.data(), pos.data(), vel.data(), nullptr, f.type.data(),
                           f.mass.data()));
    f.box = box_;
    f.id.assign(id.begin(), id.end());
    f.pos.resize(n);
    f.vel.resize(n);
    for (std::size_t k = 0; k < n; ++k) {
      f.pos[k] = {pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]};
      f.vel[k] = {vel[3 * k], vel[3 * k + 1], vel[3 * k + 2]};
    }
    return f;
  }

 private:
  void check(int rc) const {
    if (rc != TMD_OK) throw_status(rc, tmd_gpu_last_error(ctx_));
  }

  tmd_gpu_ctx* ctx_ = nullptr;
  std::int64_t n_total_ = 0;
  taskmd::BoxSpec box_;
};

}  // namespace taskmd_gpu

#endif  // TASKMD_GPU_ENGINE_HPP_
