// Device-side building blocks of the B200 LJ short-range path.
//
// Layout in HBM (one context = one GPU = one cell-sorted particle set):
//   pos   double4[N]  x, y, z, (w unused)  — one 32-B sector per gathered j
//   vel   double[3][N] SoA, force double[3][N] SoA, mass double[N], id int64[N]
//   cell  int32[N]    global cell of each particle at the last resort
//   start int32[ncells+1] cell ranges (counting sort output)
//   nbr   uint32[cap][stride] full Verlet list, ELL-transposed: entry k of
//         particle i lives at nbr[k*stride + i] so a warp reads 128 B per k
//   nnbr  int32[N]    entries per particle (unpadded)
//
// A list entry packs the neighbour slot (low 25 bits) with the periodic image
// that the reference engine would have used for the same pair (bits 25..31),
// so that every squared distance below is rounded exactly like the reference's
// (neighbor_list.hpp:82-83, 94-95, 161-164):
//   bits 25-26 / 27-28 / 29-30: image shift on x / y / z (0 none, 1 +L, 2 -L)
//                               of neighbour j as seen from particle i;
//   bit  31: the reference evaluates this pair from j's side (j's cell is the
//            half-stencil source, neighbor_list.hpp:35-44), i.e. it forms the
//            image of i (x_i - s) rather than of j (x_j + s), and the
//            difference is taken as (x_i - s) - x_j.
// With no shift both forms are plain x_i - x_j; negation is exact, so the
// squared distance is bit-identical to the reference in every case.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tmd {

constexpr int kIdxBits = 25;
constexpr uint32_t kIdxMask = (1u << kIdxBits) - 1u;
constexpr uint32_t kFlagIUpper = 1u << 31;
constexpr int64_t kMaxSlots = (int64_t{1} << kIdxBits) - 1;

// Status bits in Ctrl::status (mapped to taskmd exception types on the host).
enum : int {
  kStatOverlap = 1,      // r2 == 0 (neighbor_list.hpp:166-170) -> PhysicsError
  kStatNonFinite = 2,    // non-finite v/f (engine.hpp:231-236) -> PhysicsError
  kStatNonFinitePos = 4, // non-finite position at binning (domain.hpp:58-62)
  kStatOverflow = 8,     // neighbour list capacity exceeded -> host re-runs
  kStatStageOverflow = 16,  // a brick halo exceeded the staging capacity -> grow
  kStatStray = 32,       // slab mode: a particle outside the slab at binning (bug)
  kStatBondReach = 64,   // bonded partner not among the reachable slots (bonded.hpp:51-57)
  kStatBondStretch = 128,  // FENE bond at or beyond r_max (bonded.hpp:184-191)
};

constexpr int kMaxBonds = 8;  // bonds per particle (linear chains: 2)

struct LjConst {
  double sigma2, rc2, eps4, eps24, shift;  // lj_prepare (potentials.hpp:49-61)
  double fcap;  // > 0: cap |F_pair| (overlap warm-up only; thread-per-particle kernel)
};

struct Geom {
  double L[3];
  double cell_len[3];
  int dims[3];       // GLOBAL cell grid (build_cell_grid)
  int ncells;        // local cells: dims[0]*dims[1]*ldz
  double rv2;        // (r_cut + r_skin)^2, rounded as build_sorted_list does
  double rebuild_thr;  // 0.25 * r_skin * r_skin (needs_rebuild, nl.hpp:143)
  // z-slab decomposition (multi-GPU). zslab = 0: the context owns
  // the whole periodic box (local grid = global grid). zslab = 1: it owns
  // global z-layers [z0, z0 + zown); local layer lz = global - z0 + 1, and
  // local layers 0 and zown + 1 are ghost layers holding copies of the
  // neighbour slabs' boundary layers, with image codes zcode_lo / zcode_hi
  // (the reference's ghost shift when the layer wraps the box, subnode.hpp:84-90).
  int zslab;
  int z0, zown, ldz;
  unsigned int zcode_lo, zcode_hi;
  int owned_cells;   // dims[0]*dims[1]*zown (cells ranked before the ghost layers)
};

// Local cell of a global cell (owned region; slab mode shifts z by one layer).
__host__ __device__ __forceinline__ int local_cell(const Geom& g, int gcell) {
  if (!g.zslab) return gcell;
  const int dxy = g.dims[0] * g.dims[1];
  const int cz = gcell / dxy;
  return gcell - cz * dxy + (cz - g.z0 + 1) * dxy;
}

// Device control block: rebuild decision, counters and the error record.
struct Ctrl {
  unsigned long long max_d2;  // bits of max |x - x_snap|^2 this step (>= 0)
  int rebuild;                // decision for the current step
  int force_rebuild;          // set by the host (setup / rollback)
  long long step;             // device step counter (== host step count)
  long long rebuilds;         // list rebuilds (Engine::rebuild_count)
  int status;                 // OR of kStat* bits
  int err_lock;
  long long err_step;
  long long err_id0, err_id1;
  int max_count;              // largest per-particle entry count, last build
  int cap;                    // current list capacity per particle
  long long entries;          // total entries, last build
  int max_halo;               // largest staged halo seen (slots)
  int err_bit;                // status bit of the first error (its record below)
  double err_val;             // a value for the first error's message (bond r^2)
  int obs_rows;               // observable rows recorded in this chunk (run_observed)
  int halt;                   // native slab loop: a rebuild is due, later steps are no-ops
  double seen_d2;             // native slab loop: the global max |x - x_snap|^2 the last
                              // decision saw (the host sizes its next batch from it)
  long long tick_base;        // section timers in graph mode: step count at the chunk
                              // start (phase ticks are indexed by step - tick_base)
  unsigned long long occ_s2;  // sum over owned cells of (particles in the cell)^2 (k_occupancy)
};

// Section timers without host round trips (graph mode, the native slab loop):
// single-thread kernels of the step stamp %globaltimer into per-step phase
// slots; the host turns consecutive stamps into the five SectionTimers.
constexpr int kTickSteps = 256;      // steps a tick buffer holds (== a chunk)
constexpr int kTickPhases = 4;       // per step: block start, decide, list build, forces
enum : int { kTickBlock = 0, kTickDecide = 1, kTickBuild = 2, kTickForces = 3 };

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Stamps phase `ph` of the chunk-relative step ctrl->step - tick_base + off.
__device__ __forceinline__ void stamp(const Ctrl* ctrl, long long* ticks, int ph, int off) {
  if (!ticks) return;
  const long long s = ctrl->step - ctrl->tick_base + off;
  if (s >= 0 && s < kTickSteps) ticks[s * kTickPhases + ph] = global_ns();
}

// ---------------------------------------------------------------------------
// Exact (non-contracted) FP64 helpers. nvcc contracts a*b+c into DFMA by
// default; the reference's g++ build (no -march) never does, so every
// expression that decides a discrete outcome (wrap, cell, list membership,
// cutoff test, rebuild test) is spelled with _rn intrinsics.

__device__ __forceinline__ double exact_r2(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                   __dmul_rn(dz, dz));
}

// wrap1 (box.hpp:47-51): r = p - L*floor(p/L); r >= L folds back.
__device__ __forceinline__ double wrap1(double p, double L) {
  double r = __dsub_rn(p, __dmul_rn(L, floor(__ddiv_rn(p, L))));
  if (r >= L) r = __dsub_rn(r, L);
  return r;
}

// CellGrid::cell_coords (cell_grid.hpp:36-46), one axis.
__device__ __forceinline__ int cell_coord(double p, double len, int dims) {
  int v = static_cast<int>(floor(__ddiv_rn(p, len)));
  if (v < 0) v = 0;
  if (v >= dims) v = dims - 1;
  return v;
}

__device__ __forceinline__ double image_shift(uint32_t code2, double L) {
  return code2 == 0u ? 0.0 : (code2 == 1u ? L : -L);
}

// Displacement d = x_i - x_j(image) exactly as the reference rounds it for the
// pair encoded in `ent` (see the header comment).
__device__ __forceinline__ void pair_delta(const double4& pi, const double4& pj,
                                           uint32_t ent, const Geom& g,
                                           double& dx, double& dy, double& dz) {
  if (ent <= kIdxMask) {
    dx = __dsub_rn(pi.x, pj.x);
    dy = __dsub_rn(pi.y, pj.y);
    dz = __dsub_rn(pi.z, pj.z);
    return;
  }
  const double sx = image_shift((ent >> 25) & 3u, g.L[0]);
  const double sy = image_shift((ent >> 27) & 3u, g.L[1]);
  const double sz = image_shift((ent >> 29) & 3u, g.L[2]);
  if (ent & kFlagIUpper) {
    dx = __dsub_rn(__dsub_rn(pi.x, sx), pj.x);
    dy = __dsub_rn(__dsub_rn(pi.y, sy), pj.y);
    dz = __dsub_rn(__dsub_rn(pi.z, sz), pj.z);
  } else {
    dx = __dsub_rn(pi.x, __dadd_rn(pj.x, sx));
    dy = __dsub_rn(pi.y, __dadd_rn(pj.y, sy));
    dz = __dsub_rn(pi.z, __dadd_rn(pj.z, sz));
  }
}

// 1/x from the MUFU.RCP64H seed plus two Newton steps (~1 ulp). Used only in
// the force arithmetic (tolerance 1e-10 relative), never in a discrete test.
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  return y;
}

// Read-only 32-B gather of one packed position (two LDG.128 on one sector).
__device__ __forceinline__ double4 ldg_pos(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// The same gather as ONE 256-bit load (sm_100: LDG.E.ENL2.256.CONSTANT), so a
// lane's 32-B sector is requested once instead of twice.
__device__ __forceinline__ double4 ldg_pos256(const double4* p) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ bool finite3(double a, double b, double c) {
  return isfinite(a) && isfinite(b) && isfinite(c);
}

// First error wins the detail record; every error ORs its status bit.
__device__ __forceinline__ void record_error(Ctrl* ctrl, int bit, long long id0,
                                             long long id1, double val = 0.0) {
  atomicOr(&ctrl->status, bit);
  if (atomicCAS(&ctrl->err_lock, 0, 1) == 0) {
    ctrl->err_bit = bit;
    ctrl->err_val = val;
    ctrl->err_step = ctrl->step;
    ctrl->err_id0 = id0;
    ctrl->err_id1 = id1;
  }
}

// ---------------------------------------------------------------------------
// Counter-based normal deviates on the device (random.hpp:20-81): splitmix64
// finalizer chained over (seed, context, step, id, lane), two Box-Muller pairs
// over lanes 0..3, the fourth deviate discarded. The integer hash and the
// unit conversions are exact; log / cos / sin are CUDA's (<= 2 ulp), the
// reference's are glibc's, so a deviate can differ in its last bits.
constexpr unsigned long long kRngThermostat = 1;  // RngContext::kThermostat

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long counter_hash(unsigned long long seed,
                                                           unsigned long long ctx,
                                                           unsigned long long step,
                                                           unsigned long long id,
                                                           unsigned long long lane) {
  unsigned long long h = mix64(seed ^ 0x243f6a8885a308d3ull);
  h = mix64(h ^ ctx);
  h = mix64(h ^ step);
  h = mix64(h ^ id);
  return mix64(h ^ lane);
}

__device__ __forceinline__ void counter_normal3(unsigned long long seed, unsigned long long ctx,
                                                unsigned long long step, unsigned long long id,
                                                double& n0, double& n1, double& n2) {
  const double p53 = 1.1102230246251565e-16;  // 2^-53
  const double u0 = __dmul_rn(static_cast<double>((counter_hash(seed, ctx, step, id, 0) >> 11) + 1), p53);
  const double u1 = __dmul_rn(static_cast<double>(counter_hash(seed, ctx, step, id, 1) >> 11), p53);
  const double u2 = __dmul_rn(static_cast<double>((counter_hash(seed, ctx, step, id, 2) >> 11) + 1), p53);
  const double u3 = __dmul_rn(static_cast<double>(counter_hash(seed, ctx, step, id, 3) >> 11), p53);
  const double two_pi = 6.283185307179586476925286766559;
  const double r0 = __dsqrt_rn(__dmul_rn(-2.0, log(u0)));
  const double r1 = __dsqrt_rn(__dmul_rn(-2.0, log(u2)));
  const double a = __dmul_rn(two_pi, u1);
  n0 = __dmul_rn(r0, cos(a));
  n1 = __dmul_rn(r0, sin(a));
  n2 = __dmul_rn(r1, cos(__dmul_rn(two_pi, u3)));
}

// Langevin bath (potentials.hpp:174-197): f += -gamma m v + sqrt(2 m gamma T / dt) n,
// with n = counter_normal3(seed, kThermostat, step, id) — the force that
// thermostat_and_half_kick (engine.hpp:209-230) adds before the closing kick.
struct Thermo {
  int on;
  double gamma, temperature, dt;
  unsigned long long seed;
};

__device__ __forceinline__ void langevin_add(const Thermo& th, long long step, long long id,
                                             double m, double vx, double vy, double vz,
                                             double& fx, double& fy, double& fz) {
  double n0, n1, n2;
  counter_normal3(th.seed, kRngThermostat, static_cast<unsigned long long>(step),
                  static_cast<unsigned long long>(id), n0, n1, n2);
  const double amp = __dsqrt_rn(__ddiv_rn(
      __dmul_rn(__dmul_rn(__dmul_rn(2.0, m), th.gamma), th.temperature), th.dt));
  const double gm = __dmul_rn(-th.gamma, m);
  fx = __dadd_rn(fx, __dadd_rn(__dmul_rn(gm, vx), __dmul_rn(amp, n0)));
  fy = __dadd_rn(fy, __dadd_rn(__dmul_rn(gm, vy), __dmul_rn(amp, n1)));
  fz = __dadd_rn(fz, __dadd_rn(__dmul_rn(gm, vz), __dmul_rn(amp, n2)));
}

template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += smem[w];
  }
  return t;  // valid in thread 0
}

}  // namespace tmd
