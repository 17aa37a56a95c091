// sm_100a kernels of the LJ short-range path. One thread per particle for the
// streaming kernels; see DESIGN.md for the roofline each one is held to.
//
// Every rebuild-phase kernel reads the device-side decision ctrl->rebuild and
// returns immediately when it is 0, so a whole step (including the
// data-dependent resort + list build) is enqueued without a host round trip.
#pragma once

#include "tmd_device.cuh"

namespace tmd {

constexpr int kBlock = 128;

// ---------------------------------------------------------------------------
// Integrate: first half-kick + drift, fused with the displacement test.
// Engine::half_kick_and_drift (engine.hpp:174-189) and max_displacement2
// (neighbor_list.hpp:114-136). Arithmetic order mirrors the reference:
// v += (f * inv_m) * half_dt; x += v * dt.
__device__ __forceinline__ void kick(double& v, double f, double inv_m,
                                     double half_dt) {
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f, inv_m), half_dt));
}

// ---------------------------------------------------------------------------
// Velocity-Verlet epilogue fused into the force kernels. Modes:
//   kForcesOnly  f only (compute_forces, setup)
//   kKick2       f, then the closing half-kick of the step
//                (thermostat_and_half_kick without thermostat, engine.hpp:209-239)
//   kFused       f, closing half-kick of step n, then opening half-kick +
//                drift of step n+1 (half_kick_and_drift, engine.hpp:174-189)
//                into the OTHER position buffer (ping-pong: other CTAs are
//                still gathering the current positions), with the rebuild
//                displacement test of step n+1 (max_displacement2,
//                neighbor_list.hpp:114-136) reduced on the fly.
// Kinetic-energy partials are of the post-kick2 velocities (what observe()
// reports after the step). Arithmetic order mirrors the reference.
enum : int { kForcesOnly = 0, kKick2 = 1, kFused = 2 };

// FENE bonds resolved to slots (row f1): per owned slot up to kMaxBonds
// entries packed like list entries — partner slot (low 25 bits), the
// periodic image of the bond's second particle b as seen from its anchor a
// (bits 25-30, same codes), bit 31 set when this slot is the partner b.
struct BondTab {
  int on;
  const int* cnt;          // [n_cap] bonds per slot
  const uint32_t* ent;     // [n_cap * kMaxBonds]
  double k, rmax2;         // FeneParams k, r_max^2 (potentials.hpp:77-104)
};

struct Integ {
  double* vx;
  double* vy;
  double* vz;
  const double* mass;
  const long long* id;
  const double4* snap;
  double4* pos_out;
  double dt, half_dt;
  double* part_ke;
  Thermo th;  // Langevin bath (off: NVE)
  BondTab bt; // FENE bonds (off: LJ only)
  // Fused halo (native slab loop): exp[i] = index of slot i in the export of
  // my lowest (.x) / highest (.y) layer, or -1; rg[0] / rg[1] = those layers'
  // ghost copies in the lower / upper neighbour's next-step position buffer
  // (peer memory over NVLink, or this GPU's own ghost slots with one slab).
  const int2* exp;
  double4* rg[2];
  // Speculative graph blocks (single context): a launch after the block's
  // rebuild decision halted it still advances the position buffers (copies
  // pos -> pos_out), so the buffer parity after a block is fixed at capture.
  int halt_copy;
};

// FENE forces of slot i (compute_bonded_forces, bonded.hpp:167-199): the bond
// vector is always the anchor's, d = x_a - (x_b + s), so both ends round it
// identically and receive exactly opposite forces; each end books the
// energy -0.5 k r_max^2 log(1 - r^2/r_max^2) and the virial ff r^2 (halved
// with the pair sums at the reduction).
__device__ __forceinline__ void bond_accumulate(int i, const double4& pi,
                                                const double4* __restrict__ pos,
                                                const BondTab& bt, const Geom& g,
                                                const long long* __restrict__ id, Ctrl* ctrl,
                                                double& ax, double& ay, double& az, double& e,
                                                double& w) {
  const int nb = bt.cnt[i];
  for (int k = 0; k < nb; ++k) {
    const uint32_t ent = bt.ent[static_cast<size_t>(i) * kMaxBonds + k];
    const int j = static_cast<int>(ent & kIdxMask);
    const double4 pj = pos[j];
    const bool anchor = (ent & kFlagIUpper) == 0u;
    const double4& pa = anchor ? pi : pj;
    const double4& pb = anchor ? pj : pi;
    const double sx = image_shift((ent >> 25) & 3u, g.L[0]);
    const double sy = image_shift((ent >> 27) & 3u, g.L[1]);
    const double sz = image_shift((ent >> 29) & 3u, g.L[2]);
    const double dx = __dsub_rn(pa.x, __dadd_rn(pb.x, sx));
    const double dy = __dsub_rn(pa.y, __dadd_rn(pb.y, sy));
    const double dz = __dsub_rn(pa.z, __dadd_rn(pb.z, sz));
    const double r2 = exact_r2(dx, dy, dz);
    if (!(r2 < bt.rmax2)) {
      record_error(ctrl, kStatBondStretch, anchor ? id[i] : id[j], anchor ? id[j] : id[i], r2);
      continue;
    }
    const double gq = __dsub_rn(1.0, __ddiv_rn(r2, bt.rmax2));
    const double ff = __ddiv_rn(-bt.k, gq);
    // both ends book the (identically rounded) energy and virial: the full-
    // list partial sums are halved at the reduction
    e += __dmul_rn(__dmul_rn(__dmul_rn(-0.5, bt.k), bt.rmax2), log(gq));
    w += ff * r2;
    if (anchor) {
      ax += ff * dx;
      ay += ff * dy;
      az += ff * dz;
    } else {
      ax -= ff * dx;
      ay -= ff * dy;
      az -= ff * dz;
    }
  }
}

// Closing half-kick (+ Langevin force, which then stays in the stored force
// like the reference's st.fx += lf) and, for kFused, the next step's opening
// half-kick + drift. gx..gz come in as the pair force and leave as the force
// to store.
template <int kMode>
__device__ __forceinline__ void integrate_one(int i, const double4& pi, double& gx, double& gy,
                                              double& gz, const Integ& it, Ctrl* ctrl,
                                              double& ke, double& d2) {
  if (kMode == kForcesOnly) return;
  const double m = it.mass[i];
  const double inv_m = __ddiv_rn(1.0, m);
  double ux = it.vx[i], uy = it.vy[i], uz = it.vz[i];
  if (it.th.on) langevin_add(it.th, ctrl->step, it.id[i], m, ux, uy, uz, gx, gy, gz);
  kick(ux, gx, inv_m, it.half_dt);
  kick(uy, gy, inv_m, it.half_dt);
  kick(uz, gz, inv_m, it.half_dt);
  if (!finite3(ux, uy, uz) || !finite3(gx, gy, gz)) {
    record_error(ctrl, kStatNonFinite, it.id[i], -1);
  }
  ke += __dmul_rn(__dmul_rn(0.5, m),
                  __dadd_rn(__dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy)),
                            __dmul_rn(uz, uz)));
  if (kMode == kFused) {
    kick(ux, gx, inv_m, it.half_dt);
    kick(uy, gy, inv_m, it.half_dt);
    kick(uz, gz, inv_m, it.half_dt);
    double4 p;
    p.x = __dadd_rn(pi.x, __dmul_rn(ux, it.dt));
    p.y = __dadd_rn(pi.y, __dmul_rn(uy, it.dt));
    p.z = __dadd_rn(pi.z, __dmul_rn(uz, it.dt));
    p.w = 0.0;
    it.pos_out[i] = p;
    if (it.exp) {  // boundary particle: its new position straight into the neighbours' ghosts
      const int2 e = it.exp[i];
      if (e.x >= 0) it.rg[0][e.x] = p;
      if (e.y >= 0) it.rg[1][e.y] = p;
      if (e.x >= 0 || e.y >= 0) __threadfence_system();
    }
    const double4 s = it.snap[i];
    d2 = fmax(d2, exact_r2(__dsub_rn(p.x, s.x), __dsub_rn(p.y, s.y), __dsub_rn(p.z, s.z)));
  }
  it.vx[i] = ux;
  it.vy[i] = uy;
  it.vz[i] = uz;
}

// The block's energy, virial and (kicking modes) kinetic partial sums in one
// pass: per-warp xor trees, then the warps' sums in warp order by thread 0 —
// the same fixed order as three block_sum calls, with one barrier instead of
// six. d2: the step's largest displacement, one atomicMax per warp.
template <int kMode, int kThreads>
__device__ __forceinline__ void block_partials(double e, double w, double ke, double d2,
                                               double* red3, double* part_e, double* part_w,
                                               const Integ& it, Ctrl* ctrl) {
  constexpr int kW = kThreads / 32;
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_xor_sync(0xffffffffu, e, o);
    w += __shfl_xor_sync(0xffffffffu, w, o);
    if (kMode != kForcesOnly) ke += __shfl_xor_sync(0xffffffffu, ke, o);
    if (kMode == kFused) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red3[warp] = e;
    red3[kW + warp] = w;
    red3[2 * kW + warp] = ke;
    if (kMode == kFused && d2 > 0.0) {
      atomicMax(&ctrl->max_d2, static_cast<unsigned long long>(__double_as_longlong(d2)));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, tw = 0.0, tk = 0.0;
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      te += red3[q];
      tw += red3[kW + q];
      tk += red3[2 * kW + q];
    }
    part_e[blockIdx.x] = te;
    part_w[blockIdx.x] = tw;
    if (kMode != kForcesOnly) it.part_ke[blockIdx.x] = tk;
  }
}

// Opening half-kick + drift of the first step of a run (later steps get it
// from the fused force epilogue), with the displacement test.
__global__ void __launch_bounds__(kBlock)
    k_kick_drift(int n, double4* __restrict__ pos, double* __restrict__ vx,
                 double* __restrict__ vy, double* __restrict__ vz,
                 const double* __restrict__ fx, const double* __restrict__ fy,
                 const double* __restrict__ fz, const double* __restrict__ mass,
                 const double4* __restrict__ snap, double dt, double half_dt, Ctrl* ctrl) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  double d2 = 0.0;
  if (i < n) {
    const double inv_m = __ddiv_rn(1.0, mass[i]);
    double ux = vx[i], uy = vy[i], uz = vz[i];
    kick(ux, fx[i], inv_m, half_dt);
    kick(uy, fy[i], inv_m, half_dt);
    kick(uz, fz[i], inv_m, half_dt);
    double4 p = pos[i];
    p.x = __dadd_rn(p.x, __dmul_rn(ux, dt));
    p.y = __dadd_rn(p.y, __dmul_rn(uy, dt));
    p.z = __dadd_rn(p.z, __dmul_rn(uz, dt));
    pos[i] = p;
    vx[i] = ux;
    vy[i] = uy;
    vz[i] = uz;
    const double4 s = snap[i];
    d2 = exact_r2(__dsub_rn(p.x, s.x), __dsub_rn(p.y, s.y), __dsub_rn(p.z, s.z));
  }
  // block max of d2 (non-negative doubles order like their bit patterns)
  for (int o = 16; o > 0; o >>= 1) d2 = fmax(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  if ((threadIdx.x & 31) == 0 && d2 > 0.0) {
    atomicMax(&ctrl->max_d2, static_cast<unsigned long long>(__double_as_longlong(d2)));
  }
}

// ---------------------------------------------------------------------------
// Bond resolution at a rebuild (resolve_bonded, bonded.hpp:78-162): ids ->
// current slots through a dense id table, the partner's closest periodic image
// fixed until the next resort.

__global__ void __launch_bounds__(kBlock)
    k_fill_int(int n, int* __restrict__ a, int v, const Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void __launch_bounds__(kBlock)
    k_slot_of_id(int n_slots, const long long* __restrict__ id, long long id_min,
                 int* __restrict__ slot_of_id, const Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int s = blockIdx.x * kBlock + threadIdx.x;
  if (s < n_slots) slot_of_id[id[s] - id_min] = s;
}

__device__ __forceinline__ uint32_t closest_image_code(double xa, double xb, double L) {
  // the copy of b closest to a among x_b, x_b + L, x_b - L (bonded.hpp:46-73)
  const double t0 = fabs(__dsub_rn(xa, xb));
  const double t1 = fabs(__dsub_rn(xa, __dadd_rn(xb, L)));
  const double t2 = fabs(__dsub_rn(xa, __dadd_rn(xb, -L)));
  if (t1 < t0 && t1 <= t2) return 1u;
  if (t2 < t0 && t2 < t1) return 2u;
  return 0u;
}

__global__ void __launch_bounds__(kBlock)
    k_bond_resolve(int n, const double4* __restrict__ pos, const long long* __restrict__ id,
                   long long id_min, const int* __restrict__ bond_off,
                   const int* __restrict__ bond_nbr, const unsigned char* __restrict__ bond_anchor,
                   const int* __restrict__ slot_of_id, Geom g, int* __restrict__ cnt,
                   uint32_t* __restrict__ ent, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  const long long o = id[i] - id_min;
  const int b0 = bond_off[o], b1 = bond_off[o + 1];
  const double4 pi = pos[i];
  int c = 0;
  for (int b = b0; b < b1; ++b) {
    const int p = slot_of_id[bond_nbr[b]];
    if (p < 0) {
      record_error(ctrl, kStatBondReach, id[i], id_min + bond_nbr[b]);
      continue;
    }
    const double4 pp = pos[p];
    const bool anchor = bond_anchor[b] != 0;
    const double4& pa = anchor ? pi : pp;
    const double4& pb = anchor ? pp : pi;
    const uint32_t code = closest_image_code(pa.x, pb.x, g.L[0]) |
                          (closest_image_code(pa.y, pb.y, g.L[1]) << 2) |
                          (closest_image_code(pa.z, pb.z, g.L[2]) << 4);
    ent[static_cast<size_t>(i) * kMaxBonds + c] =
        static_cast<uint32_t>(p) | (code << 25) | (anchor ? 0u : kFlagIUpper);
    ++c;
  }
  cnt[i] = c;
}

// Langevin force of the initial evaluation (compute_forces_untimed,
// engine.hpp:244-278: noise keyed as step 0, velocities as given).
__global__ void __launch_bounds__(kBlock)
    k_thermo_init(int n, const double* __restrict__ vx, const double* __restrict__ vy,
                  const double* __restrict__ vz, const double* __restrict__ mass,
                  const long long* __restrict__ id, Thermo th, double* __restrict__ fx,
                  double* __restrict__ fy, double* __restrict__ fz) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  double gx = fx[i], gy = fy[i], gz = fz[i];
  langevin_add(th, 0, id[i], mass[i], vx[i], vy[i], vz[i], gx, gy, gz);
  fx[i] = gx;
  fy[i] = gy;
  fz[i] = gz;
}

// ---------------------------------------------------------------------------
// Brute-force check for `verify` (the role of oracle_forces_energy /
// oracle_pair_set, oracle.hpp:31-160, in the reference CLI): all pairs under
// the minimum-image convention (box.hpp:34-43), no cells, no lists — an
// independent path to compare the list-based engine against.
__device__ __forceinline__ double min_image1(double d, double L) {
  double r = remainder(d, L);
  if (r == 0.5 * L) r = -0.5 * L;
  return r;
}

__global__ void __launch_bounds__(kBlock)
    k_brute(int n, const double* __restrict__ pos, const long long* __restrict__ id,
            double Lx, double Ly, double Lz, LjConst lj, double rv2, double* __restrict__ force,
            double* __restrict__ part_e, unsigned long long* __restrict__ npairs,
            long long* __restrict__ pairs, unsigned long long cap, int* __restrict__ overlap) {
  __shared__ double red[kBlock / 32];
  const int a = blockIdx.x * kBlock + threadIdx.x;
  double e = 0.0;
  if (a < n) {
    const double xa = pos[3 * a], ya = pos[3 * a + 1], za = pos[3 * a + 2];
    double fx = 0.0, fy = 0.0, fz = 0.0;
    for (int b = 0; b < n; ++b) {
      if (b == a) continue;
      const double dx = min_image1(xa - pos[3 * b], Lx);
      const double dy = min_image1(ya - pos[3 * b + 1], Ly);
      const double dz = min_image1(za - pos[3 * b + 2], Lz);
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (a < b && r2 <= rv2) {
        const unsigned long long k = atomicAdd(npairs, 1ull);
        if (k < cap) {
          pairs[2 * k] = min(id[a], id[b]);
          pairs[2 * k + 1] = max(id[a], id[b]);
        }
      }
      if (r2 >= lj.rc2) continue;
      if (r2 == 0.0) {
        atomicOr(overlap, 1);
        continue;
      }
      const double s2 = lj.sigma2 / r2;
      const double s6 = s2 * s2 * s2;
      e += 0.5 * (lj.eps4 * (s6 * s6 - s6) - lj.shift);
      const double ff = lj.eps24 * (2.0 * s6 * s6 - s6) / r2;
      fx += ff * dx;
      fy += ff * dy;
      fz += ff * dz;
    }
    force[3 * a] = fx;
    force[3 * a + 1] = fy;
    force[3 * a + 2] = fz;
  }
  const double t = block_sum<kBlock>(e, red);
  if (threadIdx.x == 0) part_e[blockIdx.x] = t;
}

// Kinetic partials of the current velocities (observe() after setup).
__global__ void __launch_bounds__(kBlock)
    k_kinetic(int n, const double* __restrict__ vx, const double* __restrict__ vy,
              const double* __restrict__ vz, const double* __restrict__ mass,
              double* __restrict__ part_ke) {
  __shared__ double red[kBlock / 32];
  const int i = blockIdx.x * kBlock + threadIdx.x;
  double ke = 0.0;
  if (i < n) {
    const double ux = vx[i], uy = vy[i], uz = vz[i];
    ke = __dmul_rn(__dmul_rn(0.5, mass[i]),
                   __dadd_rn(__dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy)),
                             __dmul_rn(uz, uz)));
  }
  const double t = block_sum<kBlock>(ke, red);
  if (threadIdx.x == 0) part_ke[blockIdx.x] = t;
}

// Rebuild decision (Engine::step, engine.hpp:88-100): global OR of
// needs_rebuild == max |dx|^2 > 0.25 skin^2 (strict), plus a host override.
__global__ void k_decide(Ctrl* ctrl, double thr, int advance_step, int* log,
                         int log_idx, cudaGraphConditionalHandle cond, long long* ticks) {
  stamp(ctrl, ticks, kTickDecide, 0);
  const double m = __longlong_as_double(static_cast<long long>(ctrl->max_d2));
  // force_rebuild: 1 = host-forced (setup), 2 = forced after a rollback and
  // not counted (the reference would not have rebuilt here)
  const int force = ctrl->force_rebuild;
  const int r = (force != 0) || (m > thr);
  ctrl->rebuild = r;
  ctrl->seen_d2 = m;
  if (cond != 0) cudaGraphSetConditional(cond, r ? 1u : 0u);  // graph mode: gate the IF node
  if (log) log[log_idx] = r;
  ctrl->force_rebuild = 0;
  ctrl->max_d2 = 0ull;
  if (advance_step) ctrl->step += 1;
  if (advance_step && (force == 1 || m > thr)) ctrl->rebuilds += 1;
}

// The far-away sentinel slot after the last particle of both position
// buffers (the list's padding entries point at it).
__global__ void k_set_far(double4* a, double4* b, double4 far) {
  *a = far;
  *b = far;
}

// Rebuild decision of a speculative graph block (single context): a step
// that needs a rebuild (or a host-forced one) halts the block — its force
// launch and every later one only carry the positions forward — and the
// block's closing rebuild step (k_decide + resort + build + forces) takes it.
__global__ void k_decide_spec1(Ctrl* ctrl, double thr, long long* ticks) {
  if (ctrl->halt) return;
  stamp(ctrl, ticks, kTickDecide, 0);
  const double m = __longlong_as_double(static_cast<long long>(ctrl->max_d2));
  ctrl->seen_d2 = m;
  if (ctrl->force_rebuild != 0 || m > thr) {
    ctrl->halt = 1;
    return;
  }
  ctrl->rebuild = 0;
  ctrl->max_d2 = 0ull;
  ctrl->step += 1;
}

__global__ void k_clear_halt(Ctrl* ctrl) { ctrl->halt = 0; }

// A phase stamp on its own (block start: off 0; forces start: off -1, after
// the step's decision advanced the counter; the chunk end: slot `end`).
__global__ void k_tick(const Ctrl* ctrl, long long* ticks, int ph, int off, int end) {
  if (end >= 0) {
    ticks[end] = global_ns();
    return;
  }
  if (ctrl->halt) return;  // a halted speculative block's remaining steps
  stamp(ctrl, ticks, ph, off);
}

// ---------------------------------------------------------------------------
// Resort = counting sort by cell (distribute_records, domain.hpp:54-92).

// wrap_position + CellGrid::cell_of, histogram. Positions are wrapped in place
// (the reference wraps only here, domain.hpp:63).
__global__ void __launch_bounds__(kBlock)
    k_wrap_bin(int n, double4* __restrict__ pos, const long long* __restrict__ id,
               int* __restrict__ cell, int* __restrict__ slot,
               int* __restrict__ count, const int* __restrict__ cell_rank, Geom g,
               Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  double4 p = pos[i];
  if (!finite3(p.x, p.y, p.z)) {
    record_error(ctrl, kStatNonFinitePos, id[i], -1);
    p.x = p.y = p.z = 0.0;
  }
  p.x = wrap1(p.x, g.L[0]);
  p.y = wrap1(p.y, g.L[1]);
  p.z = wrap1(p.z, g.L[2]);
  pos[i] = p;
  const int cx = cell_coord(p.x, g.cell_len[0], g.dims[0]);
  const int cy = cell_coord(p.y, g.cell_len[1], g.dims[1]);
  const int cz = cell_coord(p.z, g.cell_len[2], g.dims[2]);
  const int c = cx + g.dims[0] * (cy + g.dims[1] * cz);
  cell[i] = c;
  if (g.zslab && (cz < g.z0 || cz >= g.z0 + g.zown)) {  // must have migrated first
    record_error(ctrl, kStatStray, id[i], cz);
    slot[i] = 0;
    return;
  }
  slot[i] = atomicAdd(&count[cell_rank[local_cell(g, c)]], 1);  // brick-major order
}

// Exclusive scan of the cell histogram (one block; runs once per rebuild).
// Zeroes the histogram for the next resort.
// Tiled 3-phase exclusive scan (tile = 1024 threads x 4 items): per-tile
// sums, one-block scan of the tile sums, tile-local scan + offset. Runs once
// per rebuild; zeroes the histogram for the next resort.
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    warp_tot[lane] = w;
  }
  __syncthreads();
  total = warp_tot[(blockDim.x >> 5) - 1];
  const int r = x - v + (warp > 0 ? warp_tot[warp - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan_tiles(int n, const int* __restrict__ count, int* __restrict__ tile_sum,
                 Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  __shared__ int warp_tot[32];
  const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) s += base + u < n ? count[base + u] : 0;
  int total;
  block_excl_scan(s, warp_tot, total);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan_sums(int ntiles, int* __restrict__ tile_sum, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  __shared__ int warp_tot[32];
  int carry = 0;
  for (int t0 = 0; t0 < ntiles; t0 += kScanThreads) {
    const int t = t0 + threadIdx.x;
    const int v = t < ntiles ? tile_sum[t] : 0;
    int total;
    const int r = block_excl_scan(v, warp_tot, total);
    if (t < ntiles) tile_sum[t] = carry + r;
    carry += total;
  }
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan_apply(int n, int* __restrict__ count, const int* __restrict__ tile_off,
                 int* __restrict__ start, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  __shared__ int warp_tot[32];
  const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    v[u] = base + u < n ? count[base + u] : 0;
    s += v[u];
  }
  int total;
  int run = tile_off[blockIdx.x] + block_excl_scan(s, warp_tot, total);
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    if (base + u < n) {
      start[base + u] = run;
      count[base + u] = 0;
    }
    run += v[u];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) start[n] = run;
}

__global__ void __launch_bounds__(kBlock)
    k_scatter(int n, const int* __restrict__ cell, const int* __restrict__ slot,
              const int* __restrict__ start, const int* __restrict__ cell_rank, Geom g,
              int* __restrict__ perm, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  perm[start[cell_rank[local_cell(g, cell[i])]] + slot[i]] = i;
}

// Canonical order inside each cell: ascending particle id. Makes the sorted
// layout (and so every FP summation order) a pure function of the particle
// set, independent of the previous order and of the atomic arrival order.
__global__ void __launch_bounds__(kBlock)
    k_sort_cells(int ncells, const int* __restrict__ start, int* __restrict__ perm,
                 const long long* __restrict__ id, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  // one warp per cell: cells of <= 32 particles are ranked in registers (rank =
  // number of smaller ids, ids are unique), larger ones fall back to lane 0
  const int c = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= ncells) return;
  const int b = start[c], e = start[c + 1];
  const int m = e - b;
  if (m <= 32) {
    const int p = lane < m ? perm[b + lane] : 0;
    const long long key = lane < m ? id[p] : 0;
    int rank = 0;
    for (int q = 0; q < m; ++q) {
      const long long kq = __shfl_sync(0xffffffffu, key, q);
      rank += (kq < key) ? 1 : 0;
    }
    __syncwarp();
    if (lane < m) perm[b + rank] = p;
    return;
  }
  if (lane != 0) return;
  for (int k = b + 1; k < e; ++k) {
    const int pk = perm[k];
    const long long key = id[pk];
    int m = k - 1;
    while (m >= b && id[perm[m]] > key) {
      perm[m + 1] = perm[m];
      --m;
    }
    perm[m + 1] = pk;
  }
}

// The same canonical order for sparse cells (a few particles each, e.g. the
// Kremer-Grest melt): a thread per slot counts the smaller ids of its cell and
// writes its particle to that rank of `out` (a warp per cell would leave most
// lanes idle and cost 0.2 ms at 4M beads).
__global__ void __launch_bounds__(kBlock)
    k_sort_cells_thread(int n, const int* __restrict__ start, const int* __restrict__ cell,
                        const int* __restrict__ cell_rank, Geom g,
                        const int* __restrict__ perm, const long long* __restrict__ id,
                        int* __restrict__ out, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int s = blockIdx.x * kBlock + threadIdx.x;
  if (s >= n) return;
  const int p = perm[s];
  const int r = cell_rank[local_cell(g, cell[p])];
  const int b = start[r], e = start[r + 1];
  const long long key = id[p];
  int rank = 0;
  for (int q = b; q < e; ++q) rank += id[perm[q]] < key ? 1 : 0;
  out[b + rank] = p;
}

// Gather every particle array through perm into the alternate buffers.
__global__ void __launch_bounds__(kBlock)
    k_permute(int n, const int* __restrict__ perm, const double4* __restrict__ pos,
              const double* __restrict__ vx, const double* __restrict__ vy,
              const double* __restrict__ vz, const double* __restrict__ mass,
              const long long* __restrict__ id, const int* __restrict__ cell,
              double4* __restrict__ pos2, double* __restrict__ vx2,
              double* __restrict__ vy2, double* __restrict__ vz2,
              double* __restrict__ mass2, long long* __restrict__ id2,
              int* __restrict__ cell2, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= n) return;
  const int s = perm[k];
  pos2[k] = pos[s];
  vx2[k] = vx[s];
  vy2[k] = vy[s];
  vz2[k] = vz[s];
  mass2[k] = mass[s];
  id2[k] = id[s];
  cell2[k] = cell[s];
}

__global__ void __launch_bounds__(kBlock)
    k_copy_back(int n, const double4* __restrict__ pos2,
                const double* __restrict__ vx2, const double* __restrict__ vy2,
                const double* __restrict__ vz2, const double* __restrict__ mass2,
                const long long* __restrict__ id2, const int* __restrict__ cell2,
                double4* __restrict__ pos, double* __restrict__ vx,
                double* __restrict__ vy, double* __restrict__ vz,
                double* __restrict__ mass, long long* __restrict__ id,
                int* __restrict__ cell, const Ctrl* ctrl) {
  // ctrl: gated on this step's rebuild decision (the resort); nullptr:
  // unconditional (the native slab rebuild's stayer copy). cell: nullptr
  // skips the cell column (recomputed by the resort that follows).
  if (ctrl && !ctrl->rebuild) return;
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= n) return;
  pos[k] = pos2[k];
  vx[k] = vx2[k];
  vy[k] = vy2[k];
  vz[k] = vz2[k];
  mass[k] = mass2[k];
  id[k] = id2[k];
  if (cell) cell[k] = cell2[k];
}

// ---------------------------------------------------------------------------
// Full Verlet list build (the full-list form of build_sorted_list,
// neighbor_list.hpp:51-111): for particle i, every j in the 27 surrounding
// cells (with periodic images) with exact r2 <= rv2, own image excluded
// (neighbor_list.hpp:91-93). Also snapshots positions for needs_rebuild.
__global__ void __launch_bounds__(kBlock)
    k_build_list(int n, const double4* __restrict__ pos, const int* __restrict__ cell,
                 const int* __restrict__ start, const int* __restrict__ cell_rank, Geom g,
                 uint32_t* __restrict__ nbr,
                 int* __restrict__ nnbr, int stride, int cap,
                 double4* __restrict__ snap, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  __shared__ double red[kBlock / 32];
  const int i = blockIdx.x * kBlock + threadIdx.x;
  int cnt = 0;
  if (i < n) {
    const double4 pi = pos[i];
    snap[i] = pi;
    const int c = cell[i];
    const int cx = c % g.dims[0];
    const int cy = (c / g.dims[0]) % g.dims[1];
    const int cz = c / (g.dims[0] * g.dims[1]);
    for (int oz = -1; oz <= 1; ++oz) {
      int tz = cz + oz;
      uint32_t code_z = 0;
      if (tz < 0) { tz += g.dims[2]; code_z = 2; }
      else if (tz >= g.dims[2]) { tz -= g.dims[2]; code_z = 1; }
      for (int oy = -1; oy <= 1; ++oy) {
        int ty = cy + oy;
        uint32_t code_y = 0;
        if (ty < 0) { ty += g.dims[1]; code_y = 2; }
        else if (ty >= g.dims[1]) { ty -= g.dims[1]; code_y = 1; }
        for (int ox = -1; ox <= 1; ++ox) {
          int tx = cx + ox;
          uint32_t code_x = 0;
          if (tx < 0) { tx += g.dims[0]; code_x = 2; }
          else if (tx >= g.dims[0]) { tx -= g.dims[0]; code_x = 1; }
          const int t = tx + g.dims[0] * (ty + g.dims[1] * tz);
          // half-stencil orientation: first nonzero component (x, y, z) > 0
          const int first = ox != 0 ? ox : (oy != 0 ? oy : oz);
          const uint32_t img = (code_x << 25) | (code_y << 27) | (code_z << 29);
          const uint32_t tag = img | ((img != 0u && first < 0) ? kFlagIUpper : 0u);
          const bool same = (t == c);
          const int rt = cell_rank[t];
          const int jb = start[rt], je = start[rt + 1];
          for (int j = jb; j < je; ++j) {
            if (same && j == i) continue;
            const double4 pj = pos[j];
            const uint32_t ent = static_cast<uint32_t>(j) | tag;
            double dx, dy, dz;
            pair_delta(pi, pj, ent, g, dx, dy, dz);
            if (exact_r2(dx, dy, dz) <= g.rv2) {
              if (cnt < cap) nbr[static_cast<size_t>(cnt) * stride + i] = ent;
              ++cnt;
            }
          }
        }
      }
    }
    nnbr[i] = cnt < cap ? cnt : cap;
    if (cnt > cap) atomicOr(&ctrl->status, kStatOverflow);
  }
  // block max count + total entries
  int m = cnt;
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(&ctrl->max_count, m);
  const double tot = block_sum<kBlock>(static_cast<double>(cnt), red);
  if (threadIdx.x == 0 && tot > 0.0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctrl->entries),
              static_cast<unsigned long long>(tot));
  }
}

// Resets the per-build statistics before a build (only when rebuilding).
__global__ void k_build_prologue(Ctrl* ctrl, long long* ticks) {
  if (!ctrl->rebuild) return;
  stamp(ctrl, ticks, kTickBuild, -1);
  ctrl->max_count = 0;
  ctrl->entries = 0;
}

// ---------------------------------------------------------------------------
// LJ forces + energy + virial over the full list, one thread per particle
// (compute_pair_forces, neighbor_list.hpp:150-187, in full-list form: every
// thread owns its own f_i, no Newton-3 scatter, no atomics). Cutoff test and
// r2 are rounded exactly like the reference; the force arithmetic uses one
// reciprocal. Per-block partials of sum_i e_i and sum_i w_i (each pair counted
// twice; the final reduction halves them).
template <int kMode>
__global__ void __launch_bounds__(kBlock)
    k_lj_forces(int n, const double4* __restrict__ pos,
                const uint32_t* __restrict__ nbr, const int* __restrict__ nnbr,
                int stride, Geom g, LjConst lj, double* __restrict__ fx,
                double* __restrict__ fy, double* __restrict__ fz,
                double* __restrict__ part_e, double* __restrict__ part_w,
                const long long* __restrict__ id, Integ it, Ctrl* ctrl) {
  __shared__ double red[3 * (kBlock / 32)];
  const int i = blockIdx.x * kBlock + threadIdx.x;
  double e = 0.0, w = 0.0, ke = 0.0, d2 = 0.0;
  if (i < n) {
    const double4 pi = pos[i];
    double ax = 0.0, ay = 0.0, az = 0.0;
    const int cnt = nnbr[i];
    const uint32_t* p = nbr + i;
    for (int k = 0; k < cnt; ++k) {
      const uint32_t ent = __ldg(p + static_cast<size_t>(k) * stride);
      const double4 pj = ldg_pos(pos + (ent & kIdxMask));
      double dx, dy, dz;
      pair_delta(pi, pj, ent, g, dx, dy, dz);
      const double r2 = exact_r2(dx, dy, dz);
      if (r2 < lj.rc2) {
        if (r2 == 0.0) {
          record_error(ctrl, kStatOverlap, id[i], id[ent & kIdxMask]);
          continue;
        }
        const double ri2 = rcp_nr(r2);
        const double inv = lj.sigma2 * ri2;
        const double i6 = inv * inv * inv;
        double ff = lj.eps24 * (2.0 * i6 * i6 - i6) * ri2;
        if (lj.fcap > 0.0) {  // overlap warm-up: |F| <= fcap (energy left uncapped)
          const double r = sqrt(r2);
          if (fabs(ff) * r > lj.fcap) ff = copysign(lj.fcap / r, ff);
        }
        e += lj.eps4 * (i6 * i6 - i6) - lj.shift;
        w += ff * r2;
        ax += ff * dx;
        ay += ff * dy;
        az += ff * dz;
      }
    }
    if (it.bt.on) bond_accumulate(i, pi, pos, it.bt, g, id, ctrl, ax, ay, az, e, w);
    integrate_one<kMode>(i, pi, ax, ay, az, it, ctrl, ke, d2);
    if (kMode != kFused) {  // a fused step's force only feeds its own kicks
      fx[i] = ax;
      fy[i] = ay;
      fz[i] = az;
    }
  }
  block_partials<kMode, kBlock>(e, w, ke, d2, red, part_e, part_w, it, ctrl);
}

// Sum of squared cell populations (the particle-weighted cell occupancy that
// picks the list build): integer sums, so the atomics are exact.
__global__ void __launch_bounds__(kBlock)
    k_occupancy(int ncells, const int* __restrict__ start, Ctrl* ctrl) {
  const int k = blockIdx.x * kBlock + threadIdx.x;
  unsigned long long m2 = 0;
  if (k < ncells) {
    const unsigned long long m = static_cast<unsigned long long>(start[k + 1] - start[k]);
    m2 = m * m;
  }
  for (int o = 16; o > 0; o >>= 1) m2 += __shfl_xor_sync(0xffffffffu, m2, o);
  if ((threadIdx.x & 31) == 0 && m2) atomicAdd(&ctrl->occ_s2, m2);
}

// Deterministic final reduction of per-block partials (fixed order tree).
constexpr int kRedThreads = 1024;
__global__ void __launch_bounds__(kRedThreads)
    k_reduce(const double* __restrict__ part, int nparts, double scale,
             double* __restrict__ out) {
  __shared__ double red[kRedThreads / 32];
  double s = 0.0;
  for (int k = threadIdx.x; k < nparts; k += kRedThreads) s += part[k];
  const double t = block_sum<kRedThreads>(s, red);
  if (threadIdx.x == 0) *out = t * scale;
}

// Engine construction's upload (build_domain, domain.hpp:134-189): the
// caller's (n, 3) positions and velocities as they are, unpacked to double4
// positions and SoA velocities; absent velocities are 0, absent masses 1.
__global__ void __launch_bounds__(kBlock)
    k_upload(int n, const double* __restrict__ p3, const double* __restrict__ v3,
             const double* __restrict__ m1, double4* __restrict__ pos, double* __restrict__ vx,
             double* __restrict__ vy, double* __restrict__ vz, double* __restrict__ mass) {
  const int r = blockIdx.x * kBlock + threadIdx.x;
  if (r >= n) return;
  pos[r] = make_double4(p3[3 * r], p3[3 * r + 1], p3[3 * r + 2], 0.0);
  vx[r] = v3 ? v3[3 * r] : 0.0;
  vy[r] = v3 ? v3[3 * r + 1] : 0.0;
  vz[r] = v3 ? v3[3 * r + 2] : 0.0;
  mass[r] = m1 ? m1[r] : 1.0;
}

// flatten_domain (domain.hpp:193-207) on the device for ids forming one
// dense range: slot s goes to row id[s] - lo, positions wrapped with the
// reference's wrap (wrap_position, the same rounding as the host's).
__global__ void __launch_bounds__(kBlock)
    k_download(int n, const double4* __restrict__ pos, const double* __restrict__ vx,
               const double* __restrict__ vy, const double* __restrict__ vz,
               const double* __restrict__ fx, const double* __restrict__ fy,
               const double* __restrict__ fz, const double* __restrict__ mass,
               const long long* __restrict__ id, long long lo, Geom g,
               double* __restrict__ opos, double* __restrict__ ovel, double* __restrict__ ofrc,
               double* __restrict__ omass, long long* __restrict__ oid) {
  const int s = blockIdx.x * kBlock + threadIdx.x;
  if (s >= n) return;
  const long long ident = id[s];
  const size_t r = static_cast<size_t>(ident - lo);
  oid[r] = ident;
  if (opos) {
    const double4 p = pos[s];
    opos[3 * r] = wrap1(p.x, g.L[0]);
    opos[3 * r + 1] = wrap1(p.y, g.L[1]);
    opos[3 * r + 2] = wrap1(p.z, g.L[2]);
  }
  if (ovel) {
    ovel[3 * r] = vx[s];
    ovel[3 * r + 1] = vy[s];
    ovel[3 * r + 2] = vz[s];
  }
  if (ofrc) {
    ofrc[3 * r] = fx[s];
    ofrc[3 * r + 1] = fy[s];
    ofrc[3 * r + 2] = fz[s];
  }
  if (omass) omass[r] = mass[s];
}

// The same, gathered in a given slot order (row r <- slot order[r]): the
// download of contexts whose ids are not one dense range (slab contexts,
// arbitrary ids), the order coming from a device sort of the ids.
__global__ void __launch_bounds__(kBlock)
    k_download_gather(int n, const int* __restrict__ order, const double4* __restrict__ pos,
                      const double* __restrict__ vx, const double* __restrict__ vy,
                      const double* __restrict__ vz, const double* __restrict__ fx,
                      const double* __restrict__ fy, const double* __restrict__ fz,
                      const double* __restrict__ mass, Geom g, double* __restrict__ opos,
                      double* __restrict__ ovel, double* __restrict__ ofrc,
                      double* __restrict__ omass) {
  const int r = blockIdx.x * kBlock + threadIdx.x;
  if (r >= n) return;
  const int s = order[r];
  if (opos) {
    const double4 p = pos[s];
    opos[3 * r] = wrap1(p.x, g.L[0]);
    opos[3 * r + 1] = wrap1(p.y, g.L[1]);
    opos[3 * r + 2] = wrap1(p.z, g.L[2]);
  }
  if (ovel) {
    ovel[3 * r] = vx[s];
    ovel[3 * r + 1] = vy[s];
    ovel[3 * r + 2] = vz[s];
  }
  if (ofrc) {
    ofrc[3 * r] = fx[s];
    ofrc[3 * r + 1] = fy[s];
    ofrc[3 * r + 2] = fz[s];
  }
  if (omass) omass[r] = mass[s];
}

// Slab create: particles whose wrapped position lies in this slab's z layers
// (wrap1 + cell_coord: the rounding of distribute_records, domain.hpp:56-65).
__global__ void __launch_bounds__(kBlock)
    k_slab_flags(int n, const double* __restrict__ pos, Geom g, unsigned char* __restrict__ flag) {
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= n) return;
  const double z = wrap1(pos[3 * k + 2], g.L[2]);
  const int cz = cell_coord(z, g.cell_len[2], g.dims[2]);
  flag[k] = (cz >= g.z0 && cz < g.z0 + g.zown) ? 1 : 0;
}

// Slab create: this rank's particles (input order) from the staged system
// into the slot arrays (double4 positions, SoA velocities).
__global__ void __launch_bounds__(kBlock)
    k_slab_unpack(int m, const int* __restrict__ sel, const double* __restrict__ pos,
                  const double* __restrict__ vel, const double* __restrict__ mass,
                  const long long* __restrict__ id, double4* __restrict__ opos,
                  double* __restrict__ vx, double* __restrict__ vy, double* __restrict__ vz,
                  double* __restrict__ omass, long long* __restrict__ oid) {
  const int r = blockIdx.x * kBlock + threadIdx.x;
  if (r >= m) return;
  const size_t k = static_cast<size_t>(sel[r]);
  opos[r] = make_double4(pos[3 * k], pos[3 * k + 1], pos[3 * k + 2], 0.0);
  vx[r] = vel ? vel[3 * k] : 0.0;
  vy[r] = vel ? vel[3 * k + 1] : 0.0;
  vz[r] = vel ? vel[3 * k + 2] : 0.0;
  omass[r] = mass ? mass[k] : 1.0;
  oid[r] = id[k];
}

// Velocities and masses of a system uploaded in id order (ids lo, lo + 1, ...
// in input order) placed into the slots the first resort chose.
__global__ void __launch_bounds__(kBlock)
    k_place_vm(int n, const long long* __restrict__ id, long long lo,
               const double* __restrict__ v3, const double* __restrict__ m1,
               double* __restrict__ vx, double* __restrict__ vy, double* __restrict__ vz,
               double* __restrict__ mass) {
  const int s = blockIdx.x * kBlock + threadIdx.x;
  if (s >= n) return;
  const long long r = id[s] - lo;
  if (v3) {
    vx[s] = v3[3 * r];
    vy[s] = v3[3 * r + 1];
    vz[s] = v3[3 * r + 2];
  }
  if (m1) mass[s] = m1[r];
}

__global__ void k_iota_i64(int n, long long lo, long long* __restrict__ v) {
  const int r = blockIdx.x * kBlock + threadIdx.x;
  if (r < n) v[r] = lo + r;
}

__global__ void k_iota_int(int n, int* __restrict__ v) {
  const int r = blockIdx.x * kBlock + threadIdx.x;
  if (r < n) v[r] = r;
}

// Per-step observable row (run_observed): PE and virial of this step's force
// evaluation (halved full-list sums), KE of the post-kick velocities, written
// straight into mapped pinned host memory — each recorded step's result
// crosses to the host as the step completes. Rows every `stride` steps.
__global__ void __launch_bounds__(kRedThreads)
    k_obs_record(const double* __restrict__ part_e, const double* __restrict__ part_w,
                 int npe, const double* __restrict__ part_ke, int nke, Ctrl* ctrl, int stride,
                 double* __restrict__ rows, int max_rows) {
  if (ctrl->halt) return;  // native slab loop: a halted (replayed) step records nothing
  __shared__ double red[kRedThreads / 32];
  double se = 0.0, sw = 0.0, sk = 0.0;
  for (int k = threadIdx.x; k < npe; k += kRedThreads) {
    se += part_e[k];
    sw += part_w[k];
  }
  for (int k = threadIdx.x; k < nke; k += kRedThreads) sk += part_ke[k];
  const double te = block_sum<kRedThreads>(se, red);
  const double tw = block_sum<kRedThreads>(sw, red);
  const double tk = block_sum<kRedThreads>(sk, red);
  if (threadIdx.x == 0) {
    const long long st = ctrl->step;
    if (st % stride == 0) {
      const int r = ctrl->obs_rows;
      if (r < max_rows) {
        double* o = rows + 4 * r;
        o[0] = static_cast<double>(st);
        o[1] = tk;
        o[2] = te * 0.5;
        o[3] = tw * 0.5;
      }
      ctrl->obs_rows = r + 1;
    }
  }
}

// In-cut pair count of the current list (roofline accounting only; not on
// the step path).
__global__ void __launch_bounds__(kBlock)
    k_count_incut(int n, const double4* __restrict__ pos,
                  const uint32_t* __restrict__ nbr, const int* __restrict__ nnbr,
                  int stride, Geom g, double rc2,
                  unsigned long long* __restrict__ out) {
  __shared__ double red[kBlock / 32];
  const int i = blockIdx.x * kBlock + threadIdx.x;
  double cnt = 0.0;
  if (i < n) {
    const double4 pi = pos[i];
    const int m = nnbr[i];
    for (int k = 0; k < m; ++k) {
      const uint32_t ent = nbr[static_cast<size_t>(k) * stride + i];
      const double4 pj = pos[ent & kIdxMask];
      double dx, dy, dz;
      pair_delta(pi, pj, ent, g, dx, dy, dz);
      if (exact_r2(dx, dy, dz) < rc2) cnt += 1.0;
    }
  }
  const double t = block_sum<kBlock>(cnt, red);
  if (threadIdx.x == 0 && t > 0.0) {
    atomicAdd(out, static_cast<unsigned long long>(t));
  }
}

// FP64 pipe peak probe (DFMA throughput): the roofline denominator for FLOPs
// (MEASURED_PEAKS.json has no FP64 entry).
constexpr int kDfmaChains = 8;
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters) {
  double a[kDfmaChains];
#pragma unroll
  for (int k = 0; k < kDfmaChains; ++k) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kDfmaChains; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kDfmaChains; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace tmd
