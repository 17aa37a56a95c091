// Brick-staged kernels: particles are stored brick-major (bricks of 2x2x2 or
// 2x2x4 cells, x-fastest; cells x-fastest inside a brick; particles by id
// inside a cell), so a brick's own particles are one contiguous range and its
// 27-cell neighbourhood is the (Bx+2)(By+2)(Bz+2) halo block. The list builds
// stage that halo block in shared memory once per brick (load_halo defines the
// staging layout: halo cells x-fastest, each padded to a multiple of 4 slots).
//
// List layout (sector-chunked ELL): groups of 32 consecutive particles. Entry
// k of lane l of group g lives at
//   list[g*cap*32 + (k/8)*256 + l*8 + k%8]
// so each lane owns whole 32-byte sectors: the build flushes 8 entries with
// two 16-B stores, the force kernel reads 8 entries with two 16-B loads, and
// a warp touches 1 KB of contiguous memory per chunk. A lane's last chunk is
// padded with the sentinel (coordinates far away), like the reference's
// sentinel-padded runs (neighbor_list.hpp:14-18, soa_store.hpp:47-79), so the
// force loop has no tail branch. Entries are global slots (variant 3, sentinel
// slot N) or the brick's staging indices (variant 2, sentinel = staging slot
// stage_cap), the latter gathered from shared memory by k_forces_staged.
#pragma once

#include "tmd_device.cuh"
#include "tmd_kernels.cuh"

namespace tmd {

// Bricks of 2 x 2 x kBrickZ cells: the list build stages a brick's
// (2+2) x (2+2) x (kBrickZ+2) halo once for its 2 x 2 x kBrickZ own cells.
constexpr int kBrickZ = 4;
constexpr int kMaxHalo = 4 * 4 * (kBrickZ + 2);  // 96
constexpr float kFarF = 1.0e30f;
constexpr double kFarD = 1.0e30;

struct BrickGeom {
  int B[3];      // brick edge in cells (min(2, dims))
  int nb[3];     // bricks per axis
  int nbricks;
  int cap;       // list entries per particle (multiple of 8)
  int stage_cap;  // staging capacity (slots, multiple of 4); sentinel slot = stage_cap
  float lo2, hi2;     // FP32 prefilter band around rv2 (exact FP64 inside)
  double origin_scale[3];  // cell_len (brick origin = lo * cell_len)
};

struct HaloTable {
  int n;                  // halo cells
  int H[3];               // halo extent
  int lo[3];              // first owned cell of the brick
  int e[3];               // owned extent
  int total;              // staged slots (padded)
  int bs, be;             // brick particle range
};

__device__ __forceinline__ int pad4(int v) { return (v + 3) & ~3; }

// Fills the halo metadata of brick b into shared memory (block size >= 64
// threads; synchronises). Halo cell h = hx + H0*(hy + H1*hz) mirrors global
// cell raw = lo + h - 1 with periodic wrap; its image code (bits 25..30) is
// the reference's ghost shift for that wrap (subnode.hpp:84-90).
__device__ __forceinline__ void load_halo(int b, const Geom& g, const BrickGeom& bg,
                                          const int* __restrict__ cell_rank,
                                          const int* __restrict__ brick_rank_off,
                                          const int* __restrict__ start, HaloTable& ht,
                                          int* s_gstart, int* s_cnt, int* s_off,
                                          uint32_t* s_code, int* s_gcell) {
  const int bx = b % bg.nb[0];
  const int by = (b / bg.nb[0]) % bg.nb[1];
  const int bz = b / (bg.nb[0] * bg.nb[1]);
  // slab mode: bricks tile the owned layers, which start at local layer 1
  const int zoff = g.zslab ? 1 : 0;
  const int zext = g.zslab ? g.zown : g.dims[2];
  ht.lo[0] = bx * bg.B[0];
  ht.lo[1] = by * bg.B[1];
  ht.lo[2] = zoff + bz * bg.B[2];
  ht.e[0] = min(bg.B[0], g.dims[0] - ht.lo[0]);
  ht.e[1] = min(bg.B[1], g.dims[1] - ht.lo[1]);
  ht.e[2] = min(bg.B[2], zext - (ht.lo[2] - zoff));
#pragma unroll
  for (int k = 0; k < 3; ++k) ht.H[k] = ht.e[k] + 2;
  ht.n = ht.H[0] * ht.H[1] * ht.H[2];
  const int t = threadIdx.x;
  if (t < ht.n) {
    const int h[3] = {t % ht.H[0], (t / ht.H[0]) % ht.H[1], t / (ht.H[0] * ht.H[1])};
    int gc[3];
    uint32_t code = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int raw = ht.lo[k] + h[k] - 1;
      uint32_t c2 = 0;
      if (k == 2 && g.zslab) {  // local z: ghost layers carry the wrap shift
        c2 = raw == 0 ? g.zcode_lo : (raw == g.ldz - 1 ? g.zcode_hi : 0u);
      } else if (raw < 0) {
        raw += g.dims[k];
        c2 = 2;
      } else if (raw >= g.dims[k]) {
        raw -= g.dims[k];
        c2 = 1;
      }
      gc[k] = raw;
      code |= c2 << (25 + 2 * k);
    }
    const int cl = gc[0] + g.dims[0] * (gc[1] + g.dims[1] * gc[2]);
    const int r = cell_rank[cl];
    s_gcell[t] = cl;
    s_gstart[t] = start[r];
    s_cnt[t] = start[r + 1] - start[r];
    s_code[t] = code;
  }
  __syncthreads();
  if (t < 32) {  // warp-level exclusive scan of the padded counts (<= 96 cells)
    int v[kMaxHalo / 32], sv[kMaxHalo / 32];
#pragma unroll
    for (int q = 0; q < kMaxHalo / 32; ++q) {
      v[q] = t + 32 * q < ht.n ? pad4(s_cnt[t + 32 * q]) : 0;
      sv[q] = v[q];
    }
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int q = 0; q < kMaxHalo / 32; ++q) {
        const int u = __shfl_up_sync(0xffffffffu, sv[q], o);
        if (t >= o) sv[q] += u;
      }
    }
    int base = 0;
#pragma unroll
    for (int q = 0; q < kMaxHalo / 32; ++q) {
      if (t + 32 * q < ht.n) s_off[t + 32 * q] = base + sv[q] - v[q];
      base += __shfl_sync(0xffffffffu, sv[q], 31);
    }
    if (t == 31) s_off[ht.n] = base;
  }
  __syncthreads();
  ht.total = s_off[ht.n];
  ht.bs = start[brick_rank_off[b]];
  ht.be = start[brick_rank_off[b + 1]];
}

// Halo cell of staged index k (s_off is non-decreasing, s_off[n] = total).
__device__ __forceinline__ int halo_of(int k, const int* s_off, int n) {
  int lo = 0, hi = n;  // find last h with s_off[h] <= k
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_off[mid] <= k) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ double code_shift(uint32_t code, int axis, double L) {
  return image_shift((code >> (25 + 2 * axis)) & 3u, L);
}

// Global z coordinate of a brick's origin layer (local layer lz; slab mode:
// global layer z0 + lz - 1), so that the FP32 brick-relative coordinates stay
// within a few cells of 0 on every slab (the prefilter band assumes it).
__device__ __forceinline__ double origin_z(const Geom& g, int lz, double cell_len) {
  return (g.zslab ? g.z0 + lz - 1 : lz) * cell_len;
}

// Brick-major cell ranks (setup_bricks' order: bricks x-fastest, cells
// x-fastest inside a brick; slab mode: the two ghost layers ranked after every
// owned cell, x-fastest) and each brick's first rank, in closed form: the
// cells of the bricks before brick (bx, by, bz) are the full brick layers
// below it, the full brick rows before it in its layer and the bricks before
// it in its row.
__global__ void __launch_bounds__(kBlock)
    k_brick_tables(Geom g, BrickGeom bg, int* __restrict__ cell_rank,
                   int* __restrict__ brick_rank_off) {
  const int t = blockIdx.x * kBlock + threadIdx.x;
  const int d0 = g.dims[0], d1 = g.dims[1];
  const int zoff = g.zslab ? 1 : 0;
  const int ext2 = g.zslab ? g.zown : g.dims[2];
  const int owned = d0 * d1 * ext2;
  auto before = [&](int bx, int by, int bz) {
    const int ey = min(bg.B[1], d1 - by * bg.B[1]);
    const int ez = min(bg.B[2], ext2 - bz * bg.B[2]);
    return min(bz * bg.B[2], ext2) * d0 * d1 + min(by * bg.B[1], d1) * d0 * ez +
           min(bx * bg.B[0], d0) * ey * ez;
  };
  if (t <= bg.nbricks) {
    if (t == bg.nbricks) {
      brick_rank_off[t] = owned;
    } else {
      const int bx = t % bg.nb[0], by = (t / bg.nb[0]) % bg.nb[1], bz = t / (bg.nb[0] * bg.nb[1]);
      brick_rank_off[t] = before(bx, by, bz);
    }
  }
  if (t < g.ncells) {
    const int x = t % d0, y = (t / d0) % d1, zl = t / (d0 * d1);
    int r;
    if (g.zslab && (zl == 0 || zl == g.ldz - 1)) {
      r = owned + (zl == 0 ? 0 : d0 * d1) + x + d0 * y;
    } else {
      const int z = zl - zoff;
      const int bx = x / bg.B[0], by = y / bg.B[1], bz = z / bg.B[2];
      const int ex = min(bg.B[0], d0 - bx * bg.B[0]);
      const int ey = min(bg.B[1], d1 - by * bg.B[1]);
      r = before(bx, by, bz) + (x - bx * bg.B[0]) + ex * ((y - by * bg.B[1]) + ey * (z - bz * bg.B[2]));
    }
    cell_rank[t] = r;
  }
}

__device__ __forceinline__ size_t list_slot(int group, int cap, int lane, int k) {
  return static_cast<size_t>(group) * cap * 32 + static_cast<size_t>(k >> 3) * 256 +
         lane * 8 + (k & 7);
}

// ---------------------------------------------------------------------------
// Brick-staged list builds (the full-list form of build_sorted_list,
// neighbor_list.hpp:51-111): a CTA per brick stages the brick's halo block in
// shared memory as negated brick-relative FP32 coordinates; candidates are
// tested with packed FP32 arithmetic (FADD2/FFMA2) and only those inside the
// band |r2 - rv2| <= delta take the exact FP64 test with the reference's
// rounding, so membership is bit-identical to the reference.
constexpr int kBuildThreads = 256;
#ifndef TMD_BUILD_MIN_BLOCKS
#define TMD_BUILD_MIN_BLOCKS 4
#endif
constexpr int kBuildMinBlocks = TMD_BUILD_MIN_BLOCKS;

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// ---------------------------------------------------------------------------
// Full-list build, lanes = particles, branch-free appends (k_build_brick3).
// A warp owns one cell of the brick, lanes = its particles. Candidates stream
// warp-uniformly over the 27 halo cells, two at a time (LDS.64 broadcast +
// packed FP32 FADD2/FFMA2); every lane appends its hits to a private 16-slot
// shared-memory ring with predicated stores and flushes a completed 8-entry
// chunk as one 32-B sector. Only the FP32 rounding band and r2 == 0 (self,
// or coincident particles, which the force kernel reports) take the exact
// FP64 path, so membership is bit-identical to the reference.
// 8 ring slots (stride 32 words) -> one 32-B sector of the chunked list.
__device__ __forceinline__ void flush_chunk(const uint32_t* ring8, uint32_t* dst) {
  uint4 a, b;
  a.x = ring8[0];
  a.y = ring8[32];
  a.z = ring8[64];
  a.w = ring8[96];
  b.x = ring8[128];
  b.y = ring8[160];
  b.z = ring8[192];
  b.w = ring8[224];
  reinterpret_cast<uint4*>(dst)[0] = a;
  reinterpret_cast<uint4*>(dst)[1] = b;
}

// Ring append at slot n & 15 of the lane's ring (stride 128 B): one LOP3 and
// one IMAD on a 32-bit shared-window address.
__device__ __forceinline__ void ring_put(uint32_t base, int n, uint32_t v) {
  const uint32_t a = (static_cast<uint32_t>(n) & 15u) * 128u + base;
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

template <bool kGlobal>
__global__ void __launch_bounds__(kBuildThreads, kBuildMinBlocks)
    k_build_brick3(const double4* __restrict__ pos, const int* __restrict__ cell_rank,
                   const int* __restrict__ brick_rank_off, const int* __restrict__ start,
                   Geom g, BrickGeom bg, uint32_t* __restrict__ list, int* __restrict__ nnbr,
                   double4* __restrict__ snap, uint32_t global_sentinel, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  extern __shared__ __align__(16) float s_f[];  // -x | -y | -z | base, each stage_cap + 32
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  // per-lane 16-slot ring, lane-fastest so concurrent stores never conflict
  __shared__ __align__(16) uint32_t s_ring[kBuildThreads / 32][16][32];
  __shared__ int s_maxc;
  __shared__ unsigned long long s_ent;
  const int b = blockIdx.x;
  HaloTable ht;
  if (threadIdx.x == 0) { s_maxc = 0; s_ent = 0ull; }
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  if (ht.total > bg.stage_cap) {
    if (threadIdx.x == 0) {
      atomicOr(&ctrl->status, kStatStageOverflow);
      atomicMax(&ctrl->max_halo, ht.total);
    }
    return;
  }
  const int sc = bg.stage_cap + 32;
  float* nx = s_f;
  float* ny = s_f + sc;
  float* nz = s_f + 2 * sc;
  int* sbase = reinterpret_cast<int*>(s_f + 3 * sc);  // entry index field per slot
  const double ox = ht.lo[0] * bg.origin_scale[0];
  const double oy = ht.lo[1] * bg.origin_scale[1];
  const double oz = origin_z(g, ht.lo[2], bg.origin_scale[2]);
  for (int k = threadIdx.x; k < ht.total + 32; k += kBuildThreads) {
    float x = kFarF, y = kFarF, z = kFarF;
    int base = 0;
    if (k < ht.total) {
      const int h = halo_of(k, s_off, ht.n);
      const int q = k - s_off[h];
      if (q < s_cnt[h]) {
        const double4 p = pos[s_gstart[h] + q];
        const uint32_t c = s_code[h];
        x = static_cast<float>((p.x + code_shift(c, 0, g.L[0])) - ox);
        y = static_cast<float>((p.y + code_shift(c, 1, g.L[1])) - oy);
        z = static_cast<float>((p.z + code_shift(c, 2, g.L[2])) - oz);
        base = kGlobal ? s_gstart[h] + q : k;
      }
    }
    nx[k] = -x;
    ny[k] = -y;
    nz[k] = -z;
    sbase[k] = base;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncell_own = ht.e[0] * ht.e[1] * ht.e[2];
  const uint32_t sentinel = kGlobal ? global_sentinel : static_cast<uint32_t>(bg.stage_cap);
  int my_max = 0;
  unsigned long long my_ent = 0;
  for (int oc = warp; oc < ncell_own; oc += kBuildThreads / 32) {
    const int ax = oc % ht.e[0], ay = (oc / ht.e[0]) % ht.e[1], az = oc / (ht.e[0] * ht.e[1]);
    const int hc = (ax + 1) + ht.H[0] * ((ay + 1) + ht.H[1] * (az + 1));
    const int ncl = s_cnt[hc];
    for (int p0 = 0; p0 < ncl; p0 += 32) {
      const int q = p0 + lane;
      const bool active = q < ncl;
      const int qi = active ? q : 0;
      const int i = s_gstart[hc] + qi;
      const int ki = s_off[hc] + qi;
      const float xf = -nx[ki], yf = -ny[ki], zf = -nz[ki];
      const float2 xi2 = f2(xf, xf), yi2 = f2(yf, yf), zi2 = f2(zf, zf);
      const unsigned long long row = list_slot(i >> 5, bg.cap, i & 31, 0);
      const float hi2 = active ? bg.hi2 : -1.0f;  // inactive lanes never hit
      const uint32_t lo2m1 = __float_as_uint(bg.lo2) - 1u;
      const uint32_t rbase =
          static_cast<uint32_t>(__cvta_generic_to_shared(&s_ring[warp][0][lane]));
      int n = 0;
      for (int oz2 = -1; oz2 <= 1; ++oz2) {
        for (int oy2 = -1; oy2 <= 1; ++oy2) {
          for (int ox2 = -1; ox2 <= 1; ++ox2) {
            const int h = hc + ox2 + ht.H[0] * (oy2 + ht.H[1] * oz2);
            const uint32_t code = s_code[h];
            const int first = ox2 != 0 ? ox2 : (oy2 != 0 ? oy2 : oz2);
            const uint32_t tag = code | ((code != 0u && first < 0) ? kFlagIUpper : 0u);
            const int kb = s_off[h], ke = kb + s_cnt[h];
            // four candidates per iteration: cell blocks are padded to a
            // multiple of 4 slots with far-away coordinates (never hits)
#pragma unroll 1
            for (int k = kb; k < ke; k += 4) {
              const float4 X = *reinterpret_cast<const float4*>(nx + k);
              const float4 Y = *reinterpret_cast<const float4*>(ny + k);
              const float4 Z = *reinterpret_cast<const float4*>(nz + k);
              const float2 dxa = __fadd2_rn(xi2, f2(X.x, X.y)), dxb = __fadd2_rn(xi2, f2(X.z, X.w));
              const float2 dya = __fadd2_rn(yi2, f2(Y.x, Y.y)), dyb = __fadd2_rn(yi2, f2(Y.z, Y.w));
              const float2 dza = __fadd2_rn(zi2, f2(Z.x, Z.y)), dzb = __fadd2_rn(zi2, f2(Z.z, Z.w));
              const float2 ra = __ffma2_rn(dza, dza, __ffma2_rn(dya, dya, __fmul2_rn(dxa, dxa)));
              const float2 rb = __ffma2_rn(dzb, dzb, __ffma2_rn(dyb, dyb, __fmul2_rn(dxb, dxb)));
              const float r2v[4] = {ra.x, ra.y, rb.x, rb.y};
              bool hit[4];
              bool band[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                hit[u] = r2v[u] <= hi2;
                // sure hit <=> 0 < r2 < lo2 (unsigned compare on the bits)
                band[u] = hit[u] && (__float_as_uint(r2v[u]) - 1u) >= lo2m1;
              }
              if (band[0] || band[1] || band[2] || band[3]) {  // exact FP64 (+ self)
                const double4 pi = pos[i];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (band[u]) {
                    const int j = s_gstart[h] + (k + u - kb);
                    double ex, ey, ez;
                    pair_delta(pi, pos[j], static_cast<uint32_t>(j & kIdxMask) | tag, g, ex,
                               ey, ez);
                    hit[u] = j != i && exact_r2(ex, ey, ez) <= g.rv2;
                  }
                }
              }
              // unconditional ring stores: a miss leaves junk in the next free
              // slot, which the next hit (or the sentinel padding) overwrites
              const int n0 = n;
              const uint4 sb = *reinterpret_cast<const uint4*>(sbase + k);
              ring_put(rbase, n, sb.x | tag);
              n += hit[0] ? 1 : 0;
              ring_put(rbase, n, sb.y | tag);
              n += hit[1] ? 1 : 0;
              ring_put(rbase, n, sb.z | tag);
              n += hit[2] ? 1 : 0;
              ring_put(rbase, n, sb.w | tag);
              n += hit[3] ? 1 : 0;
              if ((n0 >> 3) != (n >> 3) && n0 < bg.cap) {  // a chunk completed: flush it
                const int c = n0 >> 3;
                flush_chunk(&s_ring[warp][(c & 1) * 8][lane], list + row + c * 256);
              }
            }
          }
        }
      }
      if (active) {
        if ((n & 7) != 0 && n < bg.cap) {  // sentinel-pad and flush the last chunk
          for (int r = n; r < ((n + 7) & ~7); ++r) s_ring[warp][r & 15][lane] = sentinel;
          const int c = n >> 3;
          flush_chunk(&s_ring[warp][(c & 1) * 8][lane], list + row + c * 256);
        }
        nnbr[i] = n < bg.cap ? n : bg.cap;
        snap[i] = pos[i];
        if (n > bg.cap) atomicOr(&ctrl->status, kStatOverflow);
        my_max = max(my_max, n);
        my_ent += static_cast<unsigned long long>(n);
      }
      __syncwarp();
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
    my_ent += __shfl_xor_sync(0xffffffffu, my_ent, o);
  }
  if (lane == 0) {
    atomicMax(&s_maxc, my_max);
    atomicAdd(&s_ent, my_ent);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&ctrl->max_count, s_maxc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctrl->entries), s_ent);
  }
}

// ---------------------------------------------------------------------------
// Full-list build over a culled candidate stream (k_build_cull, build kind 6,
// the default for dense cells). Same warp/lane roles, staging, FP32 band and
// entry order as k_build_brick3; what changes is how much work a candidate
// costs (about half the warp instructions of k_build_brick3 per particle):
//  1. Culling: the warp first drops, 32 candidates at a time, every candidate
//     farther than r_v from the bounding box of its lanes' particles, and
//     appends the survivors in stencil order to a per-warp stream of
//     4-candidate chunks {x4, y4, z4, entry4}. Corner and edge cells of the
//     27-cell stencil lose about half and a quarter of their particles and
//     the per-cell padding disappears: ~40 % fewer candidate iterations at
//     the BASELINE density. A culled candidate is a sure miss of the FP32 test
//     for every lane (box distance <= each lane's distance; 1e-3 relative
//     margin for FP32 rounding), so membership is unchanged.
//  2. Entries and their tags are formed once per candidate at compaction.
//  3. Appends advance a running shared-memory address (one predicated add per
//     candidate). Flushes are warp-synchronous: when any lane has two whole
//     chunks in its 20-slot ring, every lane writes its whole chunks (32-B
//     sectors) and moves its partial chunk to the front, so the warp pays
//     for a flush every ~15 iterations instead of whenever one lane fills a
//     chunk.
//  4. The band test is one packed subtract per candidate pair and a 4-way
//     unsigned min.
// The own cell (self exclusion) is a stream segment of its own.
constexpr int kCullCap = 96;    // stream candidates per warp (multiple of 32)
#ifndef TMD_RING_SLOTS
#define TMD_RING_SLOTS 28
#endif
#ifndef TMD_RING_TRIGGER
#define TMD_RING_TRIGGER 16
#endif
#ifndef TMD_FLUSH_EVERY
#define TMD_FLUSH_EVERY 3
#endif
// per-lane ring: flushed when any lane holds kRingTrigger entries, checked
// every kFlushEvery chunks of 4 (so up to kRingTrigger - 1 + 4 kFlushEvery
// entries in flight)
constexpr int kRingSlots = TMD_RING_SLOTS;
constexpr int kRingTrigger = TMD_RING_TRIGGER;
constexpr int kFlushEvery = TMD_FLUSH_EVERY;
static_assert(kRingTrigger - 1 + 4 * kFlushEvery <= kRingSlots, "ring too small");

struct CullLane {
  float2 xi2, yi2, zi2;
  float hi2;       // -1 for inactive lanes: never a hit
  float2 nlo2;     // -lo2, or -inf for inactive lanes: never in the band
  uint32_t wb;     // bit pattern of the band width bound (r2 - lo2 <= width)
  uint32_t a;      // shared address of the next ring slot
  uint32_t rbase;  // shared address of ring slot 0
  int i;           // global slot
  uint32_t self;   // the lane's own entry index (global slot, or its staging index)
  int nflush;      // chunks flushed (or counted past the capacity)
  uint32_t* dst;   // list address of chunk nflush
};

// Writes the lane's whole chunks, moves its partial chunk to ring slot 0.
__device__ __forceinline__ void cull_flush(CullLane& L, int cap8, uint32_t* ring_lane) {
  const int fill = static_cast<int>((L.a - L.rbase) >> 7);
  const int whole = fill >> 3;
  for (int c = 0; c < whole; ++c) {
    if (L.nflush < cap8) flush_chunk(ring_lane + c * 8 * 32, L.dst);
    ++L.nflush;
    L.dst += 256;
  }
  if (whole > 0) {
    const int part = fill & 7;
    const uint32_t* src = ring_lane + whole * 8 * 32;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
      if (r < part) ring_lane[r * 32] = src[r * 32];
    }
    L.a = L.rbase + static_cast<uint32_t>(part) * 128u;
  }
}

// The exact FP64 membership test of a band candidate (global slot j).
__device__ __forceinline__ bool cull_exact(const double4& pi, int i, int j, uint32_t e,
                                           const double4* __restrict__ pos, const Geom& g) {
  double ex, ey, ez;
  pair_delta(pi, pos[j], e, g, ex, ey, ez);
  return j != i && exact_r2(ex, ey, ez) <= g.rv2;
}

// Global slot of a candidate entry: the entry itself, or (kLocal: brick-local
// staging index) the halo cell's first global slot + the offset in the cell.
struct StageMap {
  const int* off;     // s_off: staging offset per halo cell (n + 1)
  const int* gstart;  // s_gstart: first global slot per halo cell
  int n;
};

template <bool kLocal>
__device__ __forceinline__ int entry_slot(uint32_t e, const StageMap& sm) {
  const int k = static_cast<int>(e & kIdxMask);
  if (!kLocal) return k;
  const int h = halo_of(k, sm.off, sm.n);
  return sm.gstart[h] + (k - sm.off[h]);
}

// Four ring appends: unconditional stores, advances predicated on the FP32
// hit test (r2 <= hi2, and entry != self for the own cell). A miss leaves
// junk in the next free slot, which the next store or the sentinel padding
// replaces.
template <bool kSelf>
__device__ __forceinline__ void cull_append4_fp32(uint32_t& a, const uint4& E, const float2& r0,
                                                  const float2& r1, float hi2, uint32_t me) {
#define TMD_APPEND(R, E)                                                     \
  if (kSelf) {                                                               \
    asm volatile(                                                            \
        "{\n\t.reg .pred p, q;\n\t"                                          \
        "setp.ne.u32 q, %2, %3;\n\t"                                         \
        "setp.le.and.f32 p, %1, %4, q;\n\t"                                  \
        "st.shared.u32 [%0], %2;\n\t"                                        \
        "@p add.u32 %0, %0, 128;\n\t}"                                       \
        : "+r"(a)                                                            \
        : "f"(R), "r"(E), "r"(me), "f"(hi2)                                  \
        : "memory");                                                         \
  } else {                                                                   \
    asm volatile(                                                            \
        "{\n\t.reg .pred p;\n\t"                                             \
        "setp.le.f32 p, %1, %3;\n\t"                                         \
        "st.shared.u32 [%0], %2;\n\t"                                        \
        "@p add.u32 %0, %0, 128;\n\t}"                                       \
        : "+r"(a)                                                            \
        : "f"(R), "r"(E), "f"(hi2)                                           \
        : "memory");                                                         \
  }
  TMD_APPEND(r0.x, E.x);
  TMD_APPEND(r0.y, E.y);
  TMD_APPEND(r1.x, E.z);
  TMD_APPEND(r1.y, E.w);
#undef TMD_APPEND
}

__device__ __forceinline__ void cull_append1(uint32_t& a, uint32_t e, bool hit) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "st.shared.u32 [%0], %1;\n\t"
      "@p add.u32 %0, %0, 128;\n\t}"
      : "+r"(a)
      : "r"(e), "r"(static_cast<uint32_t>(hit))
      : "memory");
}

// One candidate of a chunk that holds a rounding-band candidate.
template <bool kLocal>
__device__ __forceinline__ void cull_band1(uint32_t& a, uint32_t e, float r2, float d,
                                           const CullLane& L, const double4& pi,
                                           const double4* __restrict__ pos, const Geom& g,
                                           const StageMap& sm) {
  const bool hit = __float_as_uint(d) <= L.wb
                       ? (e & kIdxMask) != L.self &&
                             cull_exact(pi, L.i, entry_slot<kLocal>(e, sm), e, pos, g)
                       : (r2 <= L.hi2 && e != L.self);
  cull_append1(a, e, hit);
}

// Tests a stream segment (a multiple of 4 candidates), 4 per iteration.
template <bool kSelf, bool kLocal>
__device__ __forceinline__ void cull_segment(const float* __restrict__ strm, int fill,
                                             CullLane& L, const double4* __restrict__ pos,
                                             const Geom& g, int cap8, uint32_t* ring_lane,
                                             const StageMap& sm) {
  const uint32_t me = L.self;
  const uint32_t trig = L.rbase + static_cast<uint32_t>(kRingTrigger) * 128u;
#pragma unroll 1
  for (int c0 = 0; c0 < fill; c0 += 4 * kFlushEvery) {
#pragma unroll
  for (int c = c0; c < c0 + 4 * kFlushEvery; c += 4) {
    if (kFlushEvery > 1 && c >= fill) break;
    const float* ch = strm + c * 4;  // chunk of 4: x4 | y4 | z4 | entry4
    const float4 X = *reinterpret_cast<const float4*>(ch);
    const float4 Y = *reinterpret_cast<const float4*>(ch + 4);
    const float4 Z = *reinterpret_cast<const float4*>(ch + 8);
    const uint4 E = *reinterpret_cast<const uint4*>(ch + 12);
    const float2 dxa = __fadd2_rn(L.xi2, f2(X.x, X.y)), dxb = __fadd2_rn(L.xi2, f2(X.z, X.w));
    const float2 dya = __fadd2_rn(L.yi2, f2(Y.x, Y.y)), dyb = __fadd2_rn(L.yi2, f2(Y.z, Y.w));
    const float2 dza = __fadd2_rn(L.zi2, f2(Z.x, Z.y)), dzb = __fadd2_rn(L.zi2, f2(Z.z, Z.w));
    const float2 ra = __ffma2_rn(dza, dza, __ffma2_rn(dya, dya, __fmul2_rn(dxa, dxa)));
    const float2 rb = __ffma2_rn(dzb, dzb, __ffma2_rn(dyb, dyb, __fmul2_rn(dxb, dxb)));
    const float2 da = __fadd2_rn(ra, L.nlo2), db = __fadd2_rn(rb, L.nlo2);
    const uint32_t bmin = min(min(__float_as_uint(da.x), __float_as_uint(da.y)),
                              min(__float_as_uint(db.x), __float_as_uint(db.y)));
    uint32_t a = L.a;
    if (bmin > L.wb) {  // no candidate in the rounding band: FP32 decides
      cull_append4_fp32<kSelf>(a, E, ra, rb, L.hi2, me);
    } else {  // rounding band: the exact FP64 decision there
      const double4 pi = pos[L.i];
      cull_band1<kLocal>(a, E.x, ra.x, da.x, L, pi, pos, g, sm);
      cull_band1<kLocal>(a, E.y, ra.y, da.y, L, pi, pos, g, sm);
      cull_band1<kLocal>(a, E.z, rb.x, db.x, L, pi, pos, g, sm);
      cull_band1<kLocal>(a, E.w, rb.y, db.y, L, pi, pos, g, sm);
    }
    L.a = a;
  }
    if (__any_sync(0xffffffffu, L.a >= trig)) cull_flush(L, cap8, ring_lane);
  }
}

// 3 CTAs per SM (76 registers): at 4 the register cap forces spills and
// rematerialisation into the candidate loop (measured 5 % slower).
// kLocal = false: entries are global slots (variant 3; the sentinel is slot
// N, parked far away). kLocal = true: entries are the brick's staging indices
// (the layout load_halo defines; the sentinel is staging slot stage_cap),
// which the staged force kernel (k_forces_staged, variant 2) gathers from
// shared memory. Groups are 32 consecutive global particles either way.
template <bool kLocal>
__global__ void __launch_bounds__(kBuildThreads, 3)
    k_build_cull(const double4* __restrict__ pos, const int* __restrict__ cell_rank,
                 const int* __restrict__ brick_rank_off, const int* __restrict__ start, Geom g,
                 BrickGeom bg, uint32_t* __restrict__ list, int* __restrict__ nnbr,
                 double4* __restrict__ snap, uint32_t sentinel, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  extern __shared__ __align__(16) float s_f[];  // -x | -y | -z, each stage_cap + 32
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  __shared__ __align__(16) uint32_t s_ring[kBuildThreads / 32][kRingSlots][32];
  __shared__ __align__(16) float s_strm[kBuildThreads / 32][kCullCap * 4];
  __shared__ __align__(16) int4 s_rng[kBuildThreads / 32][11][3];  // per-warp range table
  __shared__ int s_maxc, s_next;
  __shared__ unsigned long long s_ent;
  const int b = blockIdx.x;
  HaloTable ht;
  if (threadIdx.x == 0) { s_maxc = 0; s_ent = 0ull; s_next = kBuildThreads / 32; }
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  if (ht.total > bg.stage_cap) {
    if (threadIdx.x == 0) {
      atomicOr(&ctrl->status, kStatStageOverflow);
      atomicMax(&ctrl->max_halo, ht.total);
    }
    return;
  }
  const int sc = bg.stage_cap + 32;
  float* nx = s_f;
  float* ny = s_f + sc;
  float* nz = s_f + 2 * sc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {  // staging: a warp per halo cell, lanes over its (padded) slots
    const double ox = ht.lo[0] * bg.origin_scale[0];
    const double oy = ht.lo[1] * bg.origin_scale[1];
    const double oz = origin_z(g, ht.lo[2], bg.origin_scale[2]);
    for (int h = warp; h < ht.n; h += kBuildThreads / 32) {
      const int kb = s_off[h], cnt = s_cnt[h], gs = s_gstart[h];
      const uint32_t c = s_code[h];
      for (int q = lane; q < pad4(cnt); q += 32) {
        float x = kFarF, y = kFarF, z = kFarF;
        if (q < cnt) {
          const double4 p = pos[gs + q];
          // same rounding as k_build_brick3: (p + shift) - origin
          x = static_cast<float>((p.x + code_shift(c, 0, g.L[0])) - ox);
          y = static_cast<float>((p.y + code_shift(c, 1, g.L[1])) - oy);
          z = static_cast<float>((p.z + code_shift(c, 2, g.L[2])) - oz);
        }
        nx[kb + q] = -x;
        ny[kb + q] = -y;
        nz[kb + q] = -z;
      }
    }
    if (threadIdx.x < 32) {
      nx[ht.total + threadIdx.x] = -kFarF;
      ny[ht.total + threadIdx.x] = -kFarF;
      nz[ht.total + threadIdx.x] = -kFarF;
    }
  }
  __syncthreads();

  const uint32_t lt_mask = (1u << lane) - 1u;
  const StageMap sm{s_off, s_gstart, ht.n};
  const int ncell_own = ht.e[0] * ht.e[1] * ht.e[2];
  const int cap8 = bg.cap >> 3;
  float* strm = s_strm[warp];
  uint32_t* ring_lane = &s_ring[warp][0][lane];
  const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(ring_lane));
  const float cull2 = bg.hi2 * 1.001f;
  int my_max = 0;
  unsigned long long my_ent = 0;
  // own cells handed out one at a time (cells hold 10-32 particles: a static
  // split leaves warps idle at the block's end)
  for (int oc = warp; oc < ncell_own;) {
    const int ax = oc % ht.e[0], ay = (oc / ht.e[0]) % ht.e[1], az = oc / (ht.e[0] * ht.e[1]);
    const int hc = (ax + 1) + ht.H[0] * ((ay + 1) + ht.H[1] * (az + 1));
    const int ncl = s_cnt[hc];
    if (lane < 11) {  // range table: lane r describes range r
      const int rr = lane;
      const int ri = rr <= 3 ? rr : (rr <= 6 ? 4 : rr - 2);
      const int ca = (rr >= 4 && rr <= 6) ? rr - 4 : 0;
      const int cb = (rr >= 4 && rr <= 6) ? rr - 3 : 3;
      const int oz2 = ri / 3 - 1, oy2 = ri % 3 - 1;
      const int first_yz = oy2 != 0 ? oy2 : oz2;
      const int h0 = hc - 1 + ht.H[0] * (oy2 + ht.H[1] * oz2);
      auto tag_of = [&](int t) {
        const uint32_t code = s_code[h0 + t];
        const int first = (t - 1) != 0 ? (t - 1) : first_yz;
        return code | ((code != 0u && first < 0) ? kFlagIUpper : 0u);
      };
      const int e3 = s_off[h0 + cb];
      const int e1 = ca + 1 < cb ? s_off[h0 + ca + 1] : e3;
      const int e2 = ca + 2 < cb ? s_off[h0 + ca + 2] : e3;
      const uint32_t u0 = tag_of(ca);
      const uint32_t u1 = ca + 1 < cb ? tag_of(ca + 1) : u0;
      const uint32_t u2 = ca + 2 < cb ? tag_of(ca + 2) : u1;
      // staging index -> entry index: + (first global slot - staging offset)
      // of the cell for global entries, + 0 for staging-index entries
      const int b0 = kLocal ? 0 : s_gstart[h0 + ca] - s_off[h0 + ca];
      const int b1 = kLocal ? 0 : (ca + 1 < cb ? s_gstart[h0 + ca + 1] - s_off[h0 + ca + 1] : b0);
      const int b2 = kLocal ? 0 : (ca + 2 < cb ? s_gstart[h0 + ca + 2] - s_off[h0 + ca + 2] : b1);
      s_rng[warp][rr][0] = make_int4(s_off[h0 + ca], e1, e2, e3);
      s_rng[warp][rr][1] = make_int4(static_cast<int>(u0), static_cast<int>(u1),
                                     static_cast<int>(u2), 0);
      s_rng[warp][rr][2] = make_int4(b0, b1, b2, 0);
    }
    __syncwarp();
    for (int p0 = 0; p0 < ncl; p0 += 32) {
      const int q = p0 + lane;
      const bool active = q < ncl;
      const int qi = active ? q : 0;
      CullLane L;
      L.i = s_gstart[hc] + qi;
      const int ki = s_off[hc] + qi;
      L.self = static_cast<uint32_t>(kLocal ? ki : L.i);
      const float xf = -nx[ki], yf = -ny[ki], zf = -nz[ki];
      L.xi2 = f2(xf, xf);
      L.yi2 = f2(yf, yf);
      L.zi2 = f2(zf, zf);
      L.hi2 = active ? bg.hi2 : -1.0f;
      const float nlo = active ? -bg.lo2 : -INFINITY;
      L.nlo2 = f2(nlo, nlo);
      L.wb = __float_as_uint(2.0f * (bg.hi2 - bg.lo2));
      L.rbase = rbase;
      L.a = rbase;
      L.nflush = 0;
      L.dst = list + list_slot(L.i >> 5, bg.cap, L.i & 31, 0);
      // bounding box of the lanes' particles (inactive lanes repeat lane 0's)
      float lox = xf, hix = xf, loy = yf, hiy = yf, loz = zf, hiz = zf;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lox = fminf(lox, __shfl_xor_sync(0xffffffffu, lox, o));
        hix = fmaxf(hix, __shfl_xor_sync(0xffffffffu, hix, o));
        loy = fminf(loy, __shfl_xor_sync(0xffffffffu, loy, o));
        hiy = fmaxf(hiy, __shfl_xor_sync(0xffffffffu, hiy, o));
        loz = fminf(loz, __shfl_xor_sync(0xffffffffu, loz, o));
        hiz = fmaxf(hiz, __shfl_xor_sync(0xffffffffu, hiz, o));
      }
      // The stencil as 11 ranges of x-adjacent halo cells, contiguous in the
      // staging: rows (oz, oy) in the reference order, the middle row split
      // into -x | own | +x so that the own cell is a stream segment of its
      // own (segments: 0 = before the own cell, 1 = own cell, 2 = after).
      // One compaction site and one test site per segment kind keep the
      // kernel small enough for the instruction cache; the ranges of the
      // owned cell are tabulated once per warp (s_rng).
      int r = 0, kq = 0, k1 = 0, k2 = 0, k3 = 0, a0 = 0, a1 = 0, a2 = 0;
      uint32_t t0 = 0, t1 = 0, t2 = 0;
      auto load_range = [&](bool reset) {  // from the warp's range table
        const int4 kk = s_rng[warp][r][0];
        const int4 tt = s_rng[warp][r][1];
        const int4 aa = s_rng[warp][r][2];
        if (reset) kq = kk.x;
        k1 = kk.y;
        k2 = kk.z;
        k3 = kk.w;
        t0 = static_cast<uint32_t>(tt.x);
        t1 = static_cast<uint32_t>(tt.y);
        t2 = static_cast<uint32_t>(tt.z);
        a0 = aa.x;
        a1 = aa.y;
        a2 = aa.z;
      };
      auto seg_of = [](int rr) { return rr < 5 ? 0 : (rr == 5 ? 1 : 2); };
      load_range(true);
      int fill = 0, cur_seg = 0;
      for (;;) {
        bool process = r >= 11;
        if (!process) {
          if (kq >= k3) {  // range exhausted: next range, maybe a new segment
            ++r;
            if (r < 11) load_range(true);
            if (r < 11 && seg_of(r) == cur_seg) continue;
            process = true;
          } else if (fill > kCullCap - 32) {
            process = true;
          } else {  // compact 32 staged slots (padding slots are far: dropped)
            const int k = kq + lane;
            const bool valid = k < k3;
            const int kk = valid ? k : kq;
            const float x = nx[kk], y = ny[kk], z = nz[kk];  // negated coordinates
            const float dx = fmaxf(fmaxf(lox + x, -x - hix), 0.0f);
            const float dy = fmaxf(fmaxf(loy + y, -y - hiy), 0.0f);
            const float dz = fmaxf(fmaxf(loz + z, -z - hiz), 0.0f);
            const bool keep = valid && dx * dx + dy * dy + dz * dz <= cull2;
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
              const uint32_t tag = k >= k2 ? t2 : (k >= k1 ? t1 : t0);
              const int add = k >= k2 ? a2 : (k >= k1 ? a1 : a0);
              const int p = fill + __popc(bal & lt_mask);
              float* ch = strm + (p >> 2) * 16 + (p & 3);
              ch[0] = x;
              ch[4] = y;
              ch[8] = z;
              ch[12] = __uint_as_float(static_cast<uint32_t>(k + add) | tag);
            }
            fill += __popc(bal);
            kq += 32;
            continue;
          }
        }
        if (fill > 0) {  // pad the stream to whole chunks and test it
          const int pad = (4 - (fill & 3)) & 3;
          if (lane < pad) {
            const int p = fill + lane;
            float* ch = strm + (p >> 2) * 16 + (p & 3);
            ch[0] = -kFarF;
            ch[4] = -kFarF;
            ch[8] = -kFarF;
          }
          __syncwarp();
          if (cur_seg == 1) {
            cull_segment<true, kLocal>(strm, fill, L, pos, g, cap8, ring_lane, sm);
          } else {
            cull_segment<false, kLocal>(strm, fill, L, pos, g, cap8, ring_lane, sm);
          }
          __syncwarp();
          fill = 0;
        }
        if (r >= 11) break;
        load_range(false);  // (recomputed rather than kept live across the test)
        cur_seg = seg_of(r);
      }
      if (active) {
        // remaining whole chunks, then the sentinel-padded partial one
        const int fl = static_cast<int>((L.a - L.rbase) >> 7);
        const int whole = fl >> 3, part = fl & 7;
        for (int c = 0; c < whole; ++c) {
          if (L.nflush < cap8) flush_chunk(ring_lane + c * 8 * 32, L.dst);
          ++L.nflush;
          L.dst += 256;
        }
        const int n = L.nflush * 8 + part;
        if (part != 0 && n < bg.cap) {
          uint32_t* pc = ring_lane + whole * 8 * 32;
          for (int r = part; r < 8; ++r) pc[r * 32] = sentinel;
          flush_chunk(pc, L.dst);
        }
        nnbr[L.i] = n < bg.cap ? n : bg.cap;
        snap[L.i] = pos[L.i];
        if (n > bg.cap) atomicOr(&ctrl->status, kStatOverflow);
        my_max = max(my_max, n);
        my_ent += static_cast<unsigned long long>(n);
      }
      __syncwarp();
    }
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(&s_next, 1);
    oc = __shfl_sync(0xffffffffu, nxt, 0);
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
    my_ent += __shfl_xor_sync(0xffffffffu, my_ent, o);
  }
  if (lane == 0) {
    atomicMax(&s_maxc, my_max);
    atomicAdd(&s_ent, my_ent);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&ctrl->max_count, s_maxc);
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctrl->entries), s_ent);
  }
}

// ---------------------------------------------------------------------------
// Full-list build, one thread per particle (k_build_thread): each thread walks
// its 27 neighbour cells in the reference stencil order with the exact FP64
// test, so membership and entry order equal k_build_brick3's. Entries collect
// in a per-thread 8-slot shared-memory buffer and leave as whole 32-B sectors
// of the chunked list. No staging: cheap per particle where cells are sparse
// (the Kremer-Grest melt holds 3 beads per cell), where the brick kernels
// spend their time on per-CTA halo setup. Each stencil row (3 x-adjacent
// cells) loads its three ranks and ranges together before testing.
// (Requesting the next row's ranges and the row after's ranks while a row is
// tested measured slower, 1.21 vs 1.14 ms at 4M: the kernel is bound by the
// instructions it issues, not by these latencies.)
#ifndef TMD_BUILD_THREAD_BATCH
#define TMD_BUILD_THREAD_BATCH 2
#endif
constexpr int kBuildThreadBatch = TMD_BUILD_THREAD_BATCH;
#ifndef TMD_BUILD_THREAD_SLOTS
#define TMD_BUILD_THREAD_SLOTS 24
#endif
constexpr int kBuildThreadSlots = TMD_BUILD_THREAD_SLOTS;  // a multiple of 8
__global__ void __launch_bounds__(kBlock)
    k_build_thread(int n, const double4* __restrict__ pos, const int* __restrict__ cell,
                   const int* __restrict__ start, const int* __restrict__ cell_rank, Geom g,
                   uint32_t* __restrict__ list, int* __restrict__ nnbr, int cap,
                   double4* __restrict__ snap, uint32_t sentinel, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  // kBuildThreadSlots entries per thread wait in shared memory (a batch more
  // rows take the stores of a batch that fills it): a sparse system's ~12 entries per particle
  // then leave together at the end, lanes side by side, instead of chunk by
  // chunk from inside the divergent hit branch
  __shared__ __align__(16) uint32_t s_buf[kBuildThreadSlots + kBuildThreadBatch][kBlock];
  __shared__ double red[kBlock / 32];
  const int i = blockIdx.x * kBlock + threadIdx.x;
  const int t = threadIdx.x;
  int cnt = 0;
  int base = 0;  // entries already written to the list (a multiple of 8)
  if (i < n) {
    const double4 pi = pos[i];
    snap[i] = pi;
    const size_t row = list_slot(i >> 5, cap, i & 31, 0);
    // chunks 0..nch-1 of the buffer become list chunks base/8 .. (capacity permitting)
    auto flush_chunks = [&](int nch) {
      for (int k = 0; k < nch; ++k) {
        const int c8 = (base >> 3) + k;
        if (c8 * 8 >= cap) break;
        uint4 a, b;
        a.x = s_buf[8 * k + 0][t]; a.y = s_buf[8 * k + 1][t];
        a.z = s_buf[8 * k + 2][t]; a.w = s_buf[8 * k + 3][t];
        b.x = s_buf[8 * k + 4][t]; b.y = s_buf[8 * k + 5][t];
        b.z = s_buf[8 * k + 6][t]; b.w = s_buf[8 * k + 7][t];
        uint4* dst = reinterpret_cast<uint4*>(list + row + static_cast<size_t>(c8) * 256);
        dst[0] = a;
        dst[1] = b;
      }
    };
    const int c = cell[i];  // global cell at the last resort
    const int dxy = g.dims[0] * g.dims[1];
    const int cx = c % g.dims[0];
    const int cy = (c / g.dims[0]) % g.dims[1];
    const int cz = c / dxy;
    const int lz = g.zslab ? cz - g.z0 + 1 : cz;  // local layer (slab: ghost layers 0, ldz-1)
    // x neighbours of the row: wrapped column and image code (fixed per particle)
    int txs[3];
    uint32_t cxs[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int tx = cx + k - 1;
      uint32_t code_x = 0;
      if (tx < 0) { tx += g.dims[0]; code_x = 2; }
      else if (tx >= g.dims[0]) { tx -= g.dims[0]; code_x = 1; }
      txs[k] = tx;
      cxs[k] = code_x << 25;
    }
    for (int oz = -1; oz <= 1; ++oz) {
      int tz = lz + oz;
      uint32_t code_z = 0;
      if (g.zslab) {
        code_z = tz == 0 ? g.zcode_lo : (tz == g.ldz - 1 ? g.zcode_hi : 0u);
      } else if (tz < 0) {
        tz += g.dims[2];
        code_z = 2;
      } else if (tz >= g.dims[2]) {
        tz -= g.dims[2];
        code_z = 1;
      }
      for (int oy = -1; oy <= 1; ++oy) {
        int ty = cy + oy;
        uint32_t code_y = 0;
        if (ty < 0) { ty += g.dims[1]; code_y = 2; }
        else if (ty >= g.dims[1]) { ty -= g.dims[1]; code_y = 1; }
        // the row's three cells: ranks and particle ranges loaded together
        // (independent loads) before any candidate is tested
        const int rowc = g.dims[0] * ty + dxy * tz;
        int jb[3], je[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int rt = cell_rank[txs[k] + rowc];
          jb[k] = start[rt];
          je[k] = start[rt + 1];
        }
        // One loop over the row's three ranges (-x, own column, +x in this
        // order): the lanes of a warp sit in ~10 different cells and a warp's
        // trip count is the largest of its lanes' — per row that is closer to
        // the mean than per cell (-3 % at 4M KG beads). Two candidates'
        // positions are requested before either is tested (-8 %; deeper
        // batches lose to their padding slots: the slot past the row's end
        // repeats its last candidate and is skipped).
        uint32_t tg[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int ox = k - 1;
          const int first = ox != 0 ? ox : (oy != 0 ? oy : oz);
          const uint32_t img = cxs[k] | (code_y << 27) | (code_z << 29);
          tg[k] = img | ((img != 0u && first < 0) ? kFlagIUpper : 0u);
        }
        const int n0 = je[0] - jb[0], n01 = n0 + (je[1] - jb[1]), nt = n01 + (je[2] - jb[2]);
        const int o1 = jb[1] - n0, o2 = jb[2] - n01;
        for (int q0 = 0; q0 < nt; q0 += kBuildThreadBatch) {
          double4 pj[kBuildThreadBatch];
          uint32_t en[kBuildThreadBatch];
#pragma unroll
          for (int u = 0; u < kBuildThreadBatch; ++u) {
            const int q = min(q0 + u, nt - 1);
            const bool s1 = q >= n0, s2 = q >= n01;
            const int j = q + (s2 ? o2 : (s1 ? o1 : jb[0]));
            en[u] = static_cast<uint32_t>(j) | (s2 ? tg[2] : (s1 ? tg[1] : tg[0]));
            pj[u] = ldg_pos256(pos + j);
          }
          // every candidate of the batch is decided before any is appended:
          // the FP64 chains are independent and interleave
          bool hit[kBuildThreadBatch];
#pragma unroll
          for (int u = 0; u < kBuildThreadBatch; ++u) {
            double dx, dy, dz;
            pair_delta(pi, pj[u], en[u], g, dx, dy, dz);
            const bool in = exact_r2(dx, dy, dz) <= g.rv2;
            hit[u] = (q0 + u < nt) & (static_cast<int>(en[u] & kIdxMask) != i) & in;
          }
#pragma unroll
          for (int u = 0; u < kBuildThreadBatch; ++u) {
            s_buf[cnt - base][t] = en[u];  // (a miss is overwritten by the next store)
            cnt += hit[u] ? 1 : 0;
          }
          if (cnt - base >= kBuildThreadSlots) {  // buffer full (dense neighbourhoods only)
            flush_chunks(kBuildThreadSlots / 8);
#pragma unroll
            for (int u = 0; u + 1 < kBuildThreadBatch; ++u) {  // entries past the flushed chunks
              if (cnt - base > kBuildThreadSlots + u) s_buf[u][t] = s_buf[kBuildThreadSlots + u][t];
            }
            base += kBuildThreadSlots;
          }
        }
      }
    }
    {  // the waiting entries: whole chunks, then the sentinel-padded last one
      const int rem = cnt - base;
      for (int r = rem; r < ((rem + 7) & ~7); ++r) s_buf[r][t] = sentinel;
      flush_chunks((rem + 7) >> 3);
    }
    nnbr[i] = cnt < cap ? cnt : cap;
    if (cnt > cap) atomicOr(&ctrl->status, kStatOverflow);
  }
  int m = cnt;
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(&ctrl->max_count, m);
  const double tot = block_sum<kBlock>(static_cast<double>(cnt), red);
  if (threadIdx.x == 0 && tot > 0.0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctrl->entries),
              static_cast<unsigned long long>(tot));
  }
}

// ---------------------------------------------------------------------------
// LJ pair term of one list entry (compute_pair_forces, neighbor_list.hpp:
// 150-187, full-list form): image shift and the reference's rounding
// orientation from the entry tag (pair_delta), so the cutoff test sees the
// reference's r2 bit for bit.
__device__ __forceinline__ void lj_accumulate(const double4& pi, double xj, double yj,
                                              double zj, uint32_t ent, const Geom& g,
                                              const LjConst& lj, double& ax, double& ay,
                                              double& az, double& e, double& w, bool& zero) {
  double dx, dy, dz;
  pair_delta(pi, make_double4(xj, yj, zj, 0.0), ent, g, dx, dy, dz);
  const double r2 = exact_r2(dx, dy, dz);
  if (r2 < lj.rc2) {
    zero |= (r2 == 0.0);
    const double ri2 = rcp_nr(r2);
    const double inv = lj.sigma2 * ri2;
    const double i6 = inv * inv * inv;
    const double ff = lj.eps24 * (2.0 * i6 * i6 - i6) * ri2;
    e += lj.eps4 * (i6 * i6 - i6) - lj.shift;
    w += ff * r2;
    ax += ff * dx;
    ay += ff * dy;
    az += ff * dz;
  }
}

// ---------------------------------------------------------------------------
// Variant 2: LJ forces with the neighbour positions gathered from SHARED
// memory. One CTA per brick stages the brick's halo block — the staging
// layout of load_halo, which the list build used, so list entries are staging
// indices (k_build_cull<true>, k_build_brick3<false>) — as x|y pairs (double2)
// and z (double) with 16-B and 8-B cp.async copies straight from the position
// buffer. Each gather is then one LDS.128 + one LDS.64 instead of a 32-B L1
// line request per entry (the bound of k_forces_l1, one L1 wavefront per
// entry): ncu measures ~0.6 shared wavefronts per gather (half
// of them bank conflicts of the random indices). Threads = the brick's
// particles (a brick fuller than the CTA loops). Same pair arithmetic and
// per-particle entry order as k_forces_l1: forces bitwise equal.
//
// Measured on B200 at 1M (scripts/force_variants.py): 0.287 ms
// against 0.273 ms for k_forces_l1 — the L1 relief is real (L1TEX 66 %), but
// the CTA-per-brick structure pays a staging phase and a tail per brick
// (barrier stalls 27 %: on the FCC lattice a fifth of the 2x2x4 bricks hold
// more than 320 particles), and a persistent warp-specialised version (cp.async
// producer warps, mbarrier-handed stage buffers) measured 0.345 ms: too few
// groups per staged brick to keep its consumers fed. So it is not the default.
#ifndef TMD_STAGED_MINB_SMALL
#define TMD_STAGED_MINB_SMALL 5
#endif
#ifndef TMD_STAGED_MINB_LARGE
#define TMD_STAGED_MINB_LARGE 3
#endif
template <int kThreads>
constexpr int staged_min_blocks() {
  return kThreads <= 192 ? TMD_STAGED_MINB_SMALL : TMD_STAGED_MINB_LARGE;
}
#ifndef TMD_STAGED_UNROLL
#define TMD_STAGED_UNROLL 1
#endif
constexpr int kStagedUnroll = TMD_STAGED_UNROLL;  // gathers in flight per thread

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int kThreads, int kMode>
__global__ void __launch_bounds__(kThreads, staged_min_blocks<kThreads>())
    k_forces_staged(const double4* __restrict__ pos, const int* __restrict__ cell_rank,
                    const int* __restrict__ brick_rank_off, const int* __restrict__ start,
                    Geom g, BrickGeom bg, LjConst lj, const uint32_t* __restrict__ list,
                    const int* __restrict__ nnbr, double* __restrict__ fx,
                    double* __restrict__ fy, double* __restrict__ fz,
                    double* __restrict__ part_e, double* __restrict__ part_w,
                    const long long* __restrict__ id, Integ it, Ctrl* ctrl) {
  const int b = blockIdx.x;
  if (ctrl->halt) {  // speculative blocks: positions carried to the other buffer
    if (kMode == kFused && it.halt_copy) {
      const int bs = start[brick_rank_off[b]], be = start[brick_rank_off[b + 1]];
      for (int i = bs + threadIdx.x; i < be; i += kThreads) it.pos_out[i] = pos[i];
    }
    return;
  }
  extern __shared__ __align__(16) double2 s_xy[];  // [stage_cap + 1], then z [stage_cap + 1]
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  __shared__ double red[3 * (kThreads / 32)];
  double* s_z = reinterpret_cast<double*>(s_xy + bg.stage_cap + 1);
  HaloTable ht;
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  const bool fits = ht.total <= bg.stage_cap;  // (the build flags an overfull halo)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (fits) {
    // a warp per x-row of the halo (H0 cells, contiguous in the staging),
    // lanes over the row's slots; padding slots are never listed
    const int H0 = ht.H[0];
    const int rows = ht.H[1] * ht.H[2];
    for (int r = warp; r < rows; r += kThreads / 32) {
      const int h0 = r * H0;
      const int k0 = s_off[h0], k1 = s_off[h0 + H0];
      for (int k = k0 + lane; k < k1; k += 32) {
        int h = h0;
#pragma unroll
        for (int t = 1; t < 4; ++t) h += (t < H0 && k >= s_off[h0 + t]) ? 1 : 0;
        const int q = k - s_off[h];
        if (q < s_cnt[h]) {
          const double4* src = pos + s_gstart[h] + q;
          cp_async16(s_xy + k, src);
          cp_async8(s_z + k, reinterpret_cast<const double*>(src) + 2);
        }
      }
    }
    if (threadIdx.x == 0) {  // the sentinel slot
      s_xy[bg.stage_cap] = make_double2(kFarD, kFarD);
      s_z[bg.stage_cap] = kFarD;
    }
    cp_async_wait_all();
  }
  __syncthreads();
  double e = 0.0, w = 0.0, ke = 0.0, d2 = 0.0;
  if (fits) {
    for (int i = ht.bs + threadIdx.x; i < ht.be; i += kThreads) {
      const double4 pi = pos[i];
      const int cnt = nnbr[i];
      const uint32_t* row = list + list_slot(i >> 5, bg.cap, i & 31, 0);
      double ax = 0.0, ay = 0.0, az = 0.0;
      bool zero = false;
      // the next chunk's entries are loaded while this one is evaluated (the
      // list streams from DRAM; shared-memory gathers leave little latency
      // for the warp schedulers to hide it behind)
      uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
      if (cnt > 0) {
        n0 = __ldg(reinterpret_cast<const uint4*>(row));
        n1 = __ldg(reinterpret_cast<const uint4*>(row + 4));
      }
      for (int c0 = 0; c0 < cnt; c0 += 8) {
        const uint32_t ents[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
        if (c0 + 8 < cnt) {
          n0 = __ldg(reinterpret_cast<const uint4*>(row + (c0 + 8) * 32));
          n1 = __ldg(reinterpret_cast<const uint4*>(row + (c0 + 8) * 32 + 4));
        }
#pragma unroll
        for (int u0 = 0; u0 < 8; u0 += kStagedUnroll) {
          double2 xy[kStagedUnroll];
          double zj[kStagedUnroll];
#pragma unroll
          for (int u = 0; u < kStagedUnroll; ++u) {
            const int k = static_cast<int>(ents[u0 + u] & kIdxMask);
            xy[u] = s_xy[k];
            zj[u] = s_z[k];
          }
#pragma unroll
          for (int u = 0; u < kStagedUnroll; ++u) {
            lj_accumulate(pi, xy[u].x, xy[u].y, zj[u], ents[u0 + u], g, lj, ax, ay, az, e, w,
                          zero);
          }
        }
      }
      if (zero) {  // r2 == 0: coincident particles (neighbor_list.hpp:166-170)
        for (int k = 0; k < cnt; ++k) {
          const uint32_t ent = row[(k >> 3) * 256 + (k & 7)];
          const int kk = static_cast<int>(ent & kIdxMask);
          double dx, dy, dz;
          pair_delta(pi, make_double4(s_xy[kk].x, s_xy[kk].y, s_z[kk], 0.0), ent, g, dx, dy,
                     dz);
          if (exact_r2(dx, dy, dz) == 0.0) {
            const int h = halo_of(kk, s_off, ht.n);
            record_error(ctrl, kStatOverlap, id[i], id[s_gstart[h] + (kk - s_off[h])]);
            break;
          }
        }
      }
      integrate_one<kMode>(i, pi, ax, ay, az, it, ctrl, ke, d2);
      if (kMode != kFused) {  // a fused step's force only feeds its own kicks
        fx[i] = ax;
        fy[i] = ay;
        fz[i] = az;
      }
    }
  }
  block_partials<kMode, kThreads>(e, w, ke, d2, red, part_e, part_w, it, ctrl);  // (b = blockIdx.x)
}

// Threads of a staged force CTA: one per particle of a brick (2x2x2 cells
// hold ~150 particles at the BASELINE density, 2x2x4 ~300).
constexpr int kStagedThreadsSmall = 192;
constexpr int kStagedThreadsLarge = 320;

// Dynamic shared memory of k_forces_staged: x|y (double2) and z (double) per
// staging slot + the sentinel.
inline size_t staged_smem_bytes(int stage_cap) {
  return static_cast<size_t>(stage_cap + 1) * 3 * sizeof(double);
}
constexpr size_t kStagedSmemMax = 200 * 1024;

// ---------------------------------------------------------------------------
// The epilogue's per-particle operands (velocities, mass, snapshot, bond
// table) stream from DRAM once per step and are first touched after the list
// loop: requested into L2 at the top of the kernel their latency runs under
// the gathers instead of after them. Matters where a thread's list is short
// (the Kremer-Grest melt: ~12 entries, the kernel waits on loads half the
// time); a long list hides it anyway. (The small-system kernel
// k_forces_lanes works out of L2: the same prefetches measured no gain.)
#ifndef TMD_FORCE_PREFETCH
#define TMD_FORCE_PREFETCH 1
#endif
// blocks ahead whose first loads (position, count, first list chunk) a block
// requests into L2: about one wave of resident blocks (148 SMs x 7), i.e. the
// block that starts when this one ends (KG 4M: 0.323 -> 0.313 ms; 2072 ahead
// 0.319; the dense fluids are indifferent)
#ifndef TMD_AHEAD_PREFETCH
#define TMD_AHEAD_PREFETCH 1036
#endif
#ifndef TMD_LIST_PREFETCH
#define TMD_LIST_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_line(const void* p) {
#if TMD_FORCE_PREFETCH == 2
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#elif TMD_FORCE_PREFETCH == 1
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
  (void)p;
#endif
}
template <int kMode>
__device__ __forceinline__ void prefetch_epilogue(int i, const Integ& it) {
  if (kMode == kForcesOnly) return;
  prefetch_line(it.vx + i);
  prefetch_line(it.vy + i);
  prefetch_line(it.vz + i);
  prefetch_line(it.mass + i);
  if (kMode == kFused) prefetch_line(it.snap + i);
  if (kMode == kFused && it.exp) prefetch_line(it.exp + i);  // fused halo's export map
  if (it.bt.on) {
    prefetch_line(it.bt.cnt + i);
    prefetch_line(it.bt.ent + static_cast<size_t>(i) * kMaxBonds);
  }
}

// ---------------------------------------------------------------------------
// Variant 3: thread per particle over the sector-chunked list with GLOBAL
// slots (groups = 32 consecutive particles of the brick-major order). Each
// chunk of 8 entries is two 16-B loads; each gather is one 256-bit
// LDG.E.ENL2.256 of the packed position (one L1 sector request per entry).
// No staging, no shared memory: occupancy is register-limited only.
template <int kUnroll, int kMode>
__global__ void __launch_bounds__(128)
    k_forces_l1(int n, const double4* __restrict__ pos, const uint32_t* __restrict__ list,
                const int* __restrict__ nnbr, int cap, Geom g, LjConst lj,
                double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz,
                double* __restrict__ part_e, double* __restrict__ part_w,
                const long long* __restrict__ id, Integ it, Ctrl* ctrl) {
  if (ctrl->halt) {  // steps after a due rebuild are no-ops (speculative blocks: positions
                     // carried to the other buffer)
    const int i = blockIdx.x * 128 + threadIdx.x;
    if (kMode == kFused && it.halt_copy && i < n) it.pos_out[i] = pos[i];
    return;
  }
  __shared__ double red[3 * 4];
  const int i = blockIdx.x * 128 + threadIdx.x;
  double e = 0.0, w = 0.0, ke = 0.0, d2 = 0.0;
  if (i < n) {
    const double4 pi = pos[i];
    const int cnt = nnbr[i];
    const uint32_t* row = list + list_slot(i >> 5, cap, i & 31, 0);
    prefetch_epilogue<kMode>(i, it);
#if TMD_AHEAD_PREFETCH
    {  // the first loads of the block that starts when this one ends
      const int ia = i + TMD_AHEAD_PREFETCH * 128;
      if (ia < n) {
        prefetch_line(pos + ia);
        if ((threadIdx.x & 31) == 0) prefetch_line(nnbr + ia);
        prefetch_line(list + list_slot(ia >> 5, cap, ia & 31, 0));
      }
    }
#endif
    double ax = 0.0, ay = 0.0, az = 0.0;
    bool zero = false;
    for (int c0 = 0; c0 < cnt; c0 += 8) {
      // the next chunk of the list into L2 while this one is worked on: the
      // list streams from DRAM, and a chunk's load would otherwise wait for
      // it right before its gathers (16.4M: 4.02 -> 3.89 ms; two chunks
      // ahead, or into L1, measured no better)
      if (TMD_LIST_PREFETCH && c0 + 8 < cnt) prefetch_line(row + (c0 + 8) * 32);
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32));
      const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32 + 4));
      const uint32_t ents[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int u0 = 0; u0 < 8; u0 += kUnroll) {
        double4 pj[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) pj[u] = ldg_pos256(pos + (ents[u0 + u] & kIdxMask));
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          lj_accumulate(pi, pj[u].x, pj[u].y, pj[u].z, ents[u0 + u], g, lj, ax, ay, az, e, w,
                        zero);
        }
      }
    }
    if (zero) {
      for (int k = 0; k < cnt; ++k) {
        const uint32_t ent = row[(k >> 3) * 256 + (k & 7)];
        const double4 pj = pos[ent & kIdxMask];
        double dx, dy, dz;
        pair_delta(pi, pj, ent, g, dx, dy, dz);
        if (exact_r2(dx, dy, dz) == 0.0) {
          record_error(ctrl, kStatOverlap, id[i], id[ent & kIdxMask]);
          break;
        }
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
  block_partials<kMode, 128>(e, w, ke, d2, red, part_e, part_w, it, ctrl);
}

// ---------------------------------------------------------------------------
// Variant 3 for small systems (the 32,000-particle configs[0], or a slab of
// a many-GPU run): kLanes consecutive threads share one particle. Thread
// (p, s) takes chunks s, s + kLanes, ... of p's list, so one particle's ~10
// chunks are gathered kLanes-wide instead of by one serial thread: at 32K a
// one-lane grid is 1,000 warps (7 per SM, latency-bound); eight lanes make
// it 8,000. The lanes' partial forces are combined by a fixed xor-shuffle
// tree (deterministic, like every other reduction here); energy and virial
// partials go to the block sums lane by lane. Same list, same pair
// arithmetic as k_forces_l1; only the summation order of a particle's force
// differs (a rounding-level difference, within the parity tolerances).
// Resident blocks per SM the register budget must allow (a grid of 128-
// particle blocks fits one wave down to ~32K particles).
// Particles per block of k_forces_lanes: 32, so that a small system's grid
// (1,000 blocks at 32K) spreads evenly over the 148 SMs instead of 250
// blocks of 128 (102 SMs running two, 46 one).
constexpr int kLanesPPB = 32;
// resident blocks per SM: 768 / 1024 / 1024 threads per SM for 2 / 4 / 8 lanes
constexpr int lanes_min_blocks(int lanes) { return lanes == 2 ? 12 : (lanes == 4 ? 8 : 4); }

template <int kUnroll, int kMode, int kLanes>
__global__ void __launch_bounds__(kLanesPPB * kLanes, lanes_min_blocks(kLanes))
    k_forces_lanes(int n, const double4* __restrict__ pos, const uint32_t* __restrict__ list,
                   const int* __restrict__ nnbr, int cap, Geom g, LjConst lj,
                   double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz,
                   double* __restrict__ part_e, double* __restrict__ part_w,
                   const long long* __restrict__ id, Integ it, Ctrl* ctrl) {
  if (ctrl->halt) {  // (see k_forces_l1)
    const int i = blockIdx.x * kLanesPPB + threadIdx.x;
    if (kMode == kFused && it.halt_copy && threadIdx.x < kLanesPPB && i < n) {
      it.pos_out[i] = pos[i];
    }
    return;
  }
  constexpr int kThreads = kLanesPPB * kLanes;
  __shared__ double red[3 * (kThreads / 32)];
  const int sub = threadIdx.x % kLanes;
  const int i = blockIdx.x * kLanesPPB + threadIdx.x / kLanes;
  double e = 0.0, w = 0.0, ke = 0.0, d2 = 0.0;
  double ax = 0.0, ay = 0.0, az = 0.0;
  bool zero = false;
  double4 pi = make_double4(0.0, 0.0, 0.0, 0.0);
  int cnt = 0;
  const uint32_t* row = list;
  if (i < n) {
    pi = pos[i];
    cnt = nnbr[i];
    row = list + list_slot(i >> 5, cap, i & 31, 0);
    for (int c0 = sub * 8; c0 < cnt; c0 += 8 * kLanes) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32));
      const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32 + 4));
      const uint32_t ents[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int u0 = 0; u0 < 8; u0 += kUnroll) {
        double4 pj[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) pj[u] = ldg_pos256(pos + (ents[u0 + u] & kIdxMask));
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          lj_accumulate(pi, pj[u].x, pj[u].y, pj[u].z, ents[u0 + u], g, lj, ax, ay, az, e, w,
                        zero);
        }
      }
    }
  }
  // lanes of one particle are kLanes consecutive threads of one warp
#pragma unroll
  for (int o = 1; o < kLanes; o <<= 1) {
    ax += __shfl_xor_sync(0xffffffffu, ax, o);
    ay += __shfl_xor_sync(0xffffffffu, ay, o);
    az += __shfl_xor_sync(0xffffffffu, az, o);
  }
  // any lane of the particle saw r2 == 0: its lane 0 finds and reports it
  const unsigned zmask = __ballot_sync(0xffffffffu, zero);
  const unsigned grp = ((1u << kLanes) - 1u) << ((threadIdx.x & 31) & ~(kLanes - 1));
  if (i < n && sub == 0 && (zmask & grp)) {
    for (int k = 0; k < cnt; ++k) {
      const uint32_t ent = row[(k >> 3) * 256 + (k & 7)];
      const double4 pj = pos[ent & kIdxMask];
      double dx, dy, dz;
      pair_delta(pi, pj, ent, g, dx, dy, dz);
      if (exact_r2(dx, dy, dz) == 0.0) {
        record_error(ctrl, kStatOverlap, id[i], id[ent & kIdxMask]);
        break;
      }
    }
  }
  if (i < n && sub == 0) {
    if (it.bt.on) bond_accumulate(i, pi, pos, it.bt, g, id, ctrl, ax, ay, az, e, w);
    integrate_one<kMode>(i, pi, ax, ay, az, it, ctrl, ke, d2);
    if (kMode != kFused) {
      fx[i] = ax;
      fy[i] = ay;
      fz[i] = az;
    }
  }
  block_partials<kMode, kThreads>(e, w, ke, d2, red, part_e, part_w, it, ctrl);
}

// Tap for variant 3: chunked global-slot list -> ELL-transposed copy.
__global__ void __launch_bounds__(128)
    k_decode_chunked(int n, const uint32_t* __restrict__ list, const int* __restrict__ nnbr,
                     int cap, uint32_t* __restrict__ out, int stride) {
  const int i = blockIdx.x * 128 + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < nnbr[i]; ++k) {
    out[static_cast<size_t>(k) * stride + i] = list[list_slot(i >> 5, cap, i & 31, k)];
  }
}

// ---------------------------------------------------------------------------
// Parity/accounting tap: rewrite the staging-index list of variant 2 into the
// global-index ELL-transposed form (entry k of particle i at out[k*stride + i],
// same tag bits) consumed by the host-side pair dump and the in-cut counter.
__global__ void __launch_bounds__(128)
    k_decode_list(const int* __restrict__ cell_rank, const int* __restrict__ brick_rank_off,
                  const int* __restrict__ start, Geom g, BrickGeom bg,
                  const uint32_t* __restrict__ list, const int* __restrict__ nnbr,
                  uint32_t* __restrict__ out, int stride) {
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  const int b = blockIdx.x;
  HaloTable ht;
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  for (int i = ht.bs + threadIdx.x; i < ht.be; i += 128) {
    for (int k = 0; k < nnbr[i]; ++k) {
      const uint32_t ent = list[list_slot(i >> 5, bg.cap, i & 31, k)];
      const int loc = static_cast<int>(ent & kIdxMask);
      const int h = halo_of(loc, s_off, ht.n);
      const uint32_t j = static_cast<uint32_t>(s_gstart[h] + (loc - s_off[h]));
      out[static_cast<size_t>(k) * stride + i] = j | (ent & ~kIdxMask);
    }
  }
}

}  // namespace tmd
