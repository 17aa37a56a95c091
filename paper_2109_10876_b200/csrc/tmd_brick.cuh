// Brick-staged kernels (variant 2, the default): one CTA per brick of up to
// 2x2x2 cells. Particles are stored brick-major (brick, then cell x-fastest
// inside the brick, then id), so a brick's own particles are one contiguous
// range and its 27-cell neighbourhood is the (Bx+2)(By+2)(Bz+2) halo block.
//
// The CTA stages the halo block into shared memory once and every list entry
// is a halo-local index into that staging layout, so the gathers of the hot
// loop are LDS (bank-conflict bound) instead of L1 line fetches.
//
// List layout (sector-chunked ELL): particles of a brick form groups of 32
// (lane = brick offset % 32). Entry k of lane l of group g lives at
//   list[g*cap*32 + (k/8)*256 + l*8 + k%8]
// so each lane owns whole 32-byte sectors: the build flushes 8 entries with
// two 16-B stores, the force kernel reads 8 entries with two 16-B loads, and
// a warp touches 1 KB of contiguous memory per chunk.
#pragma once

#include "tmd_device.cuh"

namespace tmd {

constexpr int kMaxHalo = 64;  // (2+2)^3

struct BrickGeom {
  int B[3];      // brick edge in cells (min(2, dims))
  int nb[3];     // bricks per axis
  int nbricks;
  int cap;       // list entries per particle (multiple of 8)
  int stage_cap_f32;  // build staging capacity (particles)
  int stage_cap_f64;  // force staging capacity (particles)
  float lo2, hi2;     // FP32 prefilter band around rv2 (exact FP64 inside)
  double origin_scale[3];  // cell_len (brick origin = lo * cell_len)
};

struct HaloTable {
  int n;                  // halo cells
  int H[3];               // halo extent
  int lo[3];              // first owned cell of the brick
  int e[3];               // owned extent
  int total;              // staged particles
  int bs, be;             // brick particle range
};

// Fills the halo metadata of brick b into shared memory (any block size >= 64
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
  ht.lo[0] = bx * bg.B[0];
  ht.lo[1] = by * bg.B[1];
  ht.lo[2] = bz * bg.B[2];
  for (int k = 0; k < 3; ++k) {
    ht.e[k] = min(bg.B[k], g.dims[k] - ht.lo[k]);
    ht.H[k] = ht.e[k] + 2;
  }
  ht.n = ht.H[0] * ht.H[1] * ht.H[2];
  const int t = threadIdx.x;
  if (t < ht.n) {
    const int h[3] = {t % ht.H[0], (t / ht.H[0]) % ht.H[1], t / (ht.H[0] * ht.H[1])};
    int gc[3];
    uint32_t code = 0;
    for (int k = 0; k < 3; ++k) {
      int raw = ht.lo[k] + h[k] - 1;
      uint32_t c2 = 0;
      if (raw < 0) { raw += g.dims[k]; c2 = 2; }
      else if (raw >= g.dims[k]) { raw -= g.dims[k]; c2 = 1; }
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
  if (t == 0) {
    int run = 0;
    for (int h = 0; h < ht.n; ++h) {
      s_off[h] = run;
      run += s_cnt[h];
    }
    s_off[ht.n] = run;
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

// ---------------------------------------------------------------------------
// Groups per brick (for the list layout): n_groups[b] = ceil(n_b / 32).
__global__ void __launch_bounds__(128)
    k_brick_groups(int nbricks, const int* __restrict__ brick_rank_off,
                   const int* __restrict__ start, int* __restrict__ ngroups, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  const int b = blockIdx.x * 128 + threadIdx.x;
  if (b >= nbricks) return;
  const int n = start[brick_rank_off[b + 1]] - start[brick_rank_off[b]];
  ngroups[b] = (n + 31) >> 5;
}

__device__ __forceinline__ size_t list_slot(int group, int cap, int lane, int k) {
  return static_cast<size_t>(group) * cap * 32 + static_cast<size_t>(k >> 3) * 256 +
         lane * 8 + (k & 7);
}

// ---------------------------------------------------------------------------
// Full-list build, brick-staged (the full-list form of build_sorted_list,
// neighbor_list.hpp:51-111). One warp per owned cell of the brick, lanes =
// that cell's particles; candidates (the 27 surrounding halo cells, read as
// warp-broadcast LDS.128) are filtered in FP32 brick-relative coordinates.
// Only candidates inside the band |r2 - rv2| <= delta take the exact FP64
// test with the reference's rounding, so membership is bit-identical to the
// reference while almost all arithmetic runs on the FP32 pipe.
constexpr int kBuildThreads = 256;

__global__ void __launch_bounds__(kBuildThreads)
    k_build_brick(const double4* __restrict__ pos, const int* __restrict__ cell_rank,
                  const int* __restrict__ brick_rank_off, const int* __restrict__ start,
                  const int* __restrict__ group_off, Geom g, BrickGeom bg,
                  uint32_t* __restrict__ list, int* __restrict__ nnbr,
                  double4* __restrict__ snap, Ctrl* ctrl) {
  if (!ctrl->rebuild) return;
  extern __shared__ float4 s_f[];  // staged FP32 brick-relative images
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  __shared__ uint32_t s_buf[kBuildThreads / 32][32][8];
  __shared__ int s_maxc;
  __shared__ unsigned long long s_ent;
  const int b = blockIdx.x;
  HaloTable ht;
  if (threadIdx.x == 0) { s_maxc = 0; s_ent = 0ull; }
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  const bool staged = ht.total <= bg.stage_cap_f32;
  const double ox = ht.lo[0] * bg.origin_scale[0];
  const double oy = ht.lo[1] * bg.origin_scale[1];
  const double oz = ht.lo[2] * bg.origin_scale[2];
  if (staged) {
    for (int k = threadIdx.x; k < ht.total; k += kBuildThreads) {
      const int h = halo_of(k, s_off, ht.n);
      const double4 p = pos[s_gstart[h] + (k - s_off[h])];
      const uint32_t c = s_code[h];
      s_f[k] = make_float4(
          static_cast<float>((p.x + code_shift(c, 0, g.L[0])) - ox),
          static_cast<float>((p.y + code_shift(c, 1, g.L[1])) - oy),
          static_cast<float>((p.z + code_shift(c, 2, g.L[2])) - oz), 0.f);
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncell_own = ht.e[0] * ht.e[1] * ht.e[2];
  const int gbase = group_off[b];
  int my_max = 0;
  unsigned long long my_ent = 0;
  for (int oc = warp; oc < ncell_own; oc += kBuildThreads / 32) {
    const int ax = oc % ht.e[0], ay = (oc / ht.e[0]) % ht.e[1], az = oc / (ht.e[0] * ht.e[1]);
    const int hc = (ax + 1) + ht.H[0] * ((ay + 1) + ht.H[1] * (az + 1));
    const int ncl = s_cnt[hc];
    for (int p0 = 0; p0 < ncl; p0 += 32) {
      const int q = p0 + lane;
      const bool active = q < ncl;
      const int i = s_gstart[hc] + (active ? q : 0);
      const double4 pi = pos[i];
      float xf, yf, zf;
      if (staged) {
        const float4 f = s_f[s_off[hc] + (active ? q : 0)];
        xf = f.x; yf = f.y; zf = f.z;
      } else {
        xf = static_cast<float>(pi.x - ox);
        yf = static_cast<float>(pi.y - oy);
        zf = static_cast<float>(pi.z - oz);
      }
      const int ib = i - ht.bs;
      const int grp = gbase + (ib >> 5), gl = ib & 31;
      int n = 0;
      for (int oz2 = -1; oz2 <= 1; ++oz2) {
        for (int oy2 = -1; oy2 <= 1; ++oy2) {
          for (int ox2 = -1; ox2 <= 1; ++ox2) {
            const int h = hc + ox2 + ht.H[0] * (oy2 + ht.H[1] * oz2);
            const uint32_t code = s_code[h];
            const int first = ox2 != 0 ? ox2 : (oy2 != 0 ? oy2 : oz2);
            const uint32_t tag = code | ((code != 0u && first < 0) ? kFlagIUpper : 0u);
            const bool same = s_gcell[h] == s_gcell[hc];
            const int cnt = s_cnt[h], off = s_off[h], gs = s_gstart[h];
            for (int c = 0; c < cnt; ++c) {
              float4 f;
              if (staged) {
                f = s_f[off + c];
              } else {
                const double4 p = pos[gs + c];
                f = make_float4(static_cast<float>((p.x + code_shift(code, 0, g.L[0])) - ox),
                                static_cast<float>((p.y + code_shift(code, 1, g.L[1])) - oy),
                                static_cast<float>((p.z + code_shift(code, 2, g.L[2])) - oz),
                                0.f);
              }
              const float dx = xf - f.x, dy = yf - f.y, dz = zf - f.z;
              const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              if (!active || r2f > bg.hi2) continue;
              const int j = gs + c;
              if (same && j == i) continue;
              const uint32_t ent = static_cast<uint32_t>(off + c) | tag;
              bool in = r2f < bg.lo2;
              if (!in) {  // inside the rounding band: decide exactly in FP64
                const double4 pj = pos[j];
                double ex, ey, ez;
                pair_delta(pi, pj, static_cast<uint32_t>(j & kIdxMask) | tag, g, ex, ey, ez);
                in = exact_r2(ex, ey, ez) <= g.rv2;
              }
              if (in) {
                s_buf[warp][lane][n & 7] = ent;
                ++n;
                if ((n & 7) == 0 && n <= bg.cap) {
                  const uint4* src = reinterpret_cast<const uint4*>(&s_buf[warp][lane][0]);
                  uint4* dst = reinterpret_cast<uint4*>(list + list_slot(grp, bg.cap, gl, n - 8));
                  dst[0] = src[0];
                  dst[1] = src[1];
                }
              }
            }
          }
        }
      }
      if (active) {
        if ((n & 7) != 0 && n <= bg.cap) {
          const uint4* src = reinterpret_cast<const uint4*>(&s_buf[warp][lane][0]);
          uint4* dst = reinterpret_cast<uint4*>(list + list_slot(grp, bg.cap, gl, n & ~7));
          dst[0] = src[0];
          dst[1] = src[1];
        }
        nnbr[i] = n < bg.cap ? n : bg.cap;
        snap[i] = pi;
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
// LJ forces over the brick-staged list (compute_pair_forces,
// neighbor_list.hpp:150-187, full-list form). The halo block is staged as
// unshifted SoA doubles; image shifts and the reference's rounding
// orientation come from the entry tag (pair_delta), so the cutoff test sees
// the reference's r2 bit for bit.
constexpr int kForceThreads = 192;

struct StagedPos {
  const double* sx;
  const double* sy;
  const double* sz;
};

__global__ void __launch_bounds__(kForceThreads)
    k_forces_brick(const double4* __restrict__ pos, const int* __restrict__ cell_rank,
                   const int* __restrict__ brick_rank_off, const int* __restrict__ start,
                   const int* __restrict__ group_off, Geom g, BrickGeom bg, LjConst lj,
                   const uint32_t* __restrict__ list, const int* __restrict__ nnbr,
                   double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz,
                   double* __restrict__ part_e, double* __restrict__ part_w,
                   const long long* __restrict__ id, Ctrl* ctrl) {
  extern __shared__ double s_d[];
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  __shared__ double red[kForceThreads / 32];
  const int b = blockIdx.x;
  HaloTable ht;
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  const bool staged = ht.total <= bg.stage_cap_f64;
  const int cap_s = bg.stage_cap_f64;
  double* sx = s_d;
  double* sy = s_d + cap_s;
  double* sz = s_d + 2 * cap_s;
  if (staged) {
    for (int k = threadIdx.x; k < ht.total; k += kForceThreads) {
      const int h = halo_of(k, s_off, ht.n);
      const double4 p = pos[s_gstart[h] + (k - s_off[h])];
      sx[k] = p.x;
      sy[k] = p.y;
      sz[k] = p.z;
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb_i = ht.be - ht.bs;
  const int ngr = (nb_i + 31) >> 5;
  double e = 0.0, w = 0.0;
  for (int gl = warp; gl < ngr; gl += kForceThreads / 32) {
    const int ib = gl * 32 + lane;
    const bool active = ib < nb_i;
    const int i = ht.bs + (active ? ib : 0);
    const double4 pi = pos[i];
    const int cnt = active ? nnbr[i] : 0;
    const uint32_t* row = list + list_slot(group_off[b] + gl, bg.cap, lane, 0);
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int c0 = 0; c0 < cnt; c0 += 8) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32));
      const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(row + c0 * 32 + 4));
      const uint32_t ents[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + u >= cnt) break;
        const uint32_t ent = ents[u];
        const int k = static_cast<int>(ent & kIdxMask);
        double4 pj;
        if (staged) {
          pj = make_double4(sx[k], sy[k], sz[k], 0.0);
        } else {
          const int h = halo_of(k, s_off, ht.n);
          pj = pos[s_gstart[h] + (k - s_off[h])];
        }
        double dx, dy, dz;
        pair_delta(pi, pj, ent, g, dx, dy, dz);
        const double r2 = exact_r2(dx, dy, dz);
        if (r2 < lj.rc2) {
          if (r2 == 0.0) {
            const int h = halo_of(k, s_off, ht.n);
            record_error(ctrl, kStatOverlap, id[i], id[s_gstart[h] + (k - s_off[h])]);
            continue;
          }
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
    }
    if (active) {
      fx[i] = ax;
      fy[i] = ay;
      fz[i] = az;
    }
  }
  const double te = block_sum<kForceThreads>(e, red);
  const double tw = block_sum<kForceThreads>(w, red);
  if (threadIdx.x == 0) {
    part_e[b] = te;
    part_w[b] = tw;
  }
}

// ---------------------------------------------------------------------------
// Parity/accounting tap: rewrite the brick-local list into the global-index
// ELL-transposed form (entry k of particle i at out[k*stride + i], same tag
// bits) consumed by the host-side pair dump and the in-cut counter.
__global__ void __launch_bounds__(128)
    k_decode_list(const int* __restrict__ cell_rank, const int* __restrict__ brick_rank_off,
                  const int* __restrict__ start, const int* __restrict__ group_off, Geom g,
                  BrickGeom bg, const uint32_t* __restrict__ list,
                  const int* __restrict__ nnbr, uint32_t* __restrict__ out, int stride) {
  __shared__ int s_gstart[kMaxHalo], s_cnt[kMaxHalo], s_off[kMaxHalo + 1], s_gcell[kMaxHalo];
  __shared__ uint32_t s_code[kMaxHalo];
  const int b = blockIdx.x;
  HaloTable ht;
  load_halo(b, g, bg, cell_rank, brick_rank_off, start, ht, s_gstart, s_cnt, s_off, s_code,
            s_gcell);
  const int nb_i = ht.be - ht.bs;
  for (int ib = threadIdx.x; ib < nb_i; ib += 128) {
    const int i = ht.bs + ib;
    const int grp = group_off[b] + (ib >> 5), gl = ib & 31;
    for (int k = 0; k < nnbr[i]; ++k) {
      const uint32_t ent = list[list_slot(grp, bg.cap, gl, k)];
      const int loc = static_cast<int>(ent & kIdxMask);
      const int h = halo_of(loc, s_off, ht.n);
      const uint32_t j = static_cast<uint32_t>(s_gstart[h] + (loc - s_off[h]));
      out[static_cast<size_t>(k) * stride + i] = j | (ent & ~kIdxMask);
    }
  }
}

}  // namespace tmd
