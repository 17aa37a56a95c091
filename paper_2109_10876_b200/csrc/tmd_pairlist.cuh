// PairIndexList on the device: the reference's classical Verlet list of
// explicit (i, j) slot pairs and its Newton-3 traversal (PairIndexList,
// build_pair_index_list, compute_pair_forces(const PairIndexList&, ...),
// neighbor_list.hpp:193-268) — the alternative traversal the reference keeps
// as the baseline of its traversal microbenchmark (bench_traversal.cpp,
// acceptance criterion 11). Included by tmd_engine.cu.
//
// Built from the current full list: every entry (i -> j) with slot j > i,
// i.e. each unordered pair (and periodic image) once, kept from the side
// whose list entry fixes the reference's rounding of d (the entry carries
// the image code and orientation), in particle-major list order.
//
// Traversal without floating-point atomics (deterministic):
//   1. one thread per pair: r2, the LJ force ff*d of the pair, stored per
//      pair (zero beyond r_cut); energy / virial per-block partial sums;
//   2. one thread per particle: + the pairs where it is i (its own range of
//      the pair array), - the pairs where it is j (a transposed index,
//      stably sorted by pair number), in that fixed order.
// Both ends get exactly opposite pair forces (Newton 3, like the
// reference's f_b -= ff*d).
#pragma once

#include <cub/device/device_radix_sort.cuh>

namespace tmd {

// Entries of i's list that point at a later slot (j > i).
__global__ void __launch_bounds__(kBlock)
    k_pl_count(int n, const uint32_t* __restrict__ nbr, const int* __restrict__ nnbr, int stride,
               int* __restrict__ cnt) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  const int m = nnbr[i];
  int c = 0;
  for (int k = 0; k < m; ++k) {
    const uint32_t ent = nbr[static_cast<size_t>(k) * stride + i];
    c += static_cast<int>(ent & kIdxMask) > i ? 1 : 0;
  }
  cnt[i] = c;
}

// pairs[off[i] + q] = {i, entry} for i's q-th entry with j > i (list order).
__global__ void __launch_bounds__(kBlock)
    k_pl_fill(int n, const uint32_t* __restrict__ nbr, const int* __restrict__ nnbr, int stride,
              const int* __restrict__ off, uint2* __restrict__ pairs,
              uint32_t* __restrict__ jkey) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  const int m = nnbr[i];
  int p = off[i];
  for (int k = 0; k < m; ++k) {
    const uint32_t ent = nbr[static_cast<size_t>(k) * stride + i];
    const uint32_t j = ent & kIdxMask;
    if (static_cast<int>(j) > i) {
      pairs[p] = make_uint2(static_cast<uint32_t>(i), ent);
      jkey[p] = j;
      ++p;
    }
  }
}

__global__ void k_pl_iota(int64_t m, uint32_t* __restrict__ v) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x;
  if (p < m) v[p] = static_cast<uint32_t>(p);
}

// Transposed index: the pair numbers where slot j is the second particle,
// from the stably sorted (j, pair) keys: row starts by binary search.
__global__ void __launch_bounds__(kBlock)
    k_pl_jstart(int n, int64_t m, const uint32_t* __restrict__ jsorted,
                long long* __restrict__ jstart) {
  const int j = blockIdx.x * kBlock + threadIdx.x;
  if (j > n) return;
  int64_t lo = 0, hi = m;  // first position with key >= j
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (static_cast<int>(jsorted[mid]) < j) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  jstart[j] = lo;
}

// 1. per pair: the pair force (compute_pair_forces' inner body,
// neighbor_list.hpp:253-266) and the energy / virial partials.
__global__ void __launch_bounds__(kBlock)
    k_pl_forces(int64_t m, const uint2* __restrict__ pairs, const double4* __restrict__ pos,
                Geom g, LjConst lj, double* __restrict__ fp, double* __restrict__ part_e,
                double* __restrict__ part_w, const long long* __restrict__ id, Ctrl* ctrl) {
  __shared__ double red[kBlock / 32];
  const int64_t p = blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x;
  double e = 0.0, w = 0.0;
  if (p < m) {
    const uint2 pr = pairs[p];
    const int i = static_cast<int>(pr.x);
    const double4 pi = pos[i];
    const double4 pj = pos[pr.y & kIdxMask];
    double dx, dy, dz;
    pair_delta(pi, pj, pr.y, g, dx, dy, dz);
    const double r2 = exact_r2(dx, dy, dz);
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (r2 < lj.rc2) {
      if (r2 == 0.0) record_error(ctrl, kStatOverlap, id[i], id[pr.y & kIdxMask]);
      const double ri2 = rcp_nr(r2);
      const double inv = lj.sigma2 * ri2;
      const double i6 = inv * inv * inv;
      const double ff = lj.eps24 * (2.0 * i6 * i6 - i6) * ri2;
      e = lj.eps4 * (i6 * i6 - i6) - lj.shift;
      w = ff * r2;
      fx = ff * dx;
      fy = ff * dy;
      fz = ff * dz;
    }
    fp[3 * p] = fx;
    fp[3 * p + 1] = fy;
    fp[3 * p + 2] = fz;
  }
  const double se = block_sum<kBlock>(e, red);
  const double sw = block_sum<kBlock>(w, red);
  if (threadIdx.x == 0) {
    part_e[blockIdx.x] = se;
    part_w[blockIdx.x] = sw;
  }
}

// 2. per particle: its pairs as i (+), then as j (-), fixed order.
__global__ void __launch_bounds__(kBlock)
    k_pl_gather(int n, const int* __restrict__ off, const long long* __restrict__ jstart,
                const uint32_t* __restrict__ jpairs, const double* __restrict__ fp,
                double* __restrict__ fx, double* __restrict__ fy, double* __restrict__ fz) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  double ax = 0.0, ay = 0.0, az = 0.0;
  for (int p = off[i]; p < off[i + 1]; ++p) {
    ax += fp[3 * static_cast<int64_t>(p)];
    ay += fp[3 * static_cast<int64_t>(p) + 1];
    az += fp[3 * static_cast<int64_t>(p) + 2];
  }
  for (long long q = jstart[i]; q < jstart[i + 1]; ++q) {
    const int64_t p = jpairs[q];
    ax -= fp[3 * p];
    ay -= fp[3 * p + 1];
    az -= fp[3 * p + 2];
  }
  fx[i] = ax;
  fy[i] = ay;
  fz[i] = az;
}

}  // namespace tmd
