// Kernels of the z-slab domain decomposition (multi-GPU): one
// context per GPU owns the particles of a slab of cell layers, plus one ghost
// layer on each side holding copies of the neighbour slabs' boundary layers.
// With a full neighbour list there is no reverse force exchange
// (collect_ghost_forces, decomp.hpp:202-224, disappears); per step only the
// boundary positions move, and at a rebuild the slab exchanges leavers
// (migration) and re-exports its boundary layers.
#pragma once

#include "tmd_kernels.cuh"

namespace tmd {

// One migrating particle (distribute_records moves whole records,
// domain.hpp:54-92; forces are recomputed before use, soa_store.hpp:19-21).
struct MigRec {
  long long id;
  double mass;
  double x, y, z;
  double vx, vy, vz;
};

// Wrap (exactly, box.hpp:47-51) and classify every owned particle by the rank
// owning its z cell layer; count leavers per destination.
__global__ void __launch_bounds__(kBlock)
    k_mig_classify(int n, double4* __restrict__ pos, const long long* __restrict__ id,
                   const int* __restrict__ owner_of_z, int my_rank, Geom g,
                   int* __restrict__ dest, int* __restrict__ dcount, Ctrl* ctrl) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  double4 p = pos[i];
  if (!finite3(p.x, p.y, p.z)) {
    record_error(ctrl, kStatNonFinitePos, id[i], -1);
    dest[i] = my_rank;
    return;
  }
  p.x = wrap1(p.x, g.L[0]);
  p.y = wrap1(p.y, g.L[1]);
  p.z = wrap1(p.z, g.L[2]);
  pos[i] = p;
  const int cz = cell_coord(p.z, g.cell_len[2], g.dims[2]);
  const int d = owner_of_z[cz];
  dest[i] = d;
  if (d != my_rank) atomicAdd(&dcount[d], 1);
}

// Stayers are compacted into the alternate arrays (order is irrelevant: the
// resort that follows sorts by cell and id); leavers are packed per
// destination at doff[dest] + cursor.
__global__ void __launch_bounds__(kBlock)
    k_mig_pack(int n, const double4* __restrict__ pos, const double* __restrict__ vx,
               const double* __restrict__ vy, const double* __restrict__ vz,
               const double* __restrict__ mass, const long long* __restrict__ id,
               const int* __restrict__ dest, int my_rank, const int* __restrict__ doff,
               int* __restrict__ dcur, MigRec* __restrict__ out, int* __restrict__ keep,
               double4* __restrict__ pos2, double* __restrict__ vx2, double* __restrict__ vy2,
               double* __restrict__ vz2, double* __restrict__ mass2,
               long long* __restrict__ id2) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  const int d = dest[i];
  if (d == my_rank) {
    const int k = atomicAdd(keep, 1);
    pos2[k] = pos[i];
    vx2[k] = vx[i];
    vy2[k] = vy[i];
    vz2[k] = vz[i];
    mass2[k] = mass[i];
    id2[k] = id[i];
  } else {
    const int k = doff[d] + atomicAdd(&dcur[d], 1);
    MigRec r;
    r.id = id[i];
    r.mass = mass[i];
    r.x = pos[i].x;
    r.y = pos[i].y;
    r.z = pos[i].z;
    r.vx = vx[i];
    r.vy = vy[i];
    r.vz = vz[i];
    out[k] = r;
  }
}

__global__ void __launch_bounds__(kBlock)
    k_mig_unpack(int nrecv, const MigRec* __restrict__ in, int base,
                 double4* __restrict__ pos, double* __restrict__ vx, double* __restrict__ vy,
                 double* __restrict__ vz, double* __restrict__ mass,
                 long long* __restrict__ id) {
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= nrecv) return;
  const MigRec r = in[k];
  const int i = base + k;
  pos[i] = make_double4(r.x, r.y, r.z, 0.0);
  vx[i] = r.vx;
  vy[i] = r.vy;
  vz[i] = r.vz;
  mass[i] = r.mass;
  id[i] = r.id;
}

// Per-cell particle counts of one owned boundary layer (local z = lz), cells
// in x-fastest order (the ghost-layer order of the receiving slab).
__global__ void __launch_bounds__(kBlock)
    k_layer_counts(int lz, Geom g, const int* __restrict__ cell_rank,
                   const int* __restrict__ start, int* __restrict__ counts) {
  const int q = blockIdx.x * kBlock + threadIdx.x;
  const int dxy = g.dims[0] * g.dims[1];
  if (q >= dxy) return;
  const int r = cell_rank[q + dxy * lz];
  counts[q] = start[r + 1] - start[r];
}

// Boundary-layer export: slot list (for the per-step position packing), ids
// and current positions, in (cell x-fastest, then sorted slot) order.
__global__ void __launch_bounds__(kBlock)
    k_layer_gather(int lz, Geom g, const int* __restrict__ cell_rank,
                   const int* __restrict__ start, const int* __restrict__ off,
                   const double4* __restrict__ pos, const long long* __restrict__ id,
                   int* __restrict__ idx_out, long long* __restrict__ id_out,
                   double4* __restrict__ pos_out) {
  const int q = blockIdx.x * kBlock + threadIdx.x;
  const int dxy = g.dims[0] * g.dims[1];
  if (q >= dxy) return;
  const int r = cell_rank[q + dxy * lz];
  const int b = start[r], e = start[r + 1];
  int o = off[q];
  for (int s = b; s < e; ++s, ++o) {
    idx_out[o] = s;
    id_out[o] = id[s];
    pos_out[o] = pos[s];
  }
}

// Ghost cell ranges from the two received count arrays: ghost layer 0 cells
// are ranked right after the owned cells, then ghost layer ldz-1 (setup_bricks).
__global__ void __launch_bounds__(1024)
    k_ghost_starts(Geom g, int n_own, const int* __restrict__ cnt_lo,
                   const int* __restrict__ cnt_hi, int* __restrict__ start) {
  __shared__ int warp_tot[32];
  const int dxy = g.dims[0] * g.dims[1];
  const int m = 2 * dxy;
  const int per = (m + 1023) / 1024;
  const int b = min(static_cast<int>(threadIdx.x) * per, m), e = min(b + per, m);
  int s = 0;
  for (int q = b; q < e; ++q) s += q < dxy ? cnt_lo[q] : cnt_hi[q - dxy];
  int total;
  int run = n_own + block_excl_scan(s, warp_tot, total);
  for (int q = b; q < e; ++q) {
    start[g.owned_cells + q] = run;
    run += q < dxy ? cnt_lo[q] : cnt_hi[q - dxy];
  }
  if (threadIdx.x == 1023) start[g.owned_cells + m] = n_own + total;
}

// Particles per global z layer (wrapped positions), for load-aware cut
// planes. Block-private shared-memory histogram, then one global add per
// layer per block.
__global__ void __launch_bounds__(kBlock)
    k_layer_hist(int n, const double4* __restrict__ pos, Geom g,
                 unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int s_hist[];
  const int dz = g.dims[2];
  for (int z = threadIdx.x; z < dz; z += kBlock) s_hist[z] = 0u;
  __syncthreads();
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    const double z = wrap1(pos[i].z, g.L[2]);
    atomicAdd(&s_hist[cell_coord(z, g.cell_len[2], dz)], 1u);
  }
  __syncthreads();
  for (int z = threadIdx.x; z < dz; z += kBlock) {
    if (s_hist[z]) atomicAdd(&hist[z], static_cast<unsigned long long>(s_hist[z]));
  }
}

// Export map of the fused halo: slot -> index in the side's export, -1 if
// the slot is not in that boundary layer (a one-layer slab has both).
__global__ void __launch_bounds__(kBlock)
    k_export_map(int nb, const int* __restrict__ idx, int side, int2* __restrict__ exp) {
  const int e = blockIdx.x * kBlock + threadIdx.x;
  if (e >= nb) return;
  int2* t = exp + idx[e];
  if (side == 0) {
    t->x = e;
  } else {
    t->y = e;
  }
}

__global__ void __launch_bounds__(kBlock) k_fill_int2(int n, int2* __restrict__ a, int2 v) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) a[i] = v;
}

// Per-step halo packing: current positions of one boundary layer.
__global__ void __launch_bounds__(kBlock)
    k_pack_border(int nb, const int* __restrict__ idx, const double4* __restrict__ pos,
                  double4* __restrict__ out, const Ctrl* ctrl) {
  if (ctrl->halt) return;
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k < nb) out[k] = pos[idx[k]];
}

// Native slab loop, speculative steps: the decision of a step from the
// globally reduced displacement word. No rebuild due: count the step and
// reset the word. Rebuild due: raise `halt` (the step's force and pack
// kernels and every later one of the batch return at once) and leave the
// step uncounted — the host runs the rebuild protocol, which counts it.
__global__ void k_decide_spec(Ctrl* ctrl, double thr) {
  if (ctrl->halt) return;
  const double m = __longlong_as_double(static_cast<long long>(ctrl->max_d2));
  ctrl->seen_d2 = m;
  if (m > thr) {
    ctrl->halt = 1;
    return;
  }
  ctrl->rebuild = 0;
  ctrl->max_d2 = 0ull;
  ctrl->step += 1;
}

// Native rebuild (tmd_slab_nccl.cuh): this rank's leaver offsets from the
// all-gathered count matrix M[s][d], on the device (no host staging).
__global__ void k_mig_offsets(const int* __restrict__ M, int r, int R, int* __restrict__ off) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int acc = 0;
  off[0] = 0;
  for (int d = 0; d < R; ++d) {
    acc += M[r * R + d];
    off[d + 1] = acc;
  }
}

// Native rebuild: this rank's all-gathered row {border sizes, owned count,
// slot capacity, buffer generation}.
__global__ void k_slab_row(int* __restrict__ row, const int* __restrict__ nb0,
                           const int* __restrict__ nb1, int n, int ncap, int gen) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  row[0] = *nb0;
  row[1] = *nb1;
  row[2] = n;
  row[3] = ncap;
  row[4] = gen;
}

// ---------------------------------------------------------------------------
// Bond table (CSR over id - id_min) built on the device at create
// (setup_bonds): degrees, an exclusive scan (CUB), then each bond appended to
// both ends and every particle's few entries put back in bond order — the
// order the host build keeps ("bond order kept at each end").
__global__ void __launch_bounds__(kBlock)
    k_bond_degree(int64_t nb, const long long* __restrict__ bonds, long long id_min,
                  int* __restrict__ deg) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
  if (k >= nb) return;
  atomicAdd(&deg[bonds[2 * k] - id_min], 1);
  atomicAdd(&deg[bonds[2 * k + 1] - id_min], 1);
}

// Smallest id offset holding more than kMaxBonds bonds (the host's error).
__global__ void __launch_bounds__(kBlock)
    k_bond_maxdeg(int span, const int* __restrict__ deg, int* __restrict__ bad) {
  const int o = blockIdx.x * kBlock + threadIdx.x;
  if (o < span && deg[o] > kMaxBonds) atomicMin(bad, o);
}

__global__ void __launch_bounds__(kBlock)
    k_bond_fill(int64_t nb, const long long* __restrict__ bonds, long long id_min,
                const int* __restrict__ off, int* __restrict__ cur, int* __restrict__ bidx,
                int* __restrict__ nbr, unsigned char* __restrict__ anchor) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
  if (k >= nb) return;
  const int a = static_cast<int>(bonds[2 * k] - id_min);
  const int b = static_cast<int>(bonds[2 * k + 1] - id_min);
  const int pa = off[a] + atomicAdd(&cur[a], 1);
  const int pb = off[b] + atomicAdd(&cur[b], 1);
  bidx[pa] = static_cast<int>(k);
  nbr[pa] = b;
  anchor[pa] = 1;
  bidx[pb] = static_cast<int>(k);
  nbr[pb] = a;
  anchor[pb] = 0;
}

// Each particle's entries by bond index (<= kMaxBonds of them; a bond to the
// same partner twice keeps its two entries apart by index).
__global__ void __launch_bounds__(kBlock)
    k_bond_order(int span, const int* __restrict__ off, int* __restrict__ bidx,
                 int* __restrict__ nbr, unsigned char* __restrict__ anchor) {
  const int o = blockIdx.x * kBlock + threadIdx.x;
  if (o >= span) return;
  const int b0 = off[o], m = off[o + 1] - b0;
  for (int x = 1; x < m; ++x) {
    const int kx = bidx[b0 + x], nx = nbr[b0 + x];
    const unsigned char ax = anchor[b0 + x];
    int y = x - 1;
    while (y >= 0 && bidx[b0 + y] > kx) {
      bidx[b0 + y + 1] = bidx[b0 + y];
      nbr[b0 + y + 1] = nbr[b0 + y];
      anchor[b0 + y + 1] = anchor[b0 + y];
      --y;
    }
    bidx[b0 + y + 1] = kx;
    nbr[b0 + y + 1] = nx;
    anchor[b0 + y + 1] = ax;
  }
}

}  // namespace tmd
