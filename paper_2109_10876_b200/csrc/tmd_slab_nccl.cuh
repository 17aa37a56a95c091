// Native multi-GPU step loop of the z-slab decomposition: the
// protocol of paper_2109_10876_b200/decomp.py, driven from C++ with its
// collectives on the context's stream, one host thread per slab. Included at
// the end of tmd_engine.cu (it drives the tmd_gpu_slab_* entry points and the
// context internals).
//
// Transport (`SlabComm`): every collective and point-to-point message of the
// loop goes through one small interface with two implementations:
//   * NcclComm — one process (or thread) per GPU, NCCL on the context stream;
//   * LocalComm — every rank's context in one process, one host thread per
//     rank: a collective is a host rendezvous of the rank threads that
//     exchanges stream events and device pointers, after which each rank's
//     stream waits on its peers' events and copies / reduces their buffers.
//     Stream-ordered like NCCL (nothing waits for the host), so the same C++
//     loop — fused peer-store halo, speculative batches, the rebuild
//     protocol — runs with R slabs on one GPU, and no kernel ever waits on
//     another rank's kernel (only on events of finished work).
//
// Per step (no rebuild): fused force + integrator kernel (whose epilogue
// stores boundary particles' new positions into the neighbours' ghost slots,
// or a pack + one group of point-to-point messages), an in-place MAX
// all-reduce of the displacement word, the on-device decision. The rebuild
// (every ~8 steps) runs the migration / border / ghost protocol with its few
// host round trips.
//
// Message order. Point-to-point operations of a group between a pair of
// ranks match in posting order (NCCL's rule; LocalComm checks it and the
// sizes), so both ends post, per peer: the message for the receiver's LOWER
// ghost layer first (the sender's highest layer), then the one for its UPPER
// ghost layer (the sender's lowest layer), each as counts, ids, positions.
// With one or two slabs the lower and upper neighbour are the same rank and
// the order still agrees.
#pragma once

#include <unistd.h>

#include <optional>

#include "tmd_comm.cuh"

namespace {

SlabComm* comm(const tmd_gpu_ctx* c) { return static_cast<SlabComm*>(c->comm); }

// Contiguous cut planes over the z layers minimising the largest slab
// population, every slab >= 1 layer (decomp.py balanced_cuts: binary search
// on the bound + greedy fill, then the widest slabs halved).
std::vector<int> balanced_cuts(const std::vector<int64_t>& cnt, int R) {
  const int dz = static_cast<int>(cnt.size());
  auto greedy = [&](int64_t bound) {
    std::vector<int> starts{0};
    int64_t acc = 0;
    for (int z = 0; z < dz; ++z) {
      if (z > starts.back() && acc + cnt[static_cast<size_t>(z)] > bound) {
        starts.push_back(z);
        acc = 0;
      }
      acc += cnt[static_cast<size_t>(z)];
    }
    return starts;
  };
  int64_t lo = *std::max_element(cnt.begin(), cnt.end()), hi = lo;
  for (int64_t v : cnt) hi += v;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (static_cast<int>(greedy(mid).size()) <= R) {
      hi = mid;
    } else {
      lo = mid + 1;
    }
  }
  std::vector<int> starts = greedy(lo);
  while (static_cast<int>(starts.size()) < R) {
    int wi = 0, wmax = -1;
    for (size_t i = 0; i < starts.size(); ++i) {
      const int e = i + 1 < starts.size() ? starts[i + 1] : dz;
      if (e - starts[i] > wmax) {
        wmax = e - starts[i];
        wi = static_cast<int>(i);
      }
    }
    starts.insert(starts.begin() + wi + 1, starts[static_cast<size_t>(wi)] + wmax / 2);
  }
  starts.push_back(dz);
  return starts;
}

int64_t max_load(const std::vector<int64_t>& cnt, const std::vector<int>& cuts) {
  int64_t m = 0;
  for (size_t r = 0; r + 1 < cuts.size(); ++r) {
    int64_t s = 0;
    for (int z = cuts[r]; z < cuts[r + 1]; ++z) s += cnt[static_cast<size_t>(z)];
    m = std::max(m, s);
  }
  return m;
}


void rck(tmd_gpu_ctx* c, int rc) {  // a tmd_gpu_slab_* call inside the native loop
  if (rc != TMD_OK) throw StatusError{rc, c->err};
}

// Both boundary layers to the neighbours' ghost layers (or, with
// positions_only, just the positions of an unchanged layout).
void nccl_ghost_exchange(tmd_gpu_ctx* c, bool positions_only) {
  const int R = c->nranks, r = c->my_rank;
  const int lo = (r - 1 + R) % R, hi = (r + 1) % R;
  const size_t dxy = static_cast<size_t>(c->g.dims[0]) * c->g.dims[1];
  double4* pos = c->pos;
  // my ghost destinations: lower ghost from lo (its side 1), upper from hi (its side 0)
  int* gl_cnt = c->gcnt[0];
  int* gh_cnt = c->gcnt[1];
  long long* gl_id = c->id + c->n;
  long long* gh_id = c->id + c->n + c->n_ghost_lo;
  double4* gl_pos = pos + c->n;
  double4* gh_pos = pos + c->n + c->n_ghost_lo;
  SlabComm* cm = comm(c);
  auto send3 = [&](int side, int peer) {
    if (!positions_only) {
      cm->send(c->bcnt[side], dxy * sizeof(int), peer, c->stream);
      if (c->nb[side]) cm->send(c->bids[side], c->nb[side] * sizeof(long long), peer, c->stream);
    }
    if (c->nb[side]) cm->send(c->bpos[side], c->nb[side] * sizeof(double4), peer, c->stream);
  };
  auto recv3 = [&](int* cnt, long long* ids, double4* p, int64_t n, int peer) {
    if (!positions_only) {
      cm->recv(cnt, dxy * sizeof(int), peer, c->stream);
      if (n) cm->recv(ids, n * sizeof(long long), peer, c->stream);
    }
    if (n) cm->recv(p, n * sizeof(double4), peer, c->stream);
  };
  cm->group_start();
  // to hi: its lower ghost (my side 1); to lo: its upper ghost (my side 0) —
  // when hi == lo the lower-ghost message goes first, as the receiver expects
  send3(1, hi);
  send3(0, lo);
  // from lo: my lower ghost; from hi: my upper ghost (lower first per peer)
  recv3(gl_cnt, gl_id, gl_pos, c->n_ghost_lo, lo);
  recv3(gh_cnt, gh_id, gh_pos, c->n_ghost_hi, hi);
  cm->group_end(c->stream);
}

// Load-aware cut planes (row f3) before a migration: per-layer counts summed
// over ranks, re-cut when the current largest slab exceeds the optimum by
// more than 5 %.
void nccl_rebalance(tmd_gpu_ctx* c) {
  const int dz = c->g.dims[2], R = c->nranks;
  std::vector<int64_t> cnt(static_cast<size_t>(dz));
  rck(c, tmd_gpu_slab_layer_counts(c, cnt.data()));
  int64_t* d = dalloc<int64_t>(static_cast<size_t>(dz));
  ck(cudaMemcpyAsync(d, cnt.data(), sizeof(int64_t) * dz, cudaMemcpyHostToDevice, c->stream),
     "H2D layer counts");
  comm(c)->allreduce(d, static_cast<size_t>(dz), CType::kI64, COp::kSum, c->stream);
  ck(cudaMemcpyAsync(cnt.data(), d, sizeof(int64_t) * dz, cudaMemcpyDeviceToHost, c->stream),
     "D2H layer counts");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  cudaFree(d);
  const std::vector<int> best = balanced_cuts(cnt, R);
  if (static_cast<double>(max_load(cnt, c->cuts)) > 1.05 * static_cast<double>(max_load(cnt, best))) {
    rck(c, tmd_gpu_slab_recut(c, best.data()));
    c->cuts = best;
    c->recuts += 1;
  }
}

// Fused halo: every rank publishes where its ghost layers live (CUDA IPC
// handles of both position buffers + the ghost offsets of the current
// layout); each rank maps its neighbours' buffers (peer memory over NVLink,
// its own buffers when the neighbour is itself) so that the force kernel's
// epilogue stores boundary particles' new positions straight into the
// neighbours' ghost slots. The per-step MAX all-reduce that precedes every
// force kernel orders those stores against the neighbours' reads (a rank's
// next force kernel starts only after every rank's previous one finished).
struct PeerInfo {
  cudaIpcMemHandle_t h[2];
  unsigned long long base[2];
  long long pid;
  long long ghost_lo_off, ghost_hi_off;
  long long gen;  // the rank's ipc_gen (buffer reallocations so far)
  long long device;
};

double4* peer_buffer(tmd_gpu_ctx* c, const PeerInfo& p, int peer, int b) {
  if (peer == c->my_rank) return c->posb[b];
  if (p.pid == static_cast<long long>(getpid())) {  // in-process group: plain pointers
    if (p.device != c->device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(static_cast<int>(p.device), 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else {
        ck(e, "cudaDeviceEnablePeerAccess");
      }
    }
    return reinterpret_cast<double4*>(p.base[b]);
  }
  std::array<char, 64> key;
  std::memcpy(key.data(), &p.h[b], 64);
  for (const auto& e : c->ipc_open) {
    if (e.first == key) return static_cast<double4*>(e.second);
  }
  void* ptr = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&ptr, p.h[b], cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaFail{std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e) + " (rank " +
                   std::to_string(c->my_rank) + " pid " + std::to_string(getpid()) +
                   ", peer " + std::to_string(peer) + " pid " + std::to_string(p.pid) +
                   " device " + std::to_string(p.device) + " buffer " + std::to_string(b) +
                   " base " + std::to_string(p.base[b]) + ", " +
                   std::to_string(c->ipc_open.size()) + " mappings open)"};
  }
  c->ipc_open.emplace_back(key, ptr);
  return static_cast<double4*>(ptr);
}

// A rank that cannot export or map a position buffer (no peer access between
// two GPUs, IPC disabled in a container, ...) must not leave the others in a
// collective: every rank finishes the exchange, the failures are MAX-reduced,
// and if any rank failed all of them drop to the message halo (pack + one
// point-to-point group per step) for the rest of the run — same trajectories,
// no peer stores. TMD_HALO_STRICT=1 turns the fallback into the error (the
// tests set it, so a silently degraded path cannot pass them);
// TMD_HALO_FAIL_INJECT=<rank> makes that rank's mapping fail (test hook).
bool env_is(const char* name, const char* v) {
  const char* e = std::getenv(name);
  return e && std::strcmp(e, v) == 0;
}

void nccl_publish_ghosts(tmd_gpu_ctx* c) {
  const int R = c->nranks, r = c->my_rank;
  PeerInfo me{};
  std::string fail_why;
  for (int b = 0; b < 2; ++b) {
    const cudaError_t e = cudaIpcGetMemHandle(&me.h[b], c->posb[b]);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail_why = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
    }
    me.base[b] = reinterpret_cast<unsigned long long>(c->posb[b]);
  }
  me.pid = static_cast<long long>(getpid());
  me.ghost_lo_off = c->n;
  me.ghost_hi_off = c->n + c->n_ghost_lo;
  me.gen = c->ipc_gen;
  me.device = c->device;
  static_assert(sizeof(PeerInfo) % 8 == 0, "the failure word follows the table, 8-aligned");
  const size_t sz = sizeof(PeerInfo);
  char* d = dalloc<char>(sz * (static_cast<size_t>(R) + 1) + sizeof(int64_t));
  int64_t* d_fail = reinterpret_cast<int64_t*>(d + sz * (static_cast<size_t>(R) + 1));
  ck(cudaMemcpyAsync(d, &me, sz, cudaMemcpyHostToDevice, c->stream), "H2D peer info");
  comm(c)->allgather(d, d + sz, sz, c->stream);
  std::vector<PeerInfo> all(static_cast<size_t>(R));
  ck(cudaMemcpyAsync(all.data(), d + sz, sz * R, cudaMemcpyDeviceToHost, c->stream),
     "D2H peer info");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  // some rank's buffers moved (the only reason for a new exchange): close
  // every mapping and open what the new layout needs — a reallocated buffer
  // may even come back under the old handle's bytes, so none is reused
  for (auto& e : c->ipc_open) cudaIpcCloseMemHandle(e.second);
  c->ipc_open.clear();
  const int lo = (r - 1 + R) % R, hi = (r + 1) % R;
  if (fail_why.empty()) {
    try {
      if (R > 1 && env_is("TMD_HALO_FAIL_INJECT", std::to_string(r).c_str())) {
        throw CudaFail{"mapping failure injected (TMD_HALO_FAIL_INJECT)"};
      }
      for (int b = 0; b < 2; ++b) {
        // my lowest layer -> lo's upper ghost; my highest layer -> hi's lower ghost
        c->peer_base[0][b] = peer_buffer(c, all[static_cast<size_t>(lo)], lo, b);
        c->peer_base[1][b] = peer_buffer(c, all[static_cast<size_t>(hi)], hi, b);
        c->rg[0][b] = c->peer_base[0][b] + all[static_cast<size_t>(lo)].ghost_hi_off;
        c->rg[1][b] = c->peer_base[1][b] + all[static_cast<size_t>(hi)].ghost_lo_off;
      }
    } catch (const CudaFail& f) {
      fail_why = f.what;
    }
  }
  // agree on the outcome: any failure anywhere turns the fused halo off everywhere
  const int64_t mine = fail_why.empty() ? 0 : 1;
  int64_t any = 0;
  ck(cudaMemcpyAsync(d_fail, &mine, sizeof mine, cudaMemcpyHostToDevice, c->stream), "H2D flag");
  comm(c)->allreduce(d_fail, 1, CType::kI64, COp::kMax, c->stream);
  ck(cudaMemcpyAsync(&any, d_fail, sizeof any, cudaMemcpyDeviceToHost, c->stream), "D2H flag");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  cudaFree(d);
  if (any) {
    for (auto& e : c->ipc_open) cudaIpcCloseMemHandle(e.second);
    c->ipc_open.clear();
    c->peer_gen.clear();
    if (env_is("TMD_HALO_STRICT", "1")) {
      throw CudaFail{"fused halo unavailable" +
                     (mine ? ": " + fail_why : std::string(" (a peer rank could not map a buffer)"))};
    }
    if (mine || r == 0) {
      std::fprintf(stderr,
                   "[tmd_gpu] rank %d: fused peer-store halo unavailable%s%s; every rank uses the "
                   "message halo (pack + point-to-point) from here on\n",
                   r, mine ? ": " : "", mine ? fail_why.c_str() : "");
    }
    c->fused_halo = false;
    c->fused_ready = false;
    return;
  }
  c->peer_gen.assign(static_cast<size_t>(R), 0);
  for (int q = 0; q < R; ++q) c->peer_gen[static_cast<size_t>(q)] = static_cast<int>(all[static_cast<size_t>(q)].gen);
  c->fused_ready = true;
}

// The rebuild protocol (decomp.py DecomposedEngine._rebuild) over NCCL, with
// three host round trips: (1) the leaver counts, all-gathered straight from
// the device; (2) after the on-device commit, one all-gathered row per rank
// {border sizes, owned count, slot capacity, buffer generation}, from which
// every rank derives every other rank's ghost counts and ghost offsets;
// (3) the list build's overflow check. The fused halo's peer addresses are
// re-exchanged (IPC handles, a fourth round trip) only when some rank's
// position buffers were or are about to be reallocated; otherwise they are
// the cached peer bases plus the derived ghost offsets.
constexpr int kRowInts = 5;  // nb0, nb1, n_own, n_cap, ipc_gen
void nccl_rebuild(tmd_gpu_ctx* c, bool advance) {
  const int R = c->nranks, r = c->my_rank;
  const size_t uR = static_cast<size_t>(R);
  std::optional<Phase> ph;
  ph.emplace(c, TMD_SECTION_RESORT);
  rck(c, tmd_gpu_slab_decide(c, 1, advance ? 1 : 0));
  if (c->balance_count) nccl_rebalance(c);
  // 1. classify; the leaver-count matrix M[s][d] all-gathered from the device
  const int n = static_cast<int>(c->n);
  ck(cudaMemsetAsync(c->mig_count, 0, 2 * sizeof(int) * uR, c->stream), "memset");
  ck(cudaMemsetAsync(c->mig_keep, 0, sizeof(int), c->stream), "memset");
  c->launches += 1;
  if (n > 0) {
    k_mig_classify<<<c->nblk, kBlock, 0, c->ls>>>(n, c->pos, c->id, c->owner_of_z, c->my_rank,
                                                  c->g, c->mig_dest, c->mig_count, c->ctrl);
  }
  int* Md = reinterpret_cast<int*>(c->nccl_i64);  // R*R ints (the buffer holds 2R^2 + 2R + 16)
  comm(c)->allgather(c->mig_count, Md, uR * sizeof(int), c->stream);
  std::vector<int> M(uR * uR);
  ck(cudaMemcpyAsync(M.data(), Md, sizeof(int) * uR * uR, cudaMemcpyDeviceToHost, c->stream),
     "D2H counts");
  sync_ctrl(c);
  raise_physics(c, true);
  // 2. stayers compacted, leavers packed by destination, records point to point
  std::vector<int> off(uR + 1, 0);
  for (int d = 0; d < R; ++d) off[static_cast<size_t>(d) + 1] = off[static_cast<size_t>(d)] + M[static_cast<size_t>(r) * uR + d];
  c->launches += 1;
  k_mig_offsets<<<1, 1, 0, c->ls>>>(Md, r, R, c->mig_off);
  const bool leavers = off[uR] > 0;  // none: the stayers are already in place
  if (n > 0 && leavers) {
    c->launches += 1;
    k_mig_pack<<<c->nblk, kBlock, 0, c->ls>>>(
        n, c->pos, c->vx, c->vy, c->vz, c->mass, c->id, c->mig_dest, c->my_rank, c->mig_off,
        c->mig_count + R, c->mig_send, c->mig_keep, c->pos2, c->vx2, c->vy2, c->vz2, c->mass2,
        c->id2);
  }
  const size_t keep = static_cast<size_t>(n - off[uR]);
  if (keep > 0 && leavers) {  // stayers back in place: one launch (no cell column:
                              // the resort that follows recomputes it)
    c->launches += 1;
    k_copy_back<<<blocks_for(static_cast<int64_t>(keep), kBlock), kBlock, 0, c->ls>>>(
        static_cast<int>(keep), c->pos2, c->vx2, c->vy2, c->vz2, c->mass2, c->id2, nullptr,
        c->pos, c->vx, c->vy, c->vz, c->mass, c->id, nullptr, nullptr);
  }
  c->n = static_cast<int64_t>(keep);
  c->n_ghost = c->n_ghost_lo = c->n_ghost_hi = 0;
  int64_t nrecv = 0;
  for (int q = 0; q < R; ++q) nrecv += M[static_cast<size_t>(q) * uR + r];
  grow_capacity(c, c->n + nrecv);  // (synchronises and bumps ipc_gen only when it grows)
  c->mig_nrecv = nrecv;
  const size_t rec = sizeof(MigRec);
  SlabComm* cm = comm(c);
  ph.emplace(c, TMD_SECTION_COMM);
  cm->group_start();
  for (int d = 0; d < R; ++d) {
    const int m = M[static_cast<size_t>(r) * uR + d];
    if (m) {
      cm->send(reinterpret_cast<char*>(c->mig_send) + static_cast<size_t>(off[static_cast<size_t>(d)]) * rec,
               static_cast<size_t>(m) * rec, d, c->stream);
    }
  }
  int64_t roff = 0;
  for (int q = 0; q < R; ++q) {
    const int m = M[static_cast<size_t>(q) * uR + r];
    if (m) {
      cm->recv(reinterpret_cast<char*>(c->mig_recv) + roff * rec, static_cast<size_t>(m) * rec, q,
               c->stream);
    }
    roff += m;
  }
  cm->group_end(c->stream);
  // 3. commit on the device; one row per rank all-gathered
  ph.emplace(c, TMD_SECTION_RESORT);
  slab_commit_launch(c);
  const int dxy = c->g.dims[0] * c->g.dims[1];
  int* row = Md;                 // this rank's row
  int* table = Md + 8;           // R rows
  c->launches += 1;
  k_slab_row<<<1, 1, 0, c->ls>>>(row, c->boff[0] + dxy, c->boff[1] + dxy, static_cast<int>(c->n),
                                 static_cast<int>(c->n_cap), c->ipc_gen);
  cm->allgather(row, table, kRowInts * sizeof(int), c->stream);
  std::vector<int> T(uR * kRowInts);
  ck(cudaMemcpyAsync(T.data(), table, sizeof(int) * T.size(), cudaMemcpyDeviceToHost, c->stream),
     "D2H rows");
  sync_ctrl(c);
  raise_physics(c, true);
  if (c->h_ctrl->status & kStatStray) throw CudaFail{"slab: particle outside its slab"};
  auto at = [&](int q, int k) { return T[static_cast<size_t>((q + R) % R) * kRowInts + k]; };
  slab_commit_finish(c, at(r, 0), at(r, 1));
  // 4. ghost layers (counts, ids, positions) from the neighbours, then the list
  const int lo = (r - 1 + R) % R, hi = (r + 1) % R;
  void* gl[3];
  void* gh[3];
  rck(c, tmd_gpu_slab_ghost_in(c, at(lo, 1), at(hi, 0), gl, gh));
  ph.emplace(c, TMD_SECTION_COMM);
  nccl_ghost_exchange(c, false);
  ph.emplace(c, TMD_SECTION_NEIGH);
  rck(c, tmd_gpu_slab_ghosts_ready(c));
  if (!c->fused_halo) return;
  ph.emplace(c, TMD_SECTION_COMM);
  // 5. peer addresses of the fused halo: q's lower ghost layer starts at its
  // owned count, its upper one after the lower (= its lower neighbour's top
  // border)
  bool remap = c->peer_gen.size() != uR;
  for (int q = 0; q < R && !remap; ++q) {
    const int64_t need = static_cast<int64_t>(at(q, 2)) + at(q - 1, 1) + at(q + 1, 0);
    remap = need > at(q, 3) || at(q, 4) != c->peer_gen[static_cast<size_t>(q)];
  }
  if (remap) {
    nccl_publish_ghosts(c);
    return;
  }
  for (int b = 0; b < 2; ++b) {
    c->rg[0][b] = c->peer_base[0][b] + (static_cast<int64_t>(at(lo, 2)) + at(lo - 1, 1));
    c->rg[1][b] = c->peer_base[1][b] + at(hi, 2);
  }
  c->fused_ready = true;
}
bool fused(const tmd_gpu_ctx* c) { return c->fused_halo && c->fused_ready; }

void nccl_halo(tmd_gpu_ctx* c) {
  for (int s = 0; s < 2; ++s) {
    if (c->nb[s] == 0) continue;
    c->launches += 1;
    k_pack_border<<<blocks_for(c->nb[s], kBlock), kBlock, 0, c->ls>>>(
        static_cast<int>(c->nb[s]), c->bidx[s], c->pos, c->bpos[s], c->ctrl);
  }
  nccl_ghost_exchange(c, true);
}

constexpr int kSpecSteps = 16;  // steps enqueued per host round trip (at most)
// Steps of the next speculative batch, aimed to end at the step whose
// decision triggers the next rebuild (the batch's later steps would be
// no-ops, each still paying its all-reduce). Right after a rebuild: the last
// interval between rebuilds; later: the global displacement the last decision
// saw, extrapolated ballistically (|x - x_snap| ~ t). Every rank computes the
// same value from all-reduced inputs, so the collectives stay matched.
int64_t spec_batch(const tmd_gpu_ctx* c, int64_t done_step) {
  if (c->last_rebuild_step < 0) return kSpecSteps;
  const int64_t t = done_step - c->last_rebuild_step;  // drifts since the list build
  const double m = c->h_ctrl->seen_d2, thr = c->g.rebuild_thr;
  double k;
  if (t <= 0 || !(m > 0.0)) {  // just rebuilt: expect the last interval again
    k = c->rebuild_gap > 0 ? static_cast<double>(c->rebuild_gap) : kSpecSteps;
  } else {  // the decision of step done_step saw m after t drifts
    k = std::ceil(static_cast<double>(t) * std::sqrt(thr / m)) - static_cast<double>(t);
  }
  return std::max<int64_t>(1, std::min<int64_t>(kSpecSteps, static_cast<int64_t>(k)));
}

void need_comm(const tmd_gpu_ctx* c) {
  if (!c->comm) throw StatusError{TMD_ERR_STATE, "slab context has no transport (attach one first)"};
}

// A failure on one rank of an in-process group releases the others from the
// collective they wait in (they fail with "a peer rank failed").
template <class F>
int native_guard(tmd_gpu_ctx* c, F&& fn) {
  return guard(c, [&] {
    try {
      fn();
    } catch (...) {
      if (c->comm) comm(c)->abort();
      throw;
    }
  });
}

}  // namespace

extern "C" {

int tmd_balanced_cuts(const int64_t* counts, int dims_z, int nranks, int32_t* cuts) {
  if (!counts || !cuts || nranks < 1 || dims_z < nranks) return TMD_ERR_CONFIG;
  const std::vector<int64_t> cnt(counts, counts + dims_z);
  const std::vector<int> best = balanced_cuts(cnt, nranks);
  for (int r = 0; r <= nranks; ++r) cuts[r] = best[static_cast<size_t>(r)];
  return TMD_OK;
}

int tmd_nccl_unique_id(void* id) {
#ifdef TMD_NO_NCCL
  (void)id;
  g_create_error = "this build of libtmd_gpu.so has no NCCL";
  return TMD_ERR_CONFIG;
#else
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) {
    g_create_error = "ncclGetUniqueId failed";
    return TMD_ERR_CUDA;
  }
  std::memcpy(id, &u, sizeof u);
  return TMD_OK;
#endif
}

namespace {
void attach_common(tmd_gpu_ctx* c, int flags) {
  need_slab(c);
  if (c->comm) throw StatusError{TMD_ERR_STATE, "slab context already has a transport"};
  c->balance_count = (flags & 1) != 0;
  c->fused_halo = (flags & 2) != 0;
  ck(cudaSetDevice(c->device), "cudaSetDevice");
}
void alloc_comm_staging(tmd_gpu_ctx* c) {
  c->nccl_i64 = dalloc<int64_t>(static_cast<size_t>(c->nranks) * (c->nranks + 1) + 8);
}
}  // namespace

int tmd_gpu_slab_attach_nccl(tmd_gpu_ctx* c, const void* unique_id, int flags) {
  return guard(c, [&] {
    attach_common(c, flags);
#ifdef TMD_NO_NCCL
    (void)unique_id;
    throw StatusError{TMD_ERR_CONFIG, "this build of libtmd_gpu.so has no NCCL"};
#else
    ncclUniqueId u;
    std::memcpy(&u, unique_id, sizeof u);
    auto nc = std::make_unique<NcclComm>();
    nc->device = c->device;
    nc->nranks = c->nranks;
    nc->rank = c->my_rank;
    nc->nc = nccl_cache_take(c->device, c->nranks, c->my_rank);
    if (!nc->nc) nck(ncclCommInitRank(&nc->nc, c->nranks, u, c->my_rank), "ncclCommInitRank");
    alloc_comm_staging(c);
    c->comm = nc.release();
#endif
  });
}

int tmd_local_group_create(int nranks, void** group) {
  if (!group || nranks < 1) {
    g_create_error = "local group: nranks >= 1 and an output pointer required";
    return TMD_ERR_CONFIG;
  }
  *group = new std::shared_ptr<LocalGroup>(std::make_shared<LocalGroup>(nranks));
  return TMD_OK;
}

void tmd_local_group_destroy(void* group) {
  delete static_cast<std::shared_ptr<LocalGroup>*>(group);
}

int tmd_gpu_slab_attach_local(tmd_gpu_ctx* c, void* group, int flags) {
  return guard(c, [&] {
    if (!group) throw StatusError{TMD_ERR_CONFIG, "local group missing"};
    const auto& g = *static_cast<std::shared_ptr<LocalGroup>*>(group);
    if (g->R != c->nranks) {
      throw StatusError{TMD_ERR_CONFIG, "local group of " + std::to_string(g->R) +
                                            " ranks for a slab of " + std::to_string(c->nranks)};
    }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      if (g->taken[static_cast<size_t>(c->my_rank)]) {
        throw StatusError{TMD_ERR_CONFIG, "rank " + std::to_string(c->my_rank) +
                                              " of the local group is already attached"};
      }
      g->taken[static_cast<size_t>(c->my_rank)] = 1;
    }
    try {
      attach_common(c, flags);
      auto lc = std::make_unique<LocalComm>(g, c->my_rank);
      alloc_comm_staging(c);
      c->comm = lc.release();
    } catch (...) {
      std::lock_guard<std::mutex> lk(g->mu);
      g->taken[static_cast<size_t>(c->my_rank)] = 0;
      throw;
    }
  });
}

int tmd_gpu_slab_attach_host(tmd_gpu_ctx* c, const char* path, int flags) {
  return guard(c, [&] {
    if (!path || !*path) throw StatusError{TMD_ERR_CONFIG, "host transport: a file path"};
    attach_common(c, flags);
    auto hc = std::make_unique<HostFileComm>(path, c->my_rank, c->nranks);
    alloc_comm_staging(c);
    c->comm = hc.release();
  });
}

int tmd_gpu_slab_setup(tmd_gpu_ctx* c) {
  return native_guard(c, [&] {
    need_slab(c);
    need_comm(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    nccl_rebuild(c, false);
    c->last_rebuild_step = c->step;
    rck(c, tmd_gpu_slab_forces(c, 0));
    sync_ctrl(c);
    raise_physics(c, false);
  });
}

// Speculative batches: up to kSpecSteps steps are enqueued without a host
// round trip, each as MAX all-reduce of the displacement word -> on-device
// decision (k_decide_spec) -> fused force/integrator kernel -> pack -> halo.
// When a step needs a rebuild its decision raises `halt`: that step's and the
// rest of the batch's kernels return at once (the halo messages still run and
// re-deliver unchanged positions), and after the batch's single sync the host
// runs the rebuild protocol and that step's forces, then continues. Every
// rank takes the same decisions (the word is all-reduced), so all halt at the
// same step.
namespace {

// Rows the device recorded since the last collection (run_observed), then
// the device counter is reset on the stream. Call right after a sync_ctrl.
void collect_slab_obs(tmd_gpu_ctx* c) {
  if (c->obs_stride <= 0) return;
  const int rows = std::min(c->h_ctrl->obs_rows, kObsRows);
  for (int r = 0; r < rows; ++r) {
    const double* o = c->obs_host + 4 * r;
    c->obs_rows.push_back({o[0], o[1], o[2], o[3]});
  }
  ck(cudaMemsetAsync(&c->ctrl->obs_rows, 0, sizeof(int), c->stream), "memset obs rows");
}

void slab_run_impl(tmd_gpu_ctx* c, int64_t nsteps) {
    need_slab(c);
    need_comm(c);
    if (nsteps < 0) throw StatusError{TMD_ERR_CONFIG, "step count must be non-negative"};
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (nsteps == 0) return;
    if (c->obs_stride > 0) {
      ck(cudaMemsetAsync(&c->ctrl->obs_rows, 0, sizeof(int), c->stream), "memset obs rows");
    }
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    const int64_t start = c->step, target = c->step + nsteps;
    {
      Phase p(c, TMD_SECTION_INTEGRATE);
      if (c->n > 0) launch_kick_drift(c);
    }
    {
      Phase p(c, TMD_SECTION_COMM);
      nccl_halo(c);
    }
    int64_t done_step = start;  // steps completed (host view)
    int64_t K_next = kSpecSteps;
    while (done_step < target) {
      const int64_t K = std::min<int64_t>(K_next, target - done_step);
      int64_t fused_launches = 0;
      for (int64_t s = 0; s < K; ++s) {
        {
          Phase p(c, TMD_SECTION_COMM);  // the global rebuild test's all-reduce
          comm(c)->allreduce(&c->ctrl->max_d2, 1, CType::kU64, COp::kMax, c->stream);
        }
        {
          Phase p(c, TMD_SECTION_NEIGH);
          c->launches += 1;
          k_decide_spec<<<1, 1, 0, c->ls>>>(c->ctrl, c->g.rebuild_thr);
        }
        const bool last = done_step + s + 1 == target;
        const bool fh = fused(c);  // the force epilogue delivers the halo itself
        {
          Phase p(c, TMD_SECTION_FORCES);
          launch_forces(c, last ? kKick2 : kFused);
          launch_obs_record(c);
        }
        if (!last) {
          ++fused_launches;
          if (!fh) {
            Phase p(c, TMD_SECTION_COMM);
            nccl_halo(c);
          }
        }
      }
      sync_ctrl(c);
      harvest_timers(c);
      raise_physics(c, true);
      collect_slab_obs(c);
      if (c->h_ctrl->status & kStatStray) throw CudaFail{"slab: particle outside its slab"};
      const int64_t advanced = c->h_ctrl->step - done_step;  // steps that ran
      if (!c->h_ctrl->halt) {
        done_step += K;
        K_next = spec_batch(c, done_step);
        continue;
      }
      // the launches from the halted step on were no-ops: undo their buffer
      // flips on the host (the device never swapped)
      const int64_t noop_fused = fused_launches - advanced;
      if (noop_fused & 1) {
        c->cur ^= 1;
        c->pos = c->posb[c->cur];
      }
      done_step += advanced;
      const int zero = 0;
      ck(cudaMemcpyAsync(&c->ctrl->halt, &zero, sizeof(int), cudaMemcpyHostToDevice, c->stream),
         "clear halt");
      nccl_rebuild(c, true);  // counts the step and the rebuild
      const bool last = done_step + 1 == target;
      const bool fh = fused(c);
      {
        Phase p(c, TMD_SECTION_FORCES);
        launch_forces(c, last ? kKick2 : kFused);
        launch_obs_record(c);
      }
      if (!last && !fh) {
        Phase p(c, TMD_SECTION_COMM);
        nccl_halo(c);
      }
      done_step += 1;
      if (c->last_rebuild_step >= 0) c->rebuild_gap = done_step - c->last_rebuild_step;
      c->last_rebuild_step = done_step;
      K_next = spec_batch(c, done_step);
    }
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    sync_ctrl(c);
    harvest_timers(c);
    raise_physics(c, true);
    collect_slab_obs(c);
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->t0, c->t1), "cudaEventElapsedTime");
    c->elapsed += 1e-3 * ms;
    c->step = c->h_ctrl->step;
    c->rebuilds = static_cast<uint64_t>(c->h_ctrl->rebuilds);
}

}  // namespace

int tmd_gpu_slab_run(tmd_gpu_ctx* c, int64_t nsteps) {
  return native_guard(c, [&] { slab_run_impl(c, nsteps); });
}

int tmd_gpu_slab_run_observed(tmd_gpu_ctx* c, int64_t nsteps, int64_t stride,
                              tmd_observables* out, int64_t cap, int64_t* n_out) {
  return native_guard(c, [&] {
    if (stride < 1) throw StatusError{TMD_ERR_CONFIG, "observable stride must be at least 1"};
    if (!n_out || (cap > 0 && !out)) throw StatusError{TMD_ERR_CONFIG, "row buffer missing"};
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (!c->obs_host) {
      c->obs_host = static_cast<double*>(pinned_small(sizeof(double) * 4 * kObsRows));
      ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->obs_dev), c->obs_host, 0),
         "cudaHostGetDevicePointer");
    }
    const int64_t s0 = c->step;
    c->obs_rows.clear();
    c->obs_stride = static_cast<int>(std::min<int64_t>(stride, 1 << 30));
    try {
      slab_run_impl(c, nsteps);
    } catch (...) {
      c->obs_stride = 0;
      throw;
    }
    c->obs_stride = 0;
    int64_t k = 0;
    for (const auto& r : c->obs_rows) {
      const int64_t st = static_cast<int64_t>(r[0]);
      if (st <= s0 || st > s0 + nsteps) continue;
      if (k < cap) {
        out[k].step = st;
        out[k].kinetic = r[1];
        out[k].potential = r[2];
        out[k].virial = r[3];
        out[k].temperature = 0.0;  // rank-local sums: the caller reduces over ranks
      }
      ++k;
    }
    *n_out = k;
  });
}

int tmd_gpu_slab_observe(tmd_gpu_ctx* c, int64_t n_total, tmd_observables* out) {
  return native_guard(c, [&] {
    need_slab(c);
    need_comm(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->launches += 1;
    launch_kinetic(c);
    launch_reduce_ke(c);
    launch_reduce_pe(c);
    comm(c)->allreduce(c->scalars, 3, CType::kF64, COp::kSum, c->stream);
    ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    out->step = c->step;
    out->potential = c->h_scalars[0];
    out->virial = c->h_scalars[1];
    out->kinetic = c->h_scalars[2];
    out->temperature = 2.0 * out->kinetic / (3.0 * static_cast<double>(n_total));
  });
}

}  // extern "C"
