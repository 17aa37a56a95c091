// libtmd_gpu.so — the B200 engine behind include/tmd_gpu.h.
//
// One context = one GPU = one cell-sorted, device-resident FP64 particle set.
// A run of K steps enqueues (engine.hpp:80-126 phase order):
//   Integrate  k_kick_drift         opening half-kick + drift of the first step
//   per step:
//   Neigh      k_decide             global max-displacement test, on device
//   Resort     k_wrap_bin, scan, k_scatter, k_sort_cells, k_permute, k_copy_back
//                                             (no-ops unless the device decided rebuild)
//   Neigh      k_build_prologue, k_build_cull / k_build_thread (no-op unless rebuild)
//   Forces     k_forces_staged / k_forces_l1 <kFused>  forces + closing half-kick
//              (+ Langevin) of this step + opening half-kick + drift of the next
//              (kKick2 on the last)
// Nothing in a chunk waits for the host. The host synchronises once per
// chunk to read the status word; a neighbour-list overflow rolls the chunk
// back to its checkpoint, grows the list and replays it.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/tmd_gpu.h"
#include "tmd_kernels.cuh"
#include "tmd_brick.cuh"
#include "tmd_slab.cuh"
#include "tmd_pairlist.cuh"

using namespace tmd;

namespace {

thread_local std::string g_create_error;

// Kernel variant used when the caller does not pick one (tmd_engine_params
// reserved[0] = 0); chosen by the ncu/CUDA-event comparison in
// profiles/ (see DESIGN.md §Force kernel variants).
constexpr int kDefaultVariant = 3;
// Below this many particles x lanes the one-thread-per-particle force grid
// leaves the SMs latency-bound; small systems split each particle's list
// over 2 or 4 threads (k_forces_lanes). Measured on B200 (scripts/
// lanes_probe.py, force kernel ms at lanes 1/2/4): 32K 0.033/0.021/0.019,
// 62.5K 0.035/0.033/0.031, 131K 0.044/0.049/0.052. Eight lanes (1024-thread
// blocks, one per SM) never won by more than 1 %.
constexpr int64_t kLanesTargetThreads = 148 * 768;
constexpr int kLanesAutoMax = 4;
// Up to this many particles graph steps keep the rebuild kernels as
// early-returning nodes instead of a conditional IF node (see if_nodes).
constexpr int64_t kChainMaxParticles = 262144;
// Up to this many particles graph runs use speculative blocks (see
// run_chunk); above, a conditional IF node per step (~7 us) is noise.
constexpr int64_t kSpecMaxParticles = 4194304;

struct CudaFail {
  std::string what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaFail{std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

struct StatusError {
  int code;
  std::string what;
};

inline int blocks_for(int64_t n, int t) {
  return static_cast<int>((n + t - 1) / t);
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

// Process-wide cache of the two big per-context blocks (the per-slot arena
// and the neighbour list). cudaMalloc / cudaFree of hundreds of MB cost from
// 0.5 to >100 ms each (page mapping), so a closed engine's blocks are kept
// for the next engine of the process (a sweep, a restart, the benchmark's
// end-to-end engine) instead of being returned to the driver; blocks are
// reused when they are at most 1.5x the request, the cache holds at most
// 16 GiB per device and is dropped whenever a cudaMalloc fails.
struct CachedBlock {
  int device;
  size_t bytes;
  void* p;
};
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;
constexpr size_t kCacheMax = size_t{16} << 30;

void cache_drop(int device) {  // (caller holds g_cache_mu)
  for (size_t k = 0; k < g_cache.size();) {
    if (g_cache[k].device == device) {
      cudaFree(g_cache[k].p);
      g_cache[k] = g_cache.back();
      g_cache.pop_back();
    } else {
      ++k;
    }
  }
}

// A block of at least `bytes` (its real size in *got).
void* big_alloc(size_t bytes, size_t* got) {
  bytes = std::max<size_t>(bytes, 256);
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t best = g_cache.size();
    for (size_t k = 0; k < g_cache.size(); ++k) {
      const CachedBlock& b = g_cache[k];
      if (b.device == dev && b.bytes >= bytes && b.bytes <= bytes + bytes / 2 &&
          (best == g_cache.size() || b.bytes < g_cache[best].bytes)) {
        best = k;
      }
    }
    if (best < g_cache.size()) {
      void* p = g_cache[best].p;
      *got = g_cache[best].bytes;
      g_cache[best] = g_cache.back();
      g_cache.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      cache_drop(dev);
    }
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  *got = bytes;
  return p;
}

void big_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  size_t held = 0;
  for (const CachedBlock& b : g_cache) held += b.device == dev ? b.bytes : 0;
  if (held + bytes > kCacheMax) {
    cudaFree(p);
    return;
  }
  g_cache.push_back({dev, bytes, p});
}

constexpr int kObsRowsAlloc = 256;  // observable rows a context's mapped buffer holds

// Device arrays that go through the block cache one by one (slab contexts'
// per-slot arrays, which regrow): their sizes are remembered so that the
// generic free path can hand them back to the cache.
std::mutex g_sized_mu;
std::vector<std::pair<void*, size_t>> g_sized;

void* sized_alloc(size_t bytes) {
  size_t got = 0;
  void* p = big_alloc(bytes, &got);
  std::lock_guard<std::mutex> lk(g_sized_mu);
  g_sized.push_back({p, got});
  return p;
}

// cudaFree, or back to the cache for a sized_alloc block.
void dev_free(void* p) {
  if (!p) return;
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_sized_mu);
    for (size_t k = 0; k < g_sized.size(); ++k) {
      if (g_sized[k].first == p) {
        bytes = g_sized[k].second;
        g_sized[k] = g_sized.back();
        g_sized.pop_back();
        break;
      }
    }
  }
  if (bytes) {
    big_free(p, bytes);
  } else {
    cudaFree(p);
  }
}

// Process-wide pool of small mapped pinned blocks (the per-context status
// mirror, scalars, observable rows): cudaHostAlloc costs milliseconds per
// call whatever the size, which an engine construction should not pay.
std::mutex g_pin_mu;
std::vector<std::pair<size_t, void*>> g_pin_free;  // (bytes, block)

void* pinned_small(size_t bytes) {
  bytes = (bytes + 255) / 256 * 256;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t k = 0; k < g_pin_free.size(); ++k) {
      if (g_pin_free[k].first == bytes) {
        void* p = g_pin_free[k].second;
        g_pin_free[k] = g_pin_free.back();
        g_pin_free.pop_back();
        return p;
      }
    }
  }
  void* p = nullptr;
  ck(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
  return p;
}

void pinned_small_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back({(bytes + 255) / 256 * 256, p});
}

std::string fmt_g(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%g", v);
  return b;
}

}  // namespace

struct tmd_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0;
  int stride = 0;
  int cap = 0;
  bool auto_cap = true;
  int nblk = 0;
  Geom g{};
  LjConst lj{};
  double dt = 0, half_dt = 0, r_skin = 0, r_cut = 0;
  bool timers_on = true;
  Thermo th{};  // Langevin bath (th.on = 0: NVE)
  // FENE bonds (row f1): static per-id bond table + per-slot resolved entries
  BondTab bt{};
  long long id_min = 0;
  int64_t id_span = 0;
  // download in id order on the device (ids forming a dense range, fixed
  // particle set): dl_lo = smallest id, dl = n * 10 doubles of scratch
  bool ids_dense = false;
  long long dl_lo = 0;
  double* dl = nullptr;
  // ParticleRec::type (flat_config.hpp:18-40): static per particle and never
  // read by the LJ path, so it stays on the host as a table by id, returned
  // by tmd_gpu_download like flatten_domain does (domain.hpp:193-207).
  // Empty: every type is 0. type_id empty: dense, type_val[id - type_lo].
  std::vector<long long> type_id;
  std::vector<int32_t> type_val;
  long long type_lo = 0;
  char* arena = nullptr;  // the per-slot arrays of a non-slab context, one allocation
  size_t arena_bytes = 0;
  size_t nbr_bytes = 0;   // size of the list block (big_alloc)
  int* slot_of_id = nullptr;       // [id_span] (owned + ghost slots), -1 = absent
  int* bond_off = nullptr;         // [id_span + 1] CSR over id - id_min
  int* bond_nbr = nullptr;         // partner id - id_min
  unsigned char* bond_anchor = nullptr;  // 1: this end is the bond's anchor a
  int* bnd_cnt = nullptr;          // [n_cap]
  uint32_t* bnd_ent = nullptr;     // [n_cap * kMaxBonds]

  // particle arrays (cell-sorted) + alternates for the permutation
  double4 *pos = nullptr, *pos2 = nullptr, *snap = nullptr;
  double4* posb[2] = {nullptr, nullptr};  // ping-pong position buffers; pos = posb[cur]
  int cur = 0;
  double *vx = nullptr, *vy = nullptr, *vz = nullptr;
  double *vx2 = nullptr, *vy2 = nullptr, *vz2 = nullptr;
  double *fx = nullptr, *fy = nullptr, *fz = nullptr;
  double *mass = nullptr, *mass2 = nullptr;
  long long *id = nullptr, *id2 = nullptr;
  int *cell = nullptr, *cell2 = nullptr, *rank = nullptr, *perm = nullptr;
  int *count = nullptr, *start = nullptr;
  uint32_t* nbr = nullptr;
  int* nnbr = nullptr;
  size_t nbr_words = 0;       // allocated list words

  // brick-major ordering + variant selection
  int variant = 2;            // 1: thread-per-particle ELL + L1 gathers; 2: brick-staged
  int unroll = 1;             // variant 3: gathers in flight per thread (1, 2, 4, 8)
  bool unroll_auto = true;    // unroll chosen with the build kind (sparse cells: 2)
  int lanes = 1;              // variant 3: threads per particle (1, 2, 4, 8)
  bool lanes_auto = true;     // lanes chosen from the particle count at create
  double occupancy = 0.0;     // particle-weighted mean cell occupancy at the first binning
  bool build_auto = false;    // build kind chosen from `occupancy` at the first binning
  int build_kind = 3;         // variant 3 list build: 3 = warp per cell (brick-staged),
                              // 5 = thread per particle (sparse cells),
                              // 6 = warp per cell over a culled candidate stream
  BrickGeom bg{};
  int* cell_rank = nullptr;       // global cell -> brick-major rank
  int* brick_rank_off = nullptr;  // brick -> first rank (nbricks + 1)
  int ngroups_max = 0;
  int nparts = 0;                 // partial-sum slots of the force kernel
  uint32_t* decoded = nullptr;    // global-index ELL copy for the taps
  size_t decoded_words = 0;
  int* scan_tmp = nullptr;               // tile sums of the tiled scan

  // PairIndexList (tmd_pairlist.cuh): explicit pairs of the current list
  uint2* pl_pairs = nullptr;      // {i, entry of j} per pair
  int64_t pl_m = 0;
  int* pl_off = nullptr;          // [n + 1] pairs of particle i start at pl_off[i]
  long long* pl_jstart = nullptr; // [n + 1] transposed index rows
  uint32_t* pl_jpairs = nullptr;  // pair numbers by j (stable)
  double* pl_fp = nullptr;        // [3 m] per-pair force
  double* pl_part = nullptr;      // [2 * blocks] energy / virial partials
  uint64_t pl_layout = 0;         // layout generation the pair list was built at
  uint64_t setups = 0;            // forced re-sorts (setup passes): slots move

  // z-slab decomposition (one context per GPU of a multi-GPU job)
  int64_t n_cap = 0;        // slot capacity (owned + ghosts in slab mode)
  int64_t n_total = 0;      // particles in the whole system
  int my_rank = 0, nranks = 1;
  int64_t n_ghost = 0, n_ghost_lo = 0, n_ghost_hi = 0;
  int* owner_of_z = nullptr;     // global z layer -> owning rank
  int* mig_dest = nullptr;
  int* mig_count = nullptr;      // [nranks] leavers per destination, then cursors
  int* mig_off = nullptr;
  int* mig_keep = nullptr;
  tmd::MigRec* mig_send = nullptr;
  tmd::MigRec* mig_recv = nullptr;
  int64_t mig_nrecv = 0;
  int* bidx[2] = {nullptr, nullptr};            // boundary-layer slots (down, up)
  long long* bids[2] = {nullptr, nullptr};
  double4* bpos[2] = {nullptr, nullptr};
  int* bcnt[2] = {nullptr, nullptr};            // per-cell counts of the layers
  int* boff[2] = {nullptr, nullptr};
  int64_t nb[2] = {0, 0};
  int* gcnt[2] = {nullptr, nullptr};            // received ghost-layer counts (lo, hi)
  void* comm = nullptr;          // SlabComm* of the native slab loop (tmd_comm.cuh): NCCL or in-process
  bool balance_count = false;    // native loop: load-aware cut planes at rebuilds
  bool fused_halo = false;       // native loop: positions to the neighbours from the epilogue
  bool fused_ready = false;      // remote ghost addresses valid for the current layout
  int2* exp = nullptr;           // [n_cap] export map (slab mode)
  double4* rg[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [side][parity]
  std::vector<std::pair<std::array<char, 64>, void*>> ipc_open;  // opened peer buffers
  int ipc_gen = 0;               // bumped whenever the position buffers are reallocated
  int64_t last_rebuild_step = -1;  // native loop: step of the last rebuild (batch sizing)
  int64_t rebuild_gap = 0;         // native loop: steps between the last two rebuilds
  std::vector<int> peer_gen;     // every rank's ipc_gen at the last full address exchange
  double4* peer_base[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [lo|hi][parity]
  std::vector<int> cuts;         // current cut planes (native loop)
  int64_t recuts = 0;
  int64_t* nccl_i64 = nullptr;   // staging for all-gathered counts
  double *part_e = nullptr, *part_w = nullptr, *part_ke = nullptr;
  double* scalars = nullptr;  // [0] pe, [1] virial, [2] ke
  Ctrl* ctrl = nullptr;
  Ctrl* h_ctrl = nullptr;      // pinned mirror
  Ctrl* h_ctrl_cyc = nullptr;  // pinned status snapshots of speculative cycles [4]
  cudaEvent_t ev_cyc[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_up[2] = {nullptr, nullptr};  // create(): positions copied / velocities copied
  double* h_scalars = nullptr; // pinned

  // chunk checkpoint (rollback on list overflow)
  double4* ck_pos = nullptr;
  double *ck_vx = nullptr, *ck_vy = nullptr, *ck_vz = nullptr, *ck_mass = nullptr;
  double *ck_fx = nullptr, *ck_fy = nullptr, *ck_fz = nullptr;  // thermostat runs only
  long long* ck_id = nullptr;

  // host mirrors
  int64_t step = 0;
  uint64_t rebuilds = 0;
  bool ke_fresh = false;  // part_ke holds the current velocities' partials
  int ke_parts = 1;       // valid part_ke slots (see force_parts)
  bool obs_fresh = false; // h_scalars holds PE, W, KE of the current state
  bool ck_valid = false;  // a rollback checkpoint exists (invalidated by state edits)
  int64_t ck_step = 0;
  Ctrl ck_ctrl{};
  double sec[5] = {0, 0, 0, 0, 0};
  double elapsed = 0.0;
  std::string err;

  std::vector<cudaEvent_t> ev;  // pool for per-phase timing
  size_t ev_used = 0;
  struct Span {
    int section;
    size_t b, e;
    int step_idx;  // chunk-relative step for Resort spans, else -1
  };
  std::vector<Span> ev_spans;
  int* rebuild_log = nullptr;     // device: rebuild decision per chunk step
  std::vector<int> h_rebuild_log;
  long long* ticks = nullptr;     // device phase stamps (graph mode with section timers)
  std::vector<long long> h_ticks;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  uint64_t launches = 0;  // kernels enqueued by this context (bench accounting)

  // CUDA-graph execution of whole step blocks (used when section timers are
  // off): one graph = kick1+drift, kGraphSteps x [decide, IF(rebuild){resort,
  // list build}, forces + fused integrator], PE reduction. The rebuild branch
  // is a conditional graph node whose condition the decide kernel sets on the
  // device, so skipped rebuilds cost nothing and nothing waits for the host.
  cudaStream_t ls = nullptr;    // stream the launch wrappers enqueue on
  cudaStream_t side = nullptr;  // capture stream for conditional bodies
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    uint64_t fixed = 0;  // kernels per launch outside the IF bodies
  };
  StepGraph sg[2][2];  // [block of kGraphSteps | single step][starting buffer parity]
  // Speculative graph mode (spec_mode, chosen at create): blocks of K steps
  // with no conditional node (k_decide_spec1 halts a block at a due rebuild)
  // each followed by one closing step that holds the rebuild kernels; keyed
  // K << 3 | open << 2 | parity << 1 | observed (K = 0: the closing step,
  // open: it starts with the opening kick + drift).
  bool spec_mode = false;
  int halt_copy = 0;  // set while capturing a speculative block's force launches
  std::map<int, StepGraph> spec;
  StepGraph sgo[2][2]; // the same with a per-step observable row (run_observed)
  int obs_stride = 0;           // > 0 while run_observed records rows
  int sgo_stride = 0;           // stride the observed graphs were captured with
  double* obs_host = nullptr;   // mapped pinned rows [kChunk][4]: step, KE, PE, W
  double* obs_dev = nullptr;    // its device alias
  std::vector<std::array<double, 4>> obs_rows;  // rows of the current run_observed
  bool graph_dirty = true;
  bool use_graphs = true;
  uint64_t graph_body_kernels = 0;   // kernels per executed IF body
  unsigned long long cond_handle = 0;  // handle the next decide sets (0: none)
  // Graph steps gate the rebuild kernels with a conditional IF node (large
  // systems), or keep them as early-returning kernel nodes (small systems,
  // where the IF node's ~9 us per step is a third of the step). At create.
  bool if_nodes = true;
};

namespace {

void destroy_graph(tmd_gpu_ctx::StepGraph& s) {
  if (s.exec) cudaGraphExecDestroy(s.exec);
  if (s.graph) cudaGraphDestroy(s.graph);
  s = tmd_gpu_ctx::StepGraph{};
}

void drop_spec_graphs(tmd_gpu_ctx* c, bool observed_only) {
  for (auto it = c->spec.begin(); it != c->spec.end();) {
    if (!observed_only || (it->first & 1)) {
      destroy_graph(it->second);
      it = c->spec.erase(it);
    } else {
      ++it;
    }
  }
}

void drop_graphs(tmd_gpu_ctx* c) {
  for (auto* fam : {&c->sg, &c->sgo}) {
    for (auto& row : *fam) {
      for (auto& s : row) destroy_graph(s);
    }
  }
  drop_spec_graphs(c, false);
  c->graph_dirty = false;
}

void free_comm(tmd_gpu_ctx* c);

void free_all(tmd_gpu_ctx* c) {
  drop_graphs(c);
  free_comm(c);
  if (c->side) cudaStreamDestroy(c->side);
  void* ptrs[] = {c->posb[0], c->posb[1], c->pos2, c->snap, c->vx, c->vy, c->vz,
                  c->vx2,  c->vy2,   c->vz2,  c->fx,    c->fy,      c->fz,
                  c->mass, c->mass2, c->id,   c->id2,   c->cell,    c->cell2,
                  c->rank, c->perm,  c->count, c->start, c->nnbr,
                  c->part_e, c->part_w, c->part_ke, c->scalars, c->ctrl,
                  c->ck_pos, c->ck_vx, c->ck_vy, c->ck_vz, c->ck_mass, c->ck_id,
                  c->ck_fx, c->ck_fy, c->ck_fz,
                  c->rebuild_log, c->ticks, c->cell_rank, c->brick_rank_off,
                  c->decoded, c->scan_tmp, c->owner_of_z, c->mig_dest,
                  c->mig_count, c->mig_off, c->mig_keep, c->mig_send, c->mig_recv,
                  c->bidx[0], c->bidx[1], c->bids[0], c->bids[1], c->bpos[0], c->bpos[1],
                  c->bcnt[0], c->bcnt[1], c->boff[0], c->boff[1], c->gcnt[0], c->gcnt[1],
                  c->slot_of_id, c->bond_off, c->bond_nbr, c->bond_anchor, c->bnd_cnt,
                  c->bnd_ent, c->nccl_i64, c->exp, c->dl, c->pl_pairs, c->pl_off,
                  c->pl_jstart, c->pl_jpairs, c->pl_fp, c->pl_part};
  const char* a0 = c->arena;
  const char* a1 = c->arena + c->arena_bytes;
  for (void* p : ptrs) {
    const char* q = static_cast<const char*>(p);
    if (p && !(a0 && q >= a0 && q < a1)) dev_free(p);
  }
  big_free(c->arena, c->arena_bytes);  // back to the process cache
  big_free(c->nbr, c->nbr_bytes);
  pinned_small_free(c->h_ctrl, sizeof(Ctrl));
  pinned_small_free(c->h_ctrl_cyc, 4 * sizeof(Ctrl));
  for (cudaEvent_t e : c->ev_cyc) {
    if (e) cudaEventDestroy(e);
  }
  for (cudaEvent_t e : c->ev_up) {
    if (e) cudaEventDestroy(e);
  }
  pinned_small_free(c->obs_host, sizeof(double) * 4 * kObsRowsAlloc);
  pinned_small_free(c->h_scalars, 4 * sizeof(double));
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  if (c->stream) cudaStreamDestroy(c->stream);
}

// --- per-phase timing ------------------------------------------------------
cudaEvent_t next_event(tmd_gpu_ctx* c) {
  if (c->ev_used == c->ev.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    c->ev.push_back(e);
  }
  return c->ev[c->ev_used++];
}

struct Phase {
  tmd_gpu_ctx* c;
  int section;
  size_t b;
  int step_idx;
  Phase(tmd_gpu_ctx* ctx, int s, int step = -1)
      : c(ctx), section(s), b(0), step_idx(step) {
    if (!c->timers_on) return;
    b = c->ev_used;
    ck(cudaEventRecord(next_event(c), c->stream), "cudaEventRecord");
  }
  ~Phase() {
    if (!c->timers_on) return;
    const size_t e = c->ev_used;
    if (cudaEventRecord(next_event(c), c->stream) == cudaSuccess) {
      c->ev_spans.push_back({section, b, e, step_idx});
    }
  }
};

// Resort spans of steps that did not rebuild ran only the early-exit
// kernels: that time is the rebuild check and is booked to Neigh, so Resort
// stays zero without rebuilds (test_engine.cpp:306-321).
void harvest_timers(tmd_gpu_ctx* c) {
  for (const auto& s : c->ev_spans) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[s.b], c->ev[s.e]) != cudaSuccess) continue;
    int sec = s.section;
    if (sec == TMD_SECTION_RESORT && s.step_idx >= 0 &&
        s.step_idx < static_cast<int>(c->h_rebuild_log.size()) &&
        c->h_rebuild_log[s.step_idx] == 0) {
      sec = TMD_SECTION_NEIGH;
    }
    c->sec[sec] += 1e-3 * ms;
  }
  c->ev_spans.clear();
  c->ev_used = 0;
}

// Graph mode: consecutive phase stamps of a chunk -> SectionTimers. The time
// from a stamp to the next one is booked to the stamp's phase: block start
// (the block's opening kick + drift) -> Integrate; decision -> Resort on
// rebuild steps (decision + resort), else Neigh (the rebuild check); list
// build -> Neigh; forces (+ fused integrator epilogue, observables) -> Forces.
void harvest_ticks(tmd_gpu_ctx* c, int64_t steps) {
  const auto& t = c->h_ticks;
  const int64_t ns = std::min<int64_t>(steps, kTickSteps);
  std::vector<std::pair<long long, int>> seq;  // (time, section)
  for (int64_t s = 0; s < ns; ++s) {
    const long long* p = t.data() + s * kTickPhases;
    const bool rebuilt = p[kTickBuild] != 0;
    if (p[kTickBlock]) seq.push_back({p[kTickBlock], TMD_SECTION_INTEGRATE});
    if (p[kTickDecide]) {
      seq.push_back({p[kTickDecide], rebuilt ? TMD_SECTION_RESORT : TMD_SECTION_NEIGH});
    }
    if (rebuilt) seq.push_back({p[kTickBuild], TMD_SECTION_NEIGH});
    if (p[kTickForces]) seq.push_back({p[kTickForces], TMD_SECTION_FORCES});
  }
  const long long end = t[static_cast<size_t>(kTickSteps * kTickPhases)];
  for (size_t k = 0; k < seq.size(); ++k) {
    const long long next = k + 1 < seq.size() ? seq[k + 1].first : end;
    if (next > seq[k].first) c->sec[seq[k].second] += 1e-9 * static_cast<double>(next - seq[k].first);
  }
}

// --- kernel launch wrappers -------------------------------------------------
// Phase stamps are taken in graph mode with section timers on (the eager
// path times phases with CUDA events instead).
long long* tick_ptr(const tmd_gpu_ctx* c) {
  return c->timers_on && c->use_graphs ? c->ticks : nullptr;
}

void launch_tick(tmd_gpu_ctx* c, int phase, int off) {
  if (!tick_ptr(c)) return;
  c->launches += 1;
  k_tick<<<1, 1, 0, c->ls>>>(c->ctrl, c->ticks, phase, off, -1);
}

void launch_decide(tmd_gpu_ctx* c, bool advance, int log_idx = -1) {
  c->launches += 1;
  k_decide<<<1, 1, 0, c->ls>>>(c->ctrl, c->g.rebuild_thr, advance ? 1 : 0,
                               log_idx >= 0 ? c->rebuild_log : nullptr, log_idx,
                               c->cond_handle, advance ? tick_ptr(c) : nullptr);
}

// Exclusive scan of counts[0..n) into out[0..n] (3 tiled kernels).
void launch_scan(tmd_gpu_ctx* c, int n, int* counts, int* out) {
  c->launches += 3;
  const int tiles = blocks_for(n, kScanTile);
  k_scan_tiles<<<tiles, kScanThreads, 0, c->ls>>>(n, counts, c->scan_tmp, c->ctrl);
  k_scan_sums<<<1, kScanThreads, 0, c->ls>>>(tiles, c->scan_tmp, c->ctrl);
  k_scan_apply<<<tiles, kScanThreads, 0, c->ls>>>(n, counts, c->scan_tmp, out, c->ctrl);
}

// Mean cell occupancy below which the in-cell id sort runs a thread per slot.
constexpr double kSortCellWarpMin = 8.0;

void launch_resort(tmd_gpu_ctx* c) {
  c->launches += 5;
  const int n = static_cast<int>(c->n);
  const int nb = c->nblk;
  k_wrap_bin<<<nb, kBlock, 0, c->ls>>>(n, c->pos, c->id, c->cell, c->rank,
                                           c->count, c->cell_rank, c->g, c->ctrl);
  launch_scan(c, c->g.owned_cells, c->count, c->start);
  k_scatter<<<nb, kBlock, 0, c->ls>>>(n, c->cell, c->rank, c->start,
                                          c->cell_rank, c->g, c->perm, c->ctrl);
  // in-cell id order: a warp per cell for dense cells, a thread per slot
  // (writing the order into the free `rank` array) for sparse ones
  const bool sparse = c->occupancy > 0.0 && c->occupancy < kSortCellWarpMin;
  if (sparse) {
    k_sort_cells_thread<<<nb, kBlock, 0, c->ls>>>(n, c->start, c->cell, c->cell_rank, c->g,
                                                  c->perm, c->id, c->rank, c->ctrl);
  } else {
    k_sort_cells<<<blocks_for(static_cast<int64_t>(c->g.owned_cells) * 32, kBlock), kBlock, 0,
                   c->ls>>>(c->g.owned_cells, c->start, c->perm, c->id, c->ctrl);
  }
  k_permute<<<nb, kBlock, 0, c->ls>>>(n, sparse ? c->rank : c->perm, c->pos, c->vx, c->vy,
                                          c->vz, c->mass, c->id, c->cell,
                                          c->pos2, c->vx2, c->vy2, c->vz2,
                                          c->mass2, c->id2, c->cell2, c->ctrl);
  k_copy_back<<<nb, kBlock, 0, c->ls>>>(n, c->pos2, c->vx2, c->vy2,
                                            c->vz2, c->mass2, c->id2, c->cell2,
                                            c->pos, c->vx, c->vy, c->vz,
                                            c->mass, c->id, c->cell, c->ctrl);
}

size_t build_smem(const tmd_gpu_ctx* c) {
  return static_cast<size_t>(c->bg.stage_cap + 32) * 4 * sizeof(float);
}
size_t force_smem(const tmd_gpu_ctx* c) { return staged_smem_bytes(c->bg.stage_cap); }
bool staged_large(const tmd_gpu_ctx* c) { return c->bg.B[0] * c->bg.B[1] * c->bg.B[2] > 8; }

// Max dynamic shared memory is a per-kernel, per-device attribute shared by
// every context of the process, while the staging capacity is per context:
// raise it to the largest any context on the device has needed, never lower
// it under another context.
constexpr int kMaxDevices = 64;
size_t g_build_smem_set[kMaxDevices] = {}, g_force_smem_set[kMaxDevices] = {};

void set_smem_attrs(tmd_gpu_ctx* c) {
  c->graph_dirty = true;
  const size_t b = build_smem(c), f = force_smem(c);
  const int d = std::min(std::max(c->device, 0), kMaxDevices - 1);
  size_t& g_build = g_build_smem_set[d];
  size_t& g_force = g_force_smem_set[d];
  if (b > g_build) {
    ck(cudaFuncSetAttribute(k_build_brick3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(b)), "smem attr build");
    ck(cudaFuncSetAttribute(k_build_brick3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(b)), "smem attr build");
    ck(cudaFuncSetAttribute(k_build_cull<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(b)), "smem attr build");
    ck(cudaFuncSetAttribute(k_build_cull<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(b)), "smem attr build");
    g_build = b;
  }
  if (f > g_force && f <= kStagedSmemMax) {  // (larger: the context runs variant 3)
    const void* ks[] = {
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsSmall, kForcesOnly>),
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsSmall, kKick2>),
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsSmall, kFused>),
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsLarge, kForcesOnly>),
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsLarge, kKick2>),
        reinterpret_cast<const void*>(k_forces_staged<kStagedThreadsLarge, kFused>)};
    for (const void* k : ks) {
      ck(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(f)), "smem attr forces");
    }
    g_force = f;
  }
}

// Bond resolution of a rebuild (gated on the device decision like the rest of
// the rebuild): id -> slot table over owned + ghost slots, then per owned slot
// its bonds' partner slots and closest images.
void launch_bond_resolve(tmd_gpu_ctx* c) {
  if (!c->bt.on) return;
  c->launches += 2;
  const int span = static_cast<int>(c->id_span);
  const int slots = static_cast<int>(c->n + c->n_ghost);
  if (c->g.zslab) {  // absent ids (other slabs' particles) must read -1; a whole-box
                     // context holds every id, each slot entry rewritten below
    c->launches += 1;
    k_fill_int<<<blocks_for(span, kBlock), kBlock, 0, c->ls>>>(span, c->slot_of_id, -1,
                                                                c->ctrl);
  }
  k_slot_of_id<<<std::max(1, blocks_for(slots, kBlock)), kBlock, 0, c->ls>>>(
      slots, c->id, c->id_min, c->slot_of_id, c->ctrl);
  k_bond_resolve<<<c->nblk, kBlock, 0, c->ls>>>(
      static_cast<int>(c->n), c->pos, c->id, c->id_min, c->bond_off, c->bond_nbr,
      c->bond_anchor, c->slot_of_id, c->g, c->bnd_cnt, c->bnd_ent, c->ctrl);
}

void launch_build(tmd_gpu_ctx* c) {
  launch_bond_resolve(c);
  c->launches += 2;
  k_build_prologue<<<1, 1, 0, c->ls>>>(c->ctrl, tick_ptr(c));
  if (c->variant == 1) {
    k_build_list<<<c->nblk, kBlock, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, c->cell, c->start, c->cell_rank, c->g, c->nbr,
        c->nnbr, c->stride, c->cap, c->snap, c->ctrl);
  } else if (c->variant == 3 && c->build_kind == 5) {
    k_build_thread<<<c->nblk, kBlock, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, c->cell, c->start, c->cell_rank, c->g, c->nbr,
        c->nnbr, c->cap, c->snap, static_cast<uint32_t>(c->n_cap), c->ctrl);
  } else if (c->build_kind == 6) {  // variant 2: staging-index entries
    auto kern = c->variant == 2 ? k_build_cull<true> : k_build_cull<false>;
    kern<<<c->bg.nbricks, kBuildThreads, build_smem(c) / 4 * 3, c->ls>>>(
        c->pos, c->cell_rank, c->brick_rank_off, c->start, c->g, c->bg, c->nbr, c->nnbr,
        c->snap,
        static_cast<uint32_t>(c->variant == 2 ? c->bg.stage_cap : c->n_cap), c->ctrl);
  } else {
    auto kern = c->variant == 2 ? k_build_brick3<false> : k_build_brick3<true>;
    kern<<<c->bg.nbricks, kBuildThreads, build_smem(c), c->ls>>>(
        c->pos, c->cell_rank, c->brick_rank_off, c->start, c->g, c->bg, c->nbr, c->nnbr,
        c->snap, static_cast<uint32_t>(c->n_cap), c->ctrl);
  }
}

int force_parts(const tmd_gpu_ctx* c);

template <int kMode>
void launch_forces_mode(tmd_gpu_ctx* c) {
  Integ it;
  it.vx = c->vx;
  it.vy = c->vy;
  it.vz = c->vz;
  it.mass = c->mass;
  it.id = c->id;
  it.snap = c->snap;
  it.pos_out = c->posb[c->cur ^ 1];
  it.dt = c->dt;
  it.half_dt = c->half_dt;
  it.part_ke = c->part_ke;
  it.th = c->th;
  it.bt = c->bt;
  it.bt.cnt = c->bnd_cnt;
  it.bt.ent = c->bnd_ent;
  const bool fh = kMode == kFused && c->fused_halo && c->fused_ready;
  it.exp = fh ? c->exp : nullptr;
  it.halt_copy = kMode == kFused ? c->halt_copy : 0;
  it.rg[0] = fh ? c->rg[0][c->cur ^ 1] : nullptr;
  it.rg[1] = fh ? c->rg[1][c->cur ^ 1] : nullptr;
  if (c->variant == 1) {
    k_lj_forces<kMode><<<c->nblk, kBlock, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, c->nbr, c->nnbr, c->stride, c->g, c->lj,
        c->fx, c->fy, c->fz, c->part_e, c->part_w, c->id, it, c->ctrl);
  } else if (c->variant == 3 && c->lanes > 1) {
    auto kern = c->lanes == 2 ? k_forces_lanes<4, kMode, 2>
                              : (c->lanes == 4 ? k_forces_lanes<2, kMode, 4>
                                               : k_forces_lanes<2, kMode, 8>);
    kern<<<force_parts(c), kLanesPPB * c->lanes, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, c->nbr, c->nnbr, c->cap, c->g, c->lj, c->fx, c->fy,
        c->fz, c->part_e, c->part_w, c->id, it, c->ctrl);
  } else if (c->variant == 3) {
    auto kern = c->unroll == 1 ? k_forces_l1<1, kMode>
                               : (c->unroll == 2 ? k_forces_l1<2, kMode>
                                                 : (c->unroll == 8 ? k_forces_l1<8, kMode>
                                                                   : k_forces_l1<4, kMode>));
    kern<<<c->nblk, 128, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, c->nbr, c->nnbr, c->cap, c->g, c->lj, c->fx, c->fy,
        c->fz, c->part_e, c->part_w, c->id, it, c->ctrl);
  } else {
    auto kern = staged_large(c) ? k_forces_staged<kStagedThreadsLarge, kMode>
                                : k_forces_staged<kStagedThreadsSmall, kMode>;
    kern<<<c->bg.nbricks, staged_large(c) ? kStagedThreadsLarge : kStagedThreadsSmall,
           force_smem(c), c->ls>>>(
        c->pos, c->cell_rank, c->brick_rank_off, c->start, c->g, c->bg, c->lj, c->nbr,
        c->nnbr, c->fx, c->fy, c->fz, c->part_e, c->part_w, c->id, it, c->ctrl);
  }
}

// Forces at the current positions, optionally with the fused integrator
// epilogue (kKick2: closing half-kick; kFused: closing half-kick + next
// step's opening half-kick and drift into the other position buffer, after
// which the buffers swap).
// Kinetic partials of the current velocities, 128 particles per slot.
void launch_kinetic(tmd_gpu_ctx* c) {
  c->ke_parts = c->nblk;
  k_kinetic<<<c->nblk, kBlock, 0, c->ls>>>(static_cast<int>(c->n), c->vx, c->vy, c->vz, c->mass,
                                          c->part_ke);
}

void launch_forces(tmd_gpu_ctx* c, int mode = kForcesOnly) {
  c->launches += 1;
  if (mode != kForcesOnly) c->ke_parts = force_parts(c);  // its kinetic partials
  if (mode == kFused) {
    launch_forces_mode<kFused>(c);
    c->cur ^= 1;
    c->pos = c->posb[c->cur];
  } else if (mode == kKick2) {
    launch_forces_mode<kKick2>(c);
  } else {
    launch_forces_mode<kForcesOnly>(c);
  }
}

// Partial-sum slots the force kernel writes (its grid), and the kinetic
// partials' count: the force grid after a kicking force launch, the
// 128-particle grid after k_kinetic (recorded when the reducer is enqueued
// or captured).
int force_parts(const tmd_gpu_ctx* c) {
  if (c->variant == 2) return c->bg.nbricks;
  if (c->variant == 3 && c->lanes > 1) return std::max(1, blocks_for(c->n, kLanesPPB));
  return c->nblk;
}

void launch_kick_drift(tmd_gpu_ctx* c) {
  c->launches += 1;
  k_kick_drift<<<c->nblk, kBlock, 0, c->ls>>>(static_cast<int>(c->n), c->pos, c->vx, c->vy,
                                             c->vz, c->fx, c->fy, c->fz, c->mass, c->snap,
                                             c->dt, c->half_dt, c->ctrl);
}


// The Langevin force of the initial evaluation (noise keyed as step 0).
void launch_thermo_init(tmd_gpu_ctx* c) {
  if (!c->th.on || c->n == 0) return;
  c->launches += 1;
  k_thermo_init<<<c->nblk, kBlock, 0, c->ls>>>(static_cast<int>(c->n), c->vx, c->vy, c->vz,
                                              c->mass, c->id, c->th, c->fx, c->fy, c->fz);
}

void launch_reduce_pe(tmd_gpu_ctx* c) {
  c->launches += 2;
  const int np = force_parts(c);
  k_reduce<<<1, kRedThreads, 0, c->ls>>>(c->part_e, np, 0.5, c->scalars + 0);
  k_reduce<<<1, kRedThreads, 0, c->ls>>>(c->part_w, np, 0.5, c->scalars + 1);
}

void launch_reduce_ke(tmd_gpu_ctx* c) {
  c->launches += 1;
  k_reduce<<<1, kRedThreads, 0, c->ls>>>(c->part_ke, c->ke_parts, 1.0,
                                             c->scalars + 2);
}

// --- status handling ---------------------------------------------------------
void sync_ctrl(tmd_gpu_ctx* c) {
  ck(cudaMemcpyAsync(c->h_ctrl, c->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost,
                     c->stream),
     "cudaMemcpyAsync(ctrl)");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  ck(cudaGetLastError(), "kernel launch");
}

// Physics errors (overlap / non-finite) -> StatusError with the reference's
// message shapes. Overflow is handled by the caller.
void raise_physics(tmd_gpu_ctx* c, bool with_step) {
  const Ctrl& h = *c->h_ctrl;
  std::string msg;
  // the first error in time wins (later ones can be its consequences, e.g. a
  // non-finite position binned at the origin then "overlaps")
  const int first = (h.err_bit & h.status) ? h.err_bit : h.status;
  if (first & kStatOverlap) {
    msg = "overlapping particles: ids " + std::to_string(h.err_id0) + " and " +
          std::to_string(h.err_id1) + " coincide";
  } else if (first & kStatNonFinite) {
    msg = "non-finite velocity or force on particle id " +
          std::to_string(h.err_id0);
  } else if (first & kStatNonFinitePos) {
    msg = "non-finite position for particle id " + std::to_string(h.err_id0);
  } else if (first & kStatBondStretch) {
    msg = "fene bond overstretched between ids " + std::to_string(h.err_id0) + " and " +
          std::to_string(h.err_id1) + ": r = " + std::to_string(std::sqrt(h.err_val)) +
          " >= r_max = " + std::to_string(std::sqrt(c->bt.rmax2));
  } else if (first & kStatBondReach) {
    msg = "bonded partner id " + std::to_string(h.err_id1) +
          " is out of reach of particle id " + std::to_string(h.err_id0) +
          " (bond stretched beyond the ghost shell)";
  } else {
    return;
  }
  if (with_step) msg += " (at step " + std::to_string(h.err_step) + ")";
  throw StatusError{TMD_ERR_PHYSICS, msg};
}

void reset_status(tmd_gpu_ctx* c) {
  // clear status + error latch (host-side write of the two ints)
  Ctrl z = *c->h_ctrl;
  z.status = 0;
  z.err_lock = 0;
  ck(cudaMemcpyAsync(&c->ctrl->status, &z.status, 2 * sizeof(int),
                     cudaMemcpyHostToDevice, c->stream),
     "cudaMemcpyAsync(status)");
}

void set_force_rebuild(tmd_gpu_ctx* c) {
  const int one = 1;
  ck(cudaMemcpyAsync(&c->ctrl->force_rebuild, &one, sizeof(int),
                     cudaMemcpyHostToDevice, c->stream),
     "cudaMemcpyAsync(force_rebuild)");
}

void set_cap_in_ctrl(tmd_gpu_ctx* c) {
  ck(cudaMemcpyAsync(&c->ctrl->cap, &c->cap, sizeof(int),
                     cudaMemcpyHostToDevice, c->stream),
     "cudaMemcpyAsync(cap)");
}

int round8(int v) { return (v + 7) / 8 * 8; }

void alloc_list(tmd_gpu_ctx* c, int cap) {
  c->graph_dirty = true;  // captured kernels hold the old list pointer / capacity
  big_free(c->nbr, c->nbr_bytes);
  c->nbr = nullptr;
  c->cap = round8(std::max(cap, 8));
  c->bg.cap = c->cap;
  c->nbr_words = c->variant == 1
                     ? static_cast<size_t>(c->cap) * c->stride
                     : static_cast<size_t>(c->ngroups_max) * c->cap * 32;
  c->nbr = static_cast<uint32_t*>(big_alloc(c->nbr_words * sizeof(uint32_t), &c->nbr_bytes));
  set_cap_in_ctrl(c);
}

// Resort + list build + forces at the current state, forced (setup / after a
// rollback). Grows the list until it fits. Leaves the PE reduced.
// Grows whatever overflowed at the last build: list capacity (entries per
// particle) and/or the brick staging capacity. A staging need beyond what a
// force CTA can hold in shared memory switches the context to variant 1
// (thread-per-particle, no staging), which has no density limit.
void grow_after_overflow(tmd_gpu_ctx* c, const Ctrl& h) {
  if (h.status & kStatStageOverflow) {
    const int want = (static_cast<int>(h.max_halo * 1.15) + 64 + 31) / 32 * 32;
    if (c->variant == 2 && staged_smem_bytes(want) > kStagedSmemMax) {
      c->variant = 3;  // staged forces: the buffers no longer fit shared memory
      c->graph_dirty = true;
    }
    if (static_cast<size_t>(want + 4) * 3 * sizeof(double) > 200 * 1024) {
      c->variant = 1;
    } else {
      c->bg.stage_cap = std::max(c->bg.stage_cap, want);
      set_smem_attrs(c);
    }
    alloc_list(c, c->cap);
  }
  if (h.status & kStatOverflow) {
    const int need = h.max_count;
    alloc_list(c, std::max(c->cap, need + need / 4 + 8));
  }
}

constexpr int kOverflowBits = kStatOverflow | kStatStageOverflow;

constexpr double kBuildCellWarpMin = 12.0;  // mean particles per cell (measured crossover)

// List build kind by the occupancy a particle sees (sum n_c^2 / sum n_c over
// the owned cells of the first binning, so a dense slab in a mostly empty box
// counts as dense): a warp per cell while cells hold most of a warp, else a
// thread per particle (sparse cells, e.g. the KG melt).
void choose_build_kind(tmd_gpu_ctx* c) {
  const int nc = c->g.owned_cells;
  // sum of n_c^2 on the device (sum of n_c = the owned particles)
  ck(cudaMemsetAsync(&c->ctrl->occ_s2, 0, sizeof(unsigned long long), c->stream), "memset");
  c->launches += 1;
  k_occupancy<<<std::max(1, blocks_for(nc, kBlock)), kBlock, 0, c->stream>>>(nc, c->start,
                                                                              c->ctrl);
  int s1i = 0;
  ck(cudaMemcpyAsync(&s1i, c->start + nc, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
     "D2H count");
  sync_ctrl(c);
  const double s1 = static_cast<double>(s1i);
  const double s2 = static_cast<double>(c->h_ctrl->occ_s2);
  c->occupancy = s1 > 0.0 ? s2 / s1 : 0.0;
  c->build_kind = c->occupancy >= kBuildCellWarpMin ? 6 : 5;
  // sparse cells (short lists, ~12 entries in the KG melt): two gathers in
  // flight per thread beat four (KG force kernel 0.281 vs 0.307 ms at 4M,
  // scripts/kg_probe.py; fewer registers, more resident warps)
  // dense cells: one gather at a time since the list's next chunk is
  // prefetched into L2 (fewer registers, more resident warps; 16.4M: 3.82 ms
  // against 3.83 / 3.88 with two / four in flight, 442K: 0.126 / 0.129 / 0.136;
  // scripts/unroll_probe.py) — four were best before the prefetches
  if (c->unroll_auto) c->unroll = c->build_kind == 5 ? 2 : 1;
  c->build_auto = false;
  c->graph_dirty = true;
}

// The staged force kernel (variant 2, on request) needs the brick build's
// staging-index list (build kinds 3 and 6) and its staging in shared memory.
void choose_variant(tmd_gpu_ctx* c) {
  if (c->variant == 2 && (c->build_kind == 5 || force_smem(c) > kStagedSmemMax)) {
    c->variant = 3;
    c->graph_dirty = true;
  }
}

// TMD_DEBUG_TIMING: synchronise and print the time since the last mark (the
// create() breakdown; no effect otherwise).
void debug_mark(tmd_gpu_ctx* c, const char* what) {
  if (!std::getenv("TMD_DEBUG_TIMING")) return;
  static thread_local auto prev = std::chrono::steady_clock::now();
  cudaStreamSynchronize(c->stream);
  const auto t = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[tmd setup ] %-24s %8.2f ms\n", what,
               std::chrono::duration<double, std::milli>(t - prev).count());
  prev = t;
}

void setup_pass(tmd_gpu_ctx* c) {
  c->setups += 1;
  debug_mark(c, "setup start");
  for (;;) {
    set_force_rebuild(c);
    launch_decide(c, false);
    launch_resort(c);
    debug_mark(c, "resort");
    if (c->build_auto) choose_build_kind(c);
    choose_variant(c);
    debug_mark(c, "build kind");
    launch_build(c);
    sync_ctrl(c);
    debug_mark(c, "build");
    raise_physics(c, false);
    if (c->h_ctrl->status & kOverflowBits) {
      const Ctrl h = *c->h_ctrl;
      reset_status(c);
      grow_after_overflow(c, h);
      continue;
    }
    break;
  }
  if (c->auto_cap) {
    // headroom for the liquid to densify locally between builds
    const int want = round8(c->h_ctrl->max_count + c->h_ctrl->max_count / 4 + 8);
    if (want > c->cap) {
      alloc_list(c, want);
      set_force_rebuild(c);
      launch_decide(c, false);
      launch_build(c);
    }
  }
  debug_mark(c, "cap");
  launch_forces(c);
  launch_thermo_init(c);
  launch_reduce_pe(c);
  sync_ctrl(c);
  debug_mark(c, "forces");
  raise_physics(c, false);
}

void checkpoint(tmd_gpu_ctx* c) {
  const size_t n = static_cast<size_t>(c->n);
  auto cp = [&](void* d, const void* s, size_t bytes) {
    ck(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, c->stream),
       "checkpoint copy");
  };
  cp(c->ck_pos, c->pos, n * sizeof(double4));
  cp(c->ck_vx, c->vx, n * sizeof(double));
  cp(c->ck_vy, c->vy, n * sizeof(double));
  cp(c->ck_vz, c->vz, n * sizeof(double));
  cp(c->ck_mass, c->mass, n * sizeof(double));
  cp(c->ck_id, c->id, n * sizeof(long long));
  if (c->th.on) {  // the stored force carries the last Langevin kick: keep it
    cp(c->ck_fx, c->fx, n * sizeof(double));
    cp(c->ck_fy, c->fy, n * sizeof(double));
    cp(c->ck_fz, c->fz, n * sizeof(double));
  }
}

void restore(tmd_gpu_ctx* c, const Ctrl& at_checkpoint) {
  const size_t n = static_cast<size_t>(c->n);
  auto cp = [&](void* d, const void* s, size_t bytes) {
    ck(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, c->stream),
       "restore copy");
  };
  cp(c->pos, c->ck_pos, n * sizeof(double4));
  cp(c->vx, c->ck_vx, n * sizeof(double));
  cp(c->vy, c->ck_vy, n * sizeof(double));
  cp(c->vz, c->ck_vz, n * sizeof(double));
  cp(c->mass, c->ck_mass, n * sizeof(double));
  cp(c->id, c->ck_id, n * sizeof(long long));
  if (c->th.on) {
    cp(c->fx, c->ck_fx, n * sizeof(double));
    cp(c->fy, c->ck_fy, n * sizeof(double));
    cp(c->fz, c->ck_fz, n * sizeof(double));
  }
  Ctrl back = at_checkpoint;
  back.status = 0;
  back.err_lock = 0;
  back.max_d2 = 0;
  back.cap = c->cap;
  ck(cudaMemcpyAsync(c->ctrl, &back, sizeof(Ctrl), cudaMemcpyHostToDevice,
                     c->stream),
     "restore ctrl");
}

constexpr int64_t kChunk = 256;

// Runs `steps` steps as one device-resident chunk. Returns false when the
// list overflowed (state is then garbage; the caller rolls back).
constexpr int kGraphSteps = 15;  // odd: the ping-pong parity is unchanged per graph

constexpr int kObsRows = kObsRowsAlloc;  // == kChunk: rows a chunk can record

void launch_obs_record(tmd_gpu_ctx* c) {
  if (c->obs_stride <= 0) return;
  c->launches += 1;
  k_obs_record<<<1, kRedThreads, 0, c->ls>>>(c->part_e, c->part_w, force_parts(c), c->part_ke,
                                             c->ke_parts, c->ctrl, c->obs_stride, c->obs_dev,
                                             kObsRows);
}

// End of a run segment: PE / virial / KE reduced and copied into the pinned
// host mirror, so observe() after a run needs neither a launch nor a sync.
void enqueue_observables(tmd_gpu_ctx* c) {
  launch_reduce_pe(c);
  if (c->variant == 2) {  // brick variant: its kinetic partials are per brick
    c->launches += 1;
    launch_kinetic(c);
  }
  launch_reduce_ke(c);
  ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                     c->ls), "D2H scalars");
}

// Captures one block of `nsteps` steps (odd; starting at buffer parity
// c->cur) as a CUDA graph whose rebuild branches are conditional IF nodes.
// Splitting a run into such blocks is bitwise identical to the eager
// sequence: the closing and opening half-kicks are the same two roundings
// whether they run in one fused epilogue or in two kernels.
void capture_graph_body(tmd_gpu_ctx* c, int nsteps, cudaGraph_t g, tmd_gpu_ctx::StepGraph& out);

void capture_graph(tmd_gpu_ctx* c, int nsteps, tmd_gpu_ctx::StepGraph& out) {
  cudaGraph_t g = nullptr;
  ck(cudaGraphCreate(&g, 0), "cudaGraphCreate");
  const int p = c->cur;
  const uint64_t l0 = c->launches;
  try {
    capture_graph_body(c, nsteps, g, out);
  } catch (...) {
    // leave no stream in capture mode and no half-built graph behind
    cudaStreamCaptureStatus st;
    cudaGraph_t junk = nullptr;
    if (cudaStreamIsCapturing(c->side, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(c->side, &junk);
    }
    if (cudaStreamIsCapturing(c->stream, &st) == cudaSuccess &&
        st != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(c->stream, &junk);
    }
    cudaGetLastError();
    cudaGraphDestroy(g);
    out = tmd_gpu_ctx::StepGraph{};
    c->ls = c->stream;
    c->cond_handle = 0;
    c->cur = p;
    c->pos = c->posb[p];
    c->launches = l0;
    throw;
  }
}

void capture_graph_body(tmd_gpu_ctx* c, int nsteps, cudaGraph_t g,
                        tmd_gpu_ctx::StepGraph& out) {
  const int p = c->cur;
  const uint64_t l0 = c->launches;
  ck(cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal),
     "begin capture");
  c->ls = c->stream;
  launch_tick(c, kTickBlock, 0);
  launch_kick_drift(c);
  uint64_t body = 0;
  // Small systems: no conditional nodes (an IF node costs ~9 us per step on
  // B200, a kernel node that returns at once well under 1 us): the rebuild
  // kernels stay in the graph and return unless the step's decision is set
  // (the eager sequence).
  for (int s = 0; s < nsteps && !c->if_nodes; ++s) {
    launch_decide(c, true);
    launch_resort(c);
    launch_build(c);
    launch_tick(c, kTickForces, -1);
    launch_forces(c, s + 1 < nsteps ? kFused : kKick2);
    launch_obs_record(c);
  }
  for (int s = 0; s < nsteps && c->if_nodes; ++s) {
    cudaGraphConditionalHandle h;
    ck(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault),
       "cudaGraphConditionalHandleCreate");
    c->cond_handle = h;
    launch_decide(c, true);
    c->cond_handle = 0;
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    ck(cudaStreamGetCaptureInfo(c->stream, &st, nullptr, nullptr, &deps, &ndeps),
       "cudaStreamGetCaptureInfo");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    ck(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp), "cudaGraphAddNode(conditional)");
    const uint64_t b0 = c->launches;
    ck(cudaStreamBeginCaptureToGraph(c->side, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                     0, cudaStreamCaptureModeThreadLocal),
       "begin body capture");
    c->ls = c->side;
    launch_resort(c);
    launch_build(c);
    c->ls = c->stream;
    cudaGraph_t bodyg;
    ck(cudaStreamEndCapture(c->side, &bodyg), "end body capture");
    body = c->launches - b0;
    ck(cudaStreamUpdateCaptureDependencies(c->stream, &cnode, 1,
                                           cudaStreamSetCaptureDependencies),
       "cudaStreamUpdateCaptureDependencies");
    launch_tick(c, kTickForces, -1);
    launch_forces(c, s + 1 < nsteps ? kFused : kKick2);
    launch_obs_record(c);
  }
  enqueue_observables(c);
  ck(cudaStreamEndCapture(c->stream, &g), "end capture");
  cudaGraphExec_t exec = nullptr;
  ck(cudaGraphInstantiate(&exec, g, 0), "cudaGraphInstantiate");
  out.exec = exec;
  out.graph = g;
  c->graph_body_kernels = body;
  out.fixed = (c->launches - l0) - static_cast<uint64_t>(nsteps) * body;
  c->launches = l0;  // capture enqueued nothing
  if (c->cur != p) throw CudaFail{"graph capture changed the buffer parity"};
}

// ---- speculative graph mode ------------------------------------------------
// A run is a sequence of cycles: a block of K steps (kick1 + drift, then per
// step k_decide_spec1 + fused force kernel; no conditional node) and one
// closing step (k_decide + resort + list build, gated on the decision, +
// forces with the closing kick). A rebuild due inside the block halts it at
// that step: the block's remaining force launches only carry the positions
// to the other buffer (so the buffer parity after a block is known at
// capture), and the closing step performs the halted step. K is predicted
// so that the closing step lands on the next rebuild; a wrong guess costs
// only time, never results. One host sync per cycle (~9 steps) replaces a
// conditional IF node per step (~7 us each on B200, scripts/exp/if_cost.cu).
constexpr int kSpecMax = 24;

int spec_key(int K, int slot, int parity, bool observed) {
  return (K << 3) | (slot << 2) | (parity << 1) | (observed ? 1 : 0);
}

// One cycle as one graph: the block (K >= 1 steps), the status snapshot A
// (a copy of the status word into pinned memory + an event), the closing
// step (opening kick + drift too when K = 0), snapshot B.
void capture_spec(tmd_gpu_ctx* c, int K, int slot, tmd_gpu_ctx::StepGraph& out) {
  const bool open = K == 0;
  cudaGraph_t g = nullptr;
  ck(cudaGraphCreate(&g, 0), "cudaGraphCreate");
  const int p = c->cur;
  const uint64_t l0 = c->launches;
  auto restore_host = [&] {
    c->ls = c->stream;
    c->halt_copy = 0;
    c->cur = p;
    c->pos = c->posb[p];
    c->launches = l0;
  };
  try {
    ck(cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal), "begin capture");
    c->ls = c->stream;
    if (K > 0) {  // block
      launch_tick(c, kTickBlock, 0);
      launch_kick_drift(c);
      for (int s = 0; s < K; ++s) {
        c->launches += 1;
        k_decide_spec1<<<1, 1, 0, c->ls>>>(c->ctrl, c->g.rebuild_thr, tick_ptr(c));
        launch_tick(c, kTickForces, -1);
        c->halt_copy = 1;
        launch_forces(c, kFused);
        c->halt_copy = 0;
        launch_obs_record(c);
      }
    }
    ck(cudaMemcpyAsync(&c->h_ctrl_cyc[2 * slot], c->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost,
                       c->stream), "D2H ctrl");
    // (external: an event record node the host can wait on, not a capture
    // dependency marker)
    ck(cudaEventRecordWithFlags(c->ev_cyc[2 * slot], c->stream, cudaEventRecordExternal),
       "cudaEventRecord");
    {  // closing step: the rebuild kernels behind one IF node per cycle
      c->launches += 1;
      k_clear_halt<<<1, 1, 0, c->ls>>>(c->ctrl);
      if (open) {
        launch_tick(c, kTickBlock, 0);
        launch_kick_drift(c);
      }
      cudaGraphConditionalHandle h;
      ck(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault),
         "cudaGraphConditionalHandleCreate");
      c->cond_handle = h;
      launch_decide(c, true);
      c->cond_handle = 0;
      cudaStreamCaptureStatus st;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      ck(cudaStreamGetCaptureInfo(c->stream, &st, nullptr, nullptr, &deps, &ndeps),
         "cudaStreamGetCaptureInfo");
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      cudaGraphNode_t cnode;
      ck(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp), "cudaGraphAddNode(conditional)");
      const uint64_t b0 = c->launches;
      ck(cudaStreamBeginCaptureToGraph(c->side, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                       0, cudaStreamCaptureModeThreadLocal),
         "begin body capture");
      c->ls = c->side;
      launch_resort(c);
      launch_build(c);
      c->ls = c->stream;
      cudaGraph_t bodyg;
      ck(cudaStreamEndCapture(c->side, &bodyg), "end body capture");
      c->graph_body_kernels = c->launches - b0;
      c->launches = b0;  // (counted when the body runs)
      ck(cudaStreamUpdateCaptureDependencies(c->stream, &cnode, 1,
                                             cudaStreamSetCaptureDependencies),
         "cudaStreamUpdateCaptureDependencies");
      launch_tick(c, kTickForces, -1);
      launch_forces(c, kKick2);
      launch_obs_record(c);
      enqueue_observables(c);
    }
    ck(cudaMemcpyAsync(&c->h_ctrl_cyc[2 * slot + 1], c->ctrl, sizeof(Ctrl),
                       cudaMemcpyDeviceToHost, c->stream), "D2H ctrl");
    ck(cudaEventRecordWithFlags(c->ev_cyc[2 * slot + 1], c->stream, cudaEventRecordExternal),
       "cudaEventRecord");
    ck(cudaStreamEndCapture(c->stream, &g), "end capture");
    cudaGraphExec_t exec = nullptr;
    ck(cudaGraphInstantiate(&exec, g, 0), "cudaGraphInstantiate");
    out.exec = exec;
    out.graph = g;
    out.fixed = c->launches - l0;
  } catch (...) {
    cudaStreamCaptureStatus st;
    cudaGraph_t junk = nullptr;
    if (cudaStreamIsCapturing(c->side, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(c->side, &junk);
    }
    if (cudaStreamIsCapturing(c->stream, &st) == cudaSuccess &&
        st != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(c->stream, &junk);
    }
    cudaGetLastError();
    cudaGraphDestroy(g);
    out = tmd_gpu_ctx::StepGraph{};
    c->cond_handle = 0;
    restore_host();
    throw;
  }
  restore_host();  // capture ran nothing: host state as before
}

tmd_gpu_ctx::StepGraph& spec_graph(tmd_gpu_ctx* c, int K, int slot, int parity) {
  const bool observed = c->obs_stride > 0;
  if (!c->h_ctrl_cyc) {
    c->h_ctrl_cyc = static_cast<Ctrl*>(pinned_small(4 * sizeof(Ctrl)));
    for (auto& e : c->ev_cyc) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ev");
  }
  tmd_gpu_ctx::StepGraph& g = c->spec[spec_key(K, slot, parity, observed)];
  if (!g.exec) {
    const int keep = c->cur;
    c->cur = parity;
    c->pos = c->posb[parity];
    try {
      capture_spec(c, K, slot, g);
    } catch (...) {
      c->cur = keep;
      c->pos = c->posb[keep];
      throw;
    }
    c->cur = keep;
    c->pos = c->posb[keep];
  }
  return g;
}

// Steps of the next block: the closing step aimed at the step whose decision
// is predicted to rebuild (right after a rebuild: the last interval; later:
// the displacement the last decision saw, extrapolated ballistically).
int64_t spec_block(const tmd_gpu_ctx* c, int64_t done_step, int64_t left, double m) {
  int64_t k = kSpecMax;
  if (c->last_rebuild_step >= 0) {
    const int64_t t = done_step - c->last_rebuild_step;
    const double thr = c->g.rebuild_thr;
    if (t <= 0 || !(m > 0.0)) {
      if (c->rebuild_gap > 0) k = c->rebuild_gap - 1 - std::max<int64_t>(t, 0);
    } else {
      k = static_cast<int64_t>(std::ceil(static_cast<double>(t) * std::sqrt(thr / m))) - t - 1;
    }
  }
  return std::max<int64_t>(0, std::min<int64_t>({k, kSpecMax, left - 1}));
}

// Enqueues `steps` steps without graphs: kick1+drift, then per step decide,
// (gated) resort + list build, forces + fused integrator; PE reduction.
void enqueue_segment(tmd_gpu_ctx* c, int64_t steps) {
  {
    Phase p(c, TMD_SECTION_INTEGRATE);
    launch_kick_drift(c);
  }
  for (int64_t s = 0; s < steps; ++s) {
    {
      Phase p(c, TMD_SECTION_NEIGH);
      launch_decide(c, true, static_cast<int>(s));
    }
    {
      Phase p(c, TMD_SECTION_RESORT, static_cast<int>(s));
      launch_resort(c);
    }
    {
      Phase p(c, TMD_SECTION_NEIGH);
      launch_build(c);
    }
    {
      // forces + fused velocity-Verlet epilogue (closing half-kick of this
      // step and, unless it is the last step of the chunk, the opening
      // half-kick + drift of the next); booked to Forces
      Phase p(c, TMD_SECTION_FORCES);
      launch_forces(c, s + 1 < steps ? kFused : kKick2);
    }
    launch_obs_record(c);
  }
  enqueue_observables(c);
}

bool run_chunk(tmd_gpu_ctx* c, int64_t steps) {
  const bool graphs = c->use_graphs;
  if (c->obs_stride > 0) {
    ck(cudaMemsetAsync(&c->ctrl->obs_rows, 0, sizeof(int), c->stream), "memset obs rows");
  }
  if (graphs && c->spec_mode && c->variant >= 2) {  // (these force kernels honour halt)
    if (c->graph_dirty) drop_graphs(c);
    if (c->obs_stride > 0 && c->sgo_stride != c->obs_stride) {
      drop_spec_graphs(c, true);  // the stride is a kernel argument of the observed graphs
      c->sgo_stride = c->obs_stride;
    }
    if (tick_ptr(c)) {
      const long long base = c->step;
      ck(cudaMemsetAsync(c->ticks, 0, sizeof(long long) * (kTickSteps * kTickPhases + 1),
                         c->stream), "memset ticks");
      ck(cudaMemcpyAsync(&c->ctrl->tick_base, &base, sizeof base, cudaMemcpyHostToDevice,
                         c->stream), "H2D tick base");
    }
    // Each cycle leaves two status snapshots in pinned memory: A after the
    // block, B after the closing step. A tells the host exactly what the
    // closing step will do (the block halted, or the displacement it left
    // exceeds the threshold: a rebuild), so the next cycle is planned and
    // enqueued while the closing step still runs — the GPU does not wait for
    // the host — and B, read after that, carries the closing step's status
    // (list overflow).
    int64_t done = c->step;
    const int64_t target = c->step + steps;
    if (c->last_rebuild_step < 0) c->last_rebuild_step = done;
    double seen = c->h_ctrl->seen_d2;
    long long rebuilds = c->h_ctrl->rebuilds;
    // cycle i uses snapshots / events [2 (i % 2)] (A) and [2 (i % 2) + 1] (B)
    auto launch_cycle = [&](int K, int slot) {
      tmd_gpu_ctx::StepGraph& g = spec_graph(c, K, slot, c->cur);
      ck(cudaGraphLaunch(g.exec, c->stream), "cudaGraphLaunch");
      c->launches += g.fixed;
      c->cur ^= K & 1;
      c->pos = c->posb[c->cur];
    };
    int K = static_cast<int>(spec_block(c, done, target - done, seen));
    int slot = 0;
    launch_cycle(K, slot);
    static const bool spec_log = std::getenv("TMD_SPEC_LOG") != nullptr;  // (diagnostics)
    auto note_step = [&](int64_t now, bool rebuilt, double m) {
      if (spec_log) {
        std::fprintf(stderr, "[spec] K=%d steps %lld..%lld rebuilt=%d m=%.4g\n", K,
                     static_cast<long long>(done), static_cast<long long>(now), rebuilt ? 1 : 0, m);
      }
      done = now;
      if (rebuilt) {
        c->rebuild_gap = done - c->last_rebuild_step;
        c->last_rebuild_step = done;
        seen = 0.0;
      } else {
        seen = m;
      }
    };
    for (;;) {
      // A (after the block): with K > 0 it fixes what the closing step does
      // (halted, or the displacement the block left exceeds the threshold:
      // a rebuild), so the next cycle goes in while the closing step runs.
      // With K = 0 the closing step's own kick and drift come after A: its
      // outcome is read from B before the next cycle is planned.
      ck(cudaEventSynchronize(c->ev_cyc[2 * slot]), "cudaEventSynchronize");
      const Ctrl a = c->h_ctrl_cyc[2 * slot];
      if (a.status & kOverflowBits) break;  // (rolled back by the caller)
      if (a.step < done || a.step - done > K) throw CudaFail{"speculative block: step count"};
      int K_next = -1;
      const bool known = K > 0;
      if (known) {
        const double m = __builtin_bit_cast(double, a.max_d2);
        note_step(a.step + 1, a.halt != 0 || a.force_rebuild != 0 || m > c->g.rebuild_thr, m);
        if (done < target) {
          K_next = static_cast<int>(spec_block(c, done, target - done, seen));
          launch_cycle(K_next, slot ^ 1);
        }
      }
      ck(cudaEventSynchronize(c->ev_cyc[2 * slot + 1]), "cudaEventSynchronize");
      const Ctrl b = c->h_ctrl_cyc[2 * slot + 1];
      *c->h_ctrl = b;
      if (b.status & kOverflowBits) break;
      if (!known) {
        note_step(b.step, b.rebuilds != rebuilds, b.seen_d2);
        if (done < target) {
          K_next = static_cast<int>(spec_block(c, done, target - done, seen));
          launch_cycle(K_next, slot ^ 1);
        }
      }
      if (b.step != done) throw CudaFail{"speculative block: closing step count"};
      if (b.rebuilds != rebuilds) {  // (only the closing step rebuilds)
        c->launches += static_cast<uint64_t>(b.rebuilds - rebuilds) * c->graph_body_kernels;
        rebuilds = b.rebuilds;
      }
      if (K_next < 0) break;
      K = K_next;
      slot ^= 1;
    }
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");  // (overflow: drain)
    if (tick_ptr(c)) {
      c->launches += 1;
      k_tick<<<1, 1, 0, c->stream>>>(c->ctrl, c->ticks, 0, 0, kTickSteps * kTickPhases);
      c->h_ticks.resize(kTickSteps * kTickPhases + 1);
      ck(cudaMemcpyAsync(c->h_ticks.data(), c->ticks, sizeof(long long) * c->h_ticks.size(),
                         cudaMemcpyDeviceToHost, c->stream), "D2H ticks");
    }
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    sync_ctrl(c);
    const bool ok = (c->h_ctrl->status & kOverflowBits) == 0;
    if (ok && tick_ptr(c)) harvest_ticks(c, steps);
    return ok;
  }
  if (graphs) {
    if (c->graph_dirty) drop_graphs(c);
    if (tick_ptr(c)) {
      const long long base = c->step;
      ck(cudaMemsetAsync(c->ticks, 0, sizeof(long long) * (kTickSteps * kTickPhases + 1),
                         c->stream), "memset ticks");
      ck(cudaMemcpyAsync(&c->ctrl->tick_base, &base, sizeof base, cudaMemcpyHostToDevice,
                         c->stream), "H2D tick base");
    }
    const long long rebuilds0 = c->h_ctrl->rebuilds;
    int64_t left = steps;
    while (left > 0) {
      const int kind = left >= kGraphSteps ? 0 : 1;  // block of 15, or single steps
      if (c->obs_stride > 0 && c->sgo_stride != c->obs_stride) {
        // the stride is a kernel argument baked into the observed graphs
        for (auto& row : c->sgo) {
          for (auto& sg : row) {
            if (sg.exec) cudaGraphExecDestroy(sg.exec);
            if (sg.graph) cudaGraphDestroy(sg.graph);
            sg = tmd_gpu_ctx::StepGraph{};
          }
        }
        c->sgo_stride = c->obs_stride;
      }
      tmd_gpu_ctx::StepGraph& sgr = (c->obs_stride > 0 ? c->sgo : c->sg)[kind][c->cur];
      if (!sgr.exec) capture_graph(c, kind == 0 ? kGraphSteps : 1, sgr);
      ck(cudaGraphLaunch(sgr.exec, c->stream), "cudaGraphLaunch");
      c->launches += sgr.fixed;
      left -= kind == 0 ? kGraphSteps : 1;
    }
    if (tick_ptr(c)) {
      c->launches += 1;
      k_tick<<<1, 1, 0, c->stream>>>(c->ctrl, c->ticks, 0, 0, kTickSteps * kTickPhases);
      c->h_ticks.resize(kTickSteps * kTickPhases + 1);
      ck(cudaMemcpyAsync(c->h_ticks.data(), c->ticks, sizeof(long long) * c->h_ticks.size(),
                         cudaMemcpyDeviceToHost, c->stream), "D2H ticks");
    }
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    sync_ctrl(c);
    c->launches += static_cast<uint64_t>(c->h_ctrl->rebuilds - rebuilds0) *
                   c->graph_body_kernels;
    const bool ok = (c->h_ctrl->status & kOverflowBits) == 0;
    if (ok && tick_ptr(c)) harvest_ticks(c, steps);
    return ok;
  }
  enqueue_segment(c, steps);
  if (c->timers_on) {
    c->h_rebuild_log.resize(static_cast<size_t>(steps));
    ck(cudaMemcpyAsync(c->h_rebuild_log.data(), c->rebuild_log,
                       sizeof(int) * static_cast<size_t>(steps),
                       cudaMemcpyDeviceToHost, c->stream),
       "D2H rebuild log");
  }
  ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
  sync_ctrl(c);
  harvest_timers(c);
  return (c->h_ctrl->status & kOverflowBits) == 0;
}

// Runs nsteps in device-resident chunks. A checkpoint (positions,
// velocities, masses, ids; forces with a thermostat) is taken every kChunk
// steps, not every call, so a loop of run(1) calls pays for it once per
// kChunk steps. A list or staging overflow rolls back to the checkpoint,
// grows, and replays everything since (at most kChunk steps).
void do_run(tmd_gpu_ctx* c, int64_t nsteps) {
  const int64_t target = c->step + nsteps;
  while (c->step < target) {
    if (!c->ck_valid || c->step - c->ck_step >= kChunk) {
      checkpoint(c);
      c->ck_ctrl = *c->h_ctrl;  // mirror is current after the last sync
      c->ck_step = c->step;
      c->ck_valid = true;
    }
    const int64_t todo = std::min(kChunk - (c->step - c->ck_step), target - c->step);
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    const bool ok = run_chunk(c, todo);  // records t1 and synchronises
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->t0, c->t1), "cudaEventElapsedTime");
    c->elapsed += 1e-3 * ms;
    if (!ok) {
      // list or staging overflow: roll back, grow, replay from the checkpoint
      const Ctrl h = *c->h_ctrl;
      restore(c, c->ck_ctrl);
      c->step = c->ck_step;
      c->rebuilds = static_cast<uint64_t>(c->ck_ctrl.rebuilds);
      grow_after_overflow(c, h);
      if (c->th.on) {
        // the restored forces hold the Langevin kick of the checkpoint step
        // (not recomputable): keep them and rebuild at the replay's first
        // step instead of re-running the setup pass (force_rebuild = 2: a
        // rebuild that is not counted as one of the reference's)
        const int two = 2;
        ck(cudaMemcpyAsync(&c->ctrl->force_rebuild, &two, sizeof(int), cudaMemcpyHostToDevice,
                           c->stream), "cudaMemcpyAsync(force_rebuild)");
        sync_ctrl(c);
      } else {
        setup_pass(c);
      }
      continue;
    }
    c->step = c->h_ctrl->step;
    c->rebuilds = static_cast<uint64_t>(c->h_ctrl->rebuilds);
    c->ke_fresh = true;
    c->obs_fresh = true;
    if (c->obs_stride > 0) {  // rows landed in mapped host memory during the chunk
      const int rows = std::min(c->h_ctrl->obs_rows, kObsRows);
      for (int r = 0; r < rows; ++r) {
        const double* o = c->obs_host + 4 * r;
        c->obs_rows.push_back({o[0], o[1], o[2], o[3]});
      }
    }
    raise_physics(c, true);
  }
}

template <class F>
int guard(tmd_gpu_ctx* c, F&& fn) {
  try {
    fn();
    return TMD_OK;
  } catch (const StatusError& e) {
    c->err = e.what;
    return e.code;
  } catch (const CudaFail& e) {
    c->err = e.what;
    return TMD_ERR_CUDA;
  } catch (const std::exception& e) {
    c->err = e.what();
    return TMD_ERR_CUDA;
  }
}

// ---- validation (build_domain's checks, domain.hpp:134-168, in its order:
// validate_flat = box, then per particle in input order a duplicate id or a
// non-positive mass, then the topology's ids (flat_config.hpp:42-61,
// topology.hpp:33-52); then the interaction / skin / bond-reach / sentinel
// checks, the cell grid, and the Engine ctor's validate_engine_config).

[[noreturn]] void cfg_error(const std::string& m) { throw StatusError{TMD_ERR_CONFIG, m}; }

// Arguments the reference cannot get wrong (null arrays, sizes).
void validate_args(const tmd_system* s, const tmd_lj_params* lj, const tmd_engine_params* p) {
  if (!s || !lj || !p) cfg_error("null argument");
  if (s->n < 0) cfg_error("negative particle count");
  if (s->n > kMaxSlots) {
    cfg_error("system too large for one GPU context: " + std::to_string(s->n) +
              " particles > " + std::to_string(kMaxSlots));
  }
  if (s->n > 0 && (!s->id || !s->pos)) cfg_error("id and pos arrays are required");
  if (s->n_bonds < 0 || (s->n_bonds > 0 && !s->bonds)) cfg_error("bond array missing");
}

// validate_box (box.hpp:21-29)
void validate_box3(const double box[3]) {
  for (int k = 0; k < 3; ++k) {
    if (!std::isfinite(box[k]) || box[k] <= 0.0) {
      cfg_error("box lengths must be finite and positive, got " + fmt_g(box[k]));
    }
  }
}

// Everything after validate_flat that needs no per-particle pass.
void validate_params(const tmd_system* s, const tmd_lj_params* lj,
                     const tmd_fene_params* fene, const tmd_engine_params* p) {
  // validate_lj (potentials.hpp:28-38)
  if (!(lj->epsilon > 0.0) || !std::isfinite(lj->epsilon))
    cfg_error("lj epsilon must be finite and positive");
  if (!(lj->sigma > 0.0) || !std::isfinite(lj->sigma))
    cfg_error("lj sigma must be finite and positive");
  if (!(lj->r_cut > 0.0) || !std::isfinite(lj->r_cut))
    cfg_error("lj r_cut must be finite and positive");
  if (fene) {  // validate_fene (potentials.hpp:84-91)
    if (!(fene->k > 0.0) || !std::isfinite(fene->k)) cfg_error("fene k must be finite and positive");
    if (!(fene->r_max > 0.0) || !std::isfinite(fene->r_max))
      cfg_error("fene r_max must be finite and positive");
  }
  if (!std::isfinite(p->r_skin) || p->r_skin < 0.0)
    cfg_error("skin radius must be finite and non-negative");
  if (s->n_bonds > 0 && !fene) cfg_error("topology has bonds but no bond parameters configured");
  if (s->n_bonds > 0 && fene->r_max > lj->r_cut + p->r_skin) {
    cfg_error("bond r_max exceeds r_cut + r_skin; bonded partners could leave the ghost shell");
  }
  // build_domain's sentinel guard (domain.hpp:162-168), kept for parity of
  // accepted inputs
  const double max_len = std::max({s->box[0], s->box[1], s->box[2]});
  if (max_len > 0.1 * 1.0e9) {
    cfg_error("box too large: positions could alias the padding sentinel coordinate");
  }
}

// validate_engine_config (engine.hpp:28-41) + the GPU path's own knob.
void validate_engine(const tmd_engine_params* p) {
  if (!std::isfinite(p->dt) || p->dt == 0.0) cfg_error("time step must be finite and nonzero");
  if (p->thermostat) {  // validate_langevin (potentials.hpp:180-189)
    if (!(p->gamma >= 0.0) || !std::isfinite(p->gamma))
      cfg_error("langevin gamma must be finite and >= 0");
    if (!(p->temperature >= 0.0) || !std::isfinite(p->temperature))
      cfg_error("langevin temperature must be finite and >= 0");
  }
  if (!std::isfinite(p->force_cap) || p->force_cap < 0.0) {
    cfg_error("force cap must be finite and non-negative");
  }
}

// Splits [0, n) over up to 16 host threads (chunks of >= 1M particles).
template <class F>
void parallel_chunks(int64_t n, F&& fn) {
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t T = std::min<int64_t>(std::min<int64_t>(hw, 16), std::max<int64_t>(1, n >> 20));
  if (T <= 1) {
    fn(0, int64_t{0}, n);
    return;
  }
  std::vector<std::thread> ts;
  for (int64_t t = 0; t < T; ++t) {
    ts.emplace_back([&, t] { fn(static_cast<int>(t), n * t / T, n * (t + 1) / T); });
  }
  for (auto& t : ts) t.join();
}

struct IdRange {
  int64_t lo = 0, hi = -1;
  bool dense = false;  // hi - lo < n: a bitmap over [lo, hi] decides uniqueness
};

IdRange id_range(const tmd_system* s) {
  IdRange r;
  if (s->n <= 0) return r;
  std::vector<std::pair<int64_t, int64_t>> part(16, {INT64_MAX, INT64_MIN});
  parallel_chunks(s->n, [&](int t, int64_t b, int64_t e) {
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    for (int64_t k = b; k < e; ++k) {
      lo = std::min(lo, static_cast<int64_t>(s->id[k]));
      hi = std::max(hi, static_cast<int64_t>(s->id[k]));
    }
    part[static_cast<size_t>(t)] = {lo, hi};
  });
  r.lo = INT64_MAX;
  r.hi = INT64_MIN;
  for (const auto& p : part) {
    r.lo = std::min(r.lo, p.first);
    r.hi = std::max(r.hi, p.second);
  }
  r.dense = static_cast<uint64_t>(r.hi - r.lo) < static_cast<uint64_t>(s->n);
  return r;
}

// validate_flat's per-particle checks + validate_topology, serially in the
// reference's order (the first failing particle in input order; then the
// first failing bond). Throws the reference's message.
void validate_particles_exact(const tmd_system* s, const IdRange& r) {
  std::vector<unsigned char> seen;
  std::unordered_set<int64_t> set;
  if (r.dense) {
    seen.assign(static_cast<size_t>(s->n), 0);
  } else {
    set.reserve(static_cast<size_t>(s->n));
  }
  for (int64_t k = 0; k < s->n; ++k) {
    const int64_t id = s->id[k];
    bool dup;
    if (r.dense) {
      unsigned char& b = seen[static_cast<size_t>(id - r.lo)];
      dup = b != 0;
      b = 1;
    } else {
      dup = !set.insert(id).second;
    }
    if (dup) cfg_error("duplicate particle id " + std::to_string(id));
    if (s->mass && !(s->mass[k] > 0.0)) {
      cfg_error("particle id " + std::to_string(id) + " has non-positive mass");
    }
  }
  auto known = [&](int64_t v) {
    if (r.dense) return v >= r.lo && v <= r.hi && seen[static_cast<size_t>(v - r.lo)] != 0;
    return set.count(v) != 0;
  };
  for (int64_t k = 0; k < s->n_bonds; ++k) {
    const int64_t a = s->bonds[2 * k], b = s->bonds[2 * k + 1];
    const bool ha = known(a), hb = known(b);
    if (!ha || !hb) cfg_error("bond references unknown particle id " + std::to_string(ha ? b : a));
    if (a == b) cfg_error("bond connects particle id " + std::to_string(a) + " to itself");
  }
}

// The same checks as a parallel pass that only answers "all good?" (a
// failure re-runs validate_particles_exact for the reference's message).
bool particles_ok_fast(const tmd_system* s, const IdRange& r) {
  if (s->n <= 0) return s->n_bonds == 0;
  std::atomic<bool> bad{false};
  std::vector<uint64_t> bits;
  std::vector<int64_t> sorted;
  if (r.dense) {
    bits.assign(static_cast<size_t>((s->n + 63) / 64), 0ull);
  } else {
    sorted.assign(s->id, s->id + s->n);
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) return false;
  }
  // dense ids: a bitmap over [lo, lo + n) with plain (racy) ORs — a bit lost
  // to a race between threads, like a duplicate, leaves fewer than n bits
  // set, and either sends the caller to the exact serial pass
  parallel_chunks(s->n, [&](int, int64_t b, int64_t e) {
    bool my_bad = false;
    for (int64_t k = b; k < e; ++k) {
      if (r.dense) {
        const uint64_t idx = static_cast<uint64_t>(s->id[k] - r.lo);
        const uint64_t bit = 1ull << (idx & 63);
        uint64_t& w = bits[idx >> 6];
        my_bad |= (w & bit) != 0;
        w |= bit;
      }
      if (s->mass) my_bad |= !(s->mass[k] > 0.0);
    }
    if (my_bad) bad.store(true, std::memory_order_relaxed);
  });
  if (bad.load()) return false;
  if (r.dense) {
    std::atomic<int64_t> set{0};
    const int64_t nw = static_cast<int64_t>(bits.size());
    parallel_chunks(nw << 6, [&](int, int64_t b, int64_t e) {
      int64_t cnt = 0;
      for (int64_t w = b >> 6; w < (e >> 6); ++w) cnt += __builtin_popcountll(bits[static_cast<size_t>(w)]);
      set.fetch_add(cnt, std::memory_order_relaxed);
    });
    if (set.load() != s->n) return false;
  }
  for (int64_t k = 0; k < s->n_bonds; ++k) {
    const int64_t a = s->bonds[2 * k], b = s->bonds[2 * k + 1];
    for (int64_t v : {a, b}) {
      const bool ok = r.dense ? (v >= r.lo && v <= r.hi &&
                                 ((bits[static_cast<size_t>(v - r.lo) >> 6] >>
                                   (static_cast<uint64_t>(v - r.lo) & 63)) & 1ull))
                              : std::binary_search(sorted.begin(), sorted.end(), v);
      if (!ok) return false;
    }
    if (a == b) return false;
  }
  return true;
}

// Brick decomposition of the cell grid (bricks of up to 2x2x2 cells), the
// brick-major cell ranks, staging capacities and the FP32 prefilter band.


void setup_bricks(tmd_gpu_ctx* c, double n, double r_verlet) {
  BrickGeom& bg = c->bg;
  // bricks tile the OWNED cells (local z offset 1 in slab mode)
  const int ext[3] = {c->g.dims[0], c->g.dims[1], c->g.zown};
  const int zoff = c->g.zslab ? 1 : 0;
  // 2 x 2 x kBrickZ cells while that still gives every SM three bricks to
  // build at once (staging amortised over 16 own cells: -7 % per build at
  // 16.4M); 2 x 2 x 2 for small systems, whose builds are latency-bound
  const int nb4 = ((ext[0] + 1) / 2) * ((ext[1] + 1) / 2) * ((ext[2] + kBrickZ - 1) / kBrickZ);
  int bz = nb4 >= 148 * 3 ? kBrickZ : 2;
  if (const char* e = std::getenv("TMD_BRICK_Z")) bz = std::atoi(e) == 2 ? 2 : kBrickZ;  // (probes)
  for (int k = 0; k < 3; ++k) {
    bg.B[k] = std::min(k == 2 ? bz : 2, ext[k]);
    bg.nb[k] = (ext[k] + bg.B[k] - 1) / bg.B[k];
    bg.origin_scale[k] = c->g.cell_len[k];
  }
  bg.nbricks = bg.nb[0] * bg.nb[1] * bg.nb[2];
  (void)zoff;  // (the brick-major ranks are filled on the device: k_brick_tables)
  c->ngroups_max = static_cast<int>(n / 32.0) + bg.nbricks + 1;
  // staging capacity: twice the expected halo population, 32-aligned
  const double vol = c->g.L[0] * c->g.L[1] * c->g.L[2];
  const double per_cell = n / vol * c->g.cell_len[0] * c->g.cell_len[1] * c->g.cell_len[2];
  const double halo = per_cell * (bg.B[0] + 2) * (bg.B[1] + 2) * (bg.B[2] + 2);
  // expected halo + per-cell padding (<= 3 slots per cell) + 6 sigma, and
  // small enough that 5 force CTAs fit an SM; overfull halos grow it at run
  // time (setup_pass / do_run).
  const int ncell_halo = (bg.B[0] + 2) * (bg.B[1] + 2) * (bg.B[2] + 2);
  const double want = halo + 1.5 * ncell_halo + 6.0 * std::sqrt(halo) + 64.0;
  bg.stage_cap = std::max(256, (static_cast<int>(want) + 31) / 32 * 32);
  // FP32 prefilter band (see DESIGN.md §List build): bound on |r2_f32 - r2_ref|
  // for brick-relative single-precision coordinates, times 4.
  const double cl = std::max({c->g.cell_len[0], c->g.cell_len[1], c->g.cell_len[2]});
  const double Lm = std::max({c->g.L[0], c->g.L[1], c->g.L[2]});
  const double u32 = std::ldexp(1.0, -24), u64 = std::ldexp(1.0, -52);
  const double rv = r_verlet, rv2 = c->g.rv2;
  const double e_coord = u32 * 3.0 * cl * 1.01 + u64 * 4.0 * (2.0 * Lm + 4.0 * cl);
  const double e_d = 2.0 * e_coord + u32 * rv * 1.01;
  const double err = 2.0 * std::sqrt(3.0) * rv * 1.01 * e_d + 3.0 * e_d * e_d +
                     3.0 * u32 * rv2 * 1.01 + std::ldexp(rv2, -50);
  const double delta = 4.0 * err;
  bg.lo2 = std::nextafter(static_cast<float>(rv2 - delta), 0.0f);
  bg.hi2 = std::nextafter(static_cast<float>(rv2 + delta), 1e30f);
}

// Brick tables (cell -> brick-major rank, brick -> first rank), filled on the
// device (allocated here unless the context's arena already holds them).
void upload_bricks(tmd_gpu_ctx* c) {
  if (!c->cell_rank) {
    c->cell_rank = dalloc<int>(static_cast<size_t>(c->g.ncells));
    c->brick_rank_off = dalloc<int>(static_cast<size_t>(c->bg.nbricks) + 1);
    c->scan_tmp = dalloc<int>(static_cast<size_t>(
        blocks_for(std::max(c->g.ncells, c->bg.nbricks), kScanTile) + 1));
  }
  c->launches += 1;
  k_brick_tables<<<blocks_for(std::max(c->g.ncells, c->bg.nbricks + 1), kBlock), kBlock, 0,
                   c->stream>>>(c->g, c->bg, c->cell_rank, c->brick_rank_off);
  ck(cudaGetLastError(), "k_brick_tables");
  set_smem_attrs(c);
}

void build_geom(tmd_gpu_ctx* c, const double box[3], double r_cut,
                double r_skin) {
  // build_cell_grid (cell_grid.hpp:54-78)
  const double r_verlet = r_cut + r_skin;
  for (int k = 0; k < 3; ++k) {
    if (box[k] < r_verlet) {
      throw StatusError{TMD_ERR_CONFIG,
                        "box length " + std::to_string(box[k]) +
                            " is smaller than one cell (r_cut + r_skin = " +
                            std::to_string(r_verlet) + ")"};
    }
    c->g.L[k] = box[k];
    c->g.dims[k] = std::max(1, static_cast<int>(std::floor(box[k] / r_verlet)));
  }
  for (int k = 0; k < 3; ++k) c->g.cell_len[k] = box[k] / c->g.dims[k];
  const int64_t nc = static_cast<int64_t>(c->g.dims[0]) * c->g.dims[1] * c->g.dims[2];
  if (nc > (int64_t{1} << 30)) {
    throw StatusError{TMD_ERR_CONFIG, "cell grid too large"};
  }
  c->g.ncells = static_cast<int>(nc);
  c->g.rv2 = r_verlet * r_verlet;
  c->g.rebuild_thr = 0.25 * r_skin * r_skin;
  // whole periodic box (slab mode is set up by make_slab)
  c->g.zslab = 0;
  c->g.z0 = 0;
  c->g.zown = c->g.dims[2];
  c->g.ldz = c->g.dims[2];
  c->g.zcode_lo = c->g.zcode_hi = 0;
  c->g.owned_cells = c->g.ncells;
}

// The slab's local grid for owned global z layers [z0, z1): local layer
// lz = global - z0 + 1, ghost layers 0 and zown + 1.
void set_slab_range(tmd_gpu_ctx* c, int z0, int z1) {
  const int dz = c->g.dims[2];
  const int dxy = c->g.dims[0] * c->g.dims[1];
  c->g.zslab = 1;
  c->g.z0 = z0;
  c->g.zown = z1 - z0;
  c->g.ldz = c->g.zown + 2;
  c->g.zcode_lo = z0 == 0 ? 2u : 0u;   // lower ghost layer wraps: image at -Lz
  c->g.zcode_hi = z1 == dz ? 1u : 0u;  // upper ghost layer wraps: image at +Lz
  c->g.ncells = dxy * c->g.ldz;
  c->g.owned_cells = dxy * c->g.zown;
}

// Cut planes of the reference's range rule i*dims/s (decomp.hpp:87-93).
std::vector<int> default_cuts(int dz, int nranks) {
  std::vector<int> cuts(static_cast<size_t>(nranks) + 1);
  for (int r = 0; r <= nranks; ++r) {
    cuts[static_cast<size_t>(r)] = static_cast<int>(static_cast<int64_t>(r) * dz / nranks);
  }
  return cuts;
}

// Slab `rank` of `nranks` along z with the default cuts, plus one ghost
// layer on each side.
void make_slab(tmd_gpu_ctx* c, int rank, int nranks) {
  const int dz = c->g.dims[2];
  if (nranks > dz) {
    throw StatusError{TMD_ERR_CONFIG, "more ranks (" + std::to_string(nranks) +
                                          ") than z cell layers (" + std::to_string(dz) + ")"};
  }
  if (dz < 3) {
    throw StatusError{TMD_ERR_CONFIG,
                      "slab decomposition needs at least 3 z cell layers, the box has " +
                          std::to_string(dz)};
  }
  const std::vector<int> cuts = default_cuts(dz, nranks);
  set_slab_range(c, cuts[static_cast<size_t>(rank)], cuts[static_cast<size_t>(rank) + 1]);
}

void upload_owner_table(tmd_gpu_ctx* c, const std::vector<int>& cuts) {
  const int dz = c->g.dims[2];
  std::vector<int> owner(static_cast<size_t>(dz));
  for (int r = 0; r < c->nranks; ++r) {
    for (int z = cuts[static_cast<size_t>(r)]; z < cuts[static_cast<size_t>(r) + 1]; ++z) {
      owner[static_cast<size_t>(z)] = r;
    }
  }
  ck(cudaMemcpy(c->owner_of_z, owner.data(), owner.size() * sizeof(int),
                cudaMemcpyHostToDevice), "H2D owner table");
}

// Device buffers of the slab exchange.
void alloc_slab(tmd_gpu_ctx* c) {
  const size_t n = static_cast<size_t>(c->n_cap);
  c->owner_of_z = dalloc<int>(static_cast<size_t>(c->g.dims[2]));
  c->cuts = default_cuts(c->g.dims[2], c->nranks);
  upload_owner_table(c, c->cuts);
  c->mig_dest = dalloc<int>(n);
  c->exp = dalloc<int2>(n);
  c->mig_count = dalloc<int>(2 * static_cast<size_t>(c->nranks));
  c->mig_off = dalloc<int>(static_cast<size_t>(c->nranks) + 1);
  c->mig_keep = dalloc<int>(1);
  c->mig_send = dalloc<MigRec>(n);
  c->mig_recv = dalloc<MigRec>(n);
  const size_t dxy = static_cast<size_t>(c->g.dims[0]) * c->g.dims[1];
  for (int s = 0; s < 2; ++s) {
    c->bidx[s] = dalloc<int>(n);
    c->bids[s] = dalloc<long long>(n);
    c->bpos[s] = dalloc<double4>(n);
    c->bcnt[s] = dalloc<int>(dxy);
    c->boff[s] = dalloc<int>(dxy + 1);
    c->gcnt[s] = dalloc<int>(dxy);
  }
}

// Grows every per-slot array to hold `need` slots (slab mode: a slab's share
// changes with migration and re-cutting). Contents are preserved; the far
// sentinel moves to the new last slot.
void grow_capacity(tmd_gpu_ctx* c, int64_t need) {
  if (need <= c->n_cap) return;
  int64_t cap = std::max<int64_t>(need + need / 4 + 4096, c->n_cap * 3 / 2);
  cap = std::min<int64_t>(cap, kMaxSlots);
  if (need > cap) {
    throw StatusError{TMD_ERR_CONFIG, "slab too large for one GPU context: " +
                                          std::to_string(need) + " slots"};
  }
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  const size_t o = static_cast<size_t>(c->n_cap), nn = static_cast<size_t>(cap);
  auto regrow = [&](auto*& p, size_t extra) {
    using T = std::remove_reference_t<decltype(*p)>;
    if (!p) return;
    T* q = static_cast<T*>(sized_alloc((nn + extra) * sizeof(T)));
    ck(cudaMemcpy(q, p, o * sizeof(T), cudaMemcpyDeviceToDevice), "regrow copy");
    dev_free(p);
    p = q;
  };
  for (int b = 0; b < 2; ++b) regrow(c->posb[b], 1);
  c->pos = c->posb[c->cur];
  c->ipc_gen += 1;  // peers holding these buffers must re-map them
  regrow(c->pos2, 0); regrow(c->snap, 0);
  regrow(c->vx, 0); regrow(c->vy, 0); regrow(c->vz, 0);
  regrow(c->vx2, 0); regrow(c->vy2, 0); regrow(c->vz2, 0);
  regrow(c->fx, 0); regrow(c->fy, 0); regrow(c->fz, 0);
  regrow(c->mass, 0); regrow(c->mass2, 0); regrow(c->id, 0); regrow(c->id2, 0);
  regrow(c->cell, 0); regrow(c->cell2, 0); regrow(c->rank, 0); regrow(c->perm, 0);
  regrow(c->nnbr, 0);
  regrow(c->ck_pos, 0); regrow(c->ck_vx, 0); regrow(c->ck_vy, 0); regrow(c->ck_vz, 0);
  regrow(c->ck_mass, 0); regrow(c->ck_id, 0);
  regrow(c->ck_fx, 0); regrow(c->ck_fy, 0); regrow(c->ck_fz, 0);
  regrow(c->mig_dest, 0); regrow(c->mig_send, 0); regrow(c->mig_recv, 0);
  regrow(c->bnd_cnt, 0);
  regrow(c->exp, 0);
  if (c->bnd_ent) {  // kMaxBonds entries per slot
    uint32_t* q = dalloc<uint32_t>(nn * kMaxBonds);
    ck(cudaMemcpy(q, c->bnd_ent, o * kMaxBonds * sizeof(uint32_t), cudaMemcpyDeviceToDevice),
       "regrow copy");
    cudaFree(c->bnd_ent);
    c->bnd_ent = q;
  }
  for (int s = 0; s < 2; ++s) {
    regrow(c->bidx[s], 0);
    regrow(c->bids[s], 0);
    regrow(c->bpos[s], 0);
  }
  const double4 far = make_double4(kFarD, kFarD, kFarD, 0.0);
  for (int b = 0; b < 2; ++b) {
    ck(cudaMemcpy(c->posb[b] + nn, &far, sizeof(double4), cudaMemcpyHostToDevice),
       "H2D sentinel");
  }
  const int parts = std::max({blocks_for(cap, kBlock), blocks_for(cap, kLanesPPB), c->bg.nbricks});
  if (parts > c->nparts) {
    cudaFree(c->part_e); cudaFree(c->part_w); cudaFree(c->part_ke);
    c->nparts = parts;
    c->part_e = dalloc<double>(parts);
    c->part_w = dalloc<double>(parts);
    c->part_ke = dalloc<double>(parts);
  }
  c->n_cap = cap;
  c->stride = static_cast<int>((cap + 31) / 32 * 32);
  c->graph_dirty = true;
}

// Moves this slab to owned layers [cuts[rank], cuts[rank+1]) (all ranks pass
// the same cuts, before the next migrate_out): new owner table, local grid,
// brick tables and cell-range arrays.
void recut(tmd_gpu_ctx* c, const std::vector<int>& cuts) {
  const int z0 = cuts[static_cast<size_t>(c->my_rank)];
  const int z1 = cuts[static_cast<size_t>(c->my_rank) + 1];
  upload_owner_table(c, cuts);
  if (z0 == c->g.z0 && z1 - z0 == c->g.zown) return;
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  set_slab_range(c, z0, z1);
  void* old[] = {c->cell_rank, c->brick_rank_off, c->scan_tmp, c->count, c->start};
  for (void* p : old) {
    if (p) cudaFree(p);
  }
  c->cell_rank = c->brick_rank_off = c->scan_tmp = nullptr;
  c->count = c->start = nullptr;
  setup_bricks(c, static_cast<double>(c->n_total), c->r_cut + c->r_skin);
  const int64_t want = c->n + c->n / 4 + 1024;
  c->ngroups_max = static_cast<int>(want / 32) + c->bg.nbricks + 1;
  upload_bricks(c);
  c->count = dalloc<int>(static_cast<size_t>(c->g.ncells));
  c->start = dalloc<int>(static_cast<size_t>(c->g.ncells) + 1);
  ck(cudaMemset(c->count, 0, sizeof(int) * static_cast<size_t>(c->g.ncells)), "memset count");
  if (c->bg.nbricks > c->nparts) {
    cudaFree(c->part_e); cudaFree(c->part_w); cudaFree(c->part_ke);
    c->nparts = c->bg.nbricks;
    c->part_e = dalloc<double>(c->nparts);
    c->part_w = dalloc<double>(c->nparts);
    c->part_ke = dalloc<double>(c->nparts);
  }
  alloc_list(c, c->cap);  // group count changed
}

// Static bond table by id (the topology never changes): CSR over
// id - id_min with each bond listed at both ends, the first id of the pair
// being the anchor (the reference computes a bond in the subnode owning its
// first particle, bonded.hpp:124-141).
void setup_bonds(tmd_gpu_ctx* c, const tmd_system* sys, const tmd_fene_params* fene) {
  const int64_t* idp = sys->id;
  const long long id_min = *std::min_element(idp, idp + sys->n);
  const long long id_max = *std::max_element(idp, idp + sys->n);
  const int64_t span = static_cast<int64_t>(id_max - id_min) + 1;
  if (span > 4 * sys->n + 1024) {
    throw StatusError{TMD_ERR_CONFIG,
                      "bonded systems need particle ids in a dense range (max - min < 4 n)"};
  }
  // CSR over id - id_min, built on the device (sizes only cross to the host)
  const int64_t nb = sys->n_bonds;
  const size_t ns = static_cast<size_t>(span);
  long long* d_bonds = dalloc<long long>(static_cast<size_t>(2 * nb));
  int* deg = dalloc<int>(ns + 1);
  int* cur = dalloc<int>(ns + 1);
  int* bidx = dalloc<int>(static_cast<size_t>(2 * nb));
  int* bad = dalloc<int>(1);
  c->id_min = id_min;
  c->id_span = span;
  c->slot_of_id = dalloc<int>(ns);
  c->bond_off = dalloc<int>(ns + 1);
  c->bond_nbr = dalloc<int>(static_cast<size_t>(2 * nb));
  c->bond_anchor = dalloc<unsigned char>(static_cast<size_t>(2 * nb));
  c->bnd_cnt = dalloc<int>(static_cast<size_t>(c->n_cap));
  c->bnd_ent = dalloc<uint32_t>(static_cast<size_t>(c->n_cap) * kMaxBonds);
  auto release = [&] {
    cudaFree(d_bonds);
    cudaFree(deg);
    cudaFree(cur);
    cudaFree(bidx);
    cudaFree(bad);
  };
  try {
    cudaStream_t st = c->stream;
    ck(cudaMemcpyAsync(d_bonds, sys->bonds, sizeof(long long) * 2 * nb, cudaMemcpyHostToDevice,
                       st), "H2D bonds");
    ck(cudaMemsetAsync(deg, 0, sizeof(int) * (ns + 1), st), "memset");
    ck(cudaMemsetAsync(cur, 0, sizeof(int) * (ns + 1), st), "memset");
    const int big = 0x7fffffff;
    ck(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    const int gb = std::max(1, blocks_for(nb, kBlock));
    const int gs = std::max(1, blocks_for(span, kBlock));
    k_bond_degree<<<gb, kBlock, 0, st>>>(nb, d_bonds, id_min, deg);
    k_bond_maxdeg<<<gs, kBlock, 0, st>>>(static_cast<int>(span), deg, bad);
    size_t tmp_bytes = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg, c->bond_off,
                                     static_cast<int>(span + 1), st), "cub scan (size)");
    void* tmp = nullptr;
    ck(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)), "cudaMalloc(scan)");
    const cudaError_t se = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, c->bond_off,
                                                         static_cast<int>(span + 1), st);
    k_bond_fill<<<gb, kBlock, 0, st>>>(nb, d_bonds, id_min, c->bond_off, cur, bidx, c->bond_nbr,
                                       c->bond_anchor);
    k_bond_order<<<gs, kBlock, 0, st>>>(static_cast<int>(span), c->bond_off, bidx, c->bond_nbr,
                                        c->bond_anchor);
    ck(cudaMemsetAsync(c->bnd_cnt, 0, sizeof(int) * static_cast<size_t>(c->n_cap), st),
       "memset");
    int h_bad = big;
    ck(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    cudaFree(tmp);
    ck(se, "cub scan");
    ck(cudaGetLastError(), "bond table kernels");
    if (h_bad != big) {
      int d = 0;
      ck(cudaMemcpy(&d, deg + h_bad, sizeof(int), cudaMemcpyDeviceToHost), "D2H degree");
      throw StatusError{TMD_ERR_CONFIG, "particle id " + std::to_string(id_min + h_bad) +
                                            " has " + std::to_string(d) +
                                            " bonds; the GPU path allows " +
                                            std::to_string(kMaxBonds)};
    }
  } catch (...) {
    release();
    throw;
  }
  release();
  c->bt.on = 1;
  c->bt.k = fene->k;
  c->bt.rmax2 = fene->r_max * fene->r_max;  // fene_eval (potentials.hpp:98)
}

// Slab mode's view of the whole system on the device (a cached block):
// positions, velocities, masses, ids as the caller passed them, and the
// input-order indices of this rank's particles.
struct SlabStage {
  char* block = nullptr;
  size_t bytes = 0;
  const double* pos = nullptr;
  const double* vel = nullptr;   // nullptr: zero
  const double* mass = nullptr;  // nullptr: 1
  const long long* id = nullptr;
  const int* sel = nullptr;
  int64_t n_keep = 0;
  void release() {
    big_free(block, bytes);
    block = nullptr;
  }
  ~SlabStage() { release(); }
};

void stage_slab_selection(tmd_gpu_ctx* c, const tmd_system* sys, SlabStage& st) {
  const size_t n = static_cast<size_t>(sys->n);
  const int ni = static_cast<int>(n);
  size_t tb = 0;
  ck(cub::DeviceSelect::Flagged(nullptr, tb, static_cast<const int*>(nullptr),
                                static_cast<const unsigned char*>(nullptr),
                                static_cast<int*>(nullptr), static_cast<int*>(nullptr), ni,
                                c->stream), "cub select size");
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_pos = al(3 * n * sizeof(double)), b_vel = sys->vel ? b_pos : 0;
  const size_t b_mass = sys->mass ? al(n * sizeof(double)) : 0, b_id = al(n * sizeof(long long));
  const size_t b_idx = al(n * sizeof(int)), b_flag = al(n), b_cnt = 256;
  st.block = static_cast<char*>(
      big_alloc(b_pos + b_vel + b_mass + b_id + 2 * b_idx + b_flag + b_cnt + al(tb), &st.bytes));
  char* q = st.block;
  auto take = [&](size_t b) { char* r = q; q += b; return r; };
  double* pos = reinterpret_cast<double*>(take(b_pos));
  double* vel = sys->vel ? reinterpret_cast<double*>(take(b_vel)) : nullptr;
  double* mass = sys->mass ? reinterpret_cast<double*>(take(b_mass)) : nullptr;
  long long* id = reinterpret_cast<long long*>(take(b_id));
  int* idx = reinterpret_cast<int*>(take(b_idx));
  int* sel = reinterpret_cast<int*>(take(b_idx));
  unsigned char* flag = reinterpret_cast<unsigned char*>(take(b_flag));
  int* d_cnt = reinterpret_cast<int*>(take(b_cnt));
  void* tmp = take(al(tb));
  if (n > 0) {
    ck(cudaMemcpyAsync(pos, sys->pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "H2D pos");
    if (vel) {
      ck(cudaMemcpyAsync(vel, sys->vel, 3 * n * sizeof(double), cudaMemcpyHostToDevice,
                         c->stream), "H2D vel");
    }
    if (mass) {
      ck(cudaMemcpyAsync(mass, sys->mass, n * sizeof(double), cudaMemcpyHostToDevice, c->stream),
         "H2D mass");
    }
    ck(cudaMemcpyAsync(id, sys->id, n * sizeof(long long), cudaMemcpyHostToDevice, c->stream),
       "H2D id");
    k_iota_int<<<blocks_for(sys->n, kBlock), kBlock, 0, c->stream>>>(ni, idx);
    k_slab_flags<<<blocks_for(sys->n, kBlock), kBlock, 0, c->stream>>>(ni, pos, c->g, flag);
    ck(cub::DeviceSelect::Flagged(tmp, tb, idx, flag, sel, d_cnt, ni, c->stream),
       "cub select");
  }
  int cnt = 0;
  if (n > 0) {
    ck(cudaMemcpyAsync(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
  }
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  st.pos = pos;
  st.vel = vel;
  st.mass = mass;
  st.id = id;
  st.sel = sel;
  st.n_keep = cnt;
}

// The type column of the caller's FlatConfig, kept by id (see tmd_gpu_ctx).
void set_type_table(tmd_gpu_ctx* c, const tmd_system* sys, const IdRange& r) {
  c->type_id.clear();
  c->type_val.clear();
  const size_t n = static_cast<size_t>(sys->n);
  if (!sys->type || n == 0) return;
  if (std::all_of(sys->type, sys->type + n, [](int32_t t) { return t == 0; })) return;
  if (static_cast<unsigned long long>(r.hi - r.lo) == n - 1) {
    c->type_lo = r.lo;
    c->type_val.assign(n, 0);
    for (size_t k = 0; k < n; ++k) c->type_val[static_cast<size_t>(sys->id[k] - c->type_lo)] = sys->type[k];
    return;
  }
  std::vector<size_t> o(n);
  std::iota(o.begin(), o.end(), size_t{0});
  std::sort(o.begin(), o.end(), [&](size_t a, size_t b) { return sys->id[a] < sys->id[b]; });
  c->type_id.resize(n);
  c->type_val.resize(n);
  for (size_t k = 0; k < n; ++k) {
    c->type_id[k] = sys->id[o[k]];
    c->type_val[k] = sys->type[o[k]];
  }
}

int32_t type_of(const tmd_gpu_ctx* c, long long id) {
  if (c->type_val.empty()) return 0;
  if (c->type_id.empty()) return c->type_val[static_cast<size_t>(id - c->type_lo)];
  const auto it = std::lower_bound(c->type_id.begin(), c->type_id.end(), id);
  return c->type_val[static_cast<size_t>(it - c->type_id.begin())];
}

int create_impl(const tmd_system* sys, const tmd_lj_params* lj, const tmd_fene_params* fene,
                const tmd_engine_params* params, int rank, int nranks, bool slab,
                tmd_gpu_ctx** out) {
  if (!out) return TMD_ERR_CONFIG;
  *out = nullptr;
  auto* c = new tmd_gpu_ctx();
  const bool dbg = std::getenv("TMD_DEBUG_TIMING") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tmd create] %-24s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_prev).count());
    t_prev = t;
  };
  const int rc = guard(c, [&] {
    validate_args(sys, lj, params);
    validate_box3(sys->box);
    try {  // (ConfigErrors before any CUDA call)
      validate_params(sys, lj, fene, params);
      build_geom(c, sys->box, lj->r_cut, params->r_skin);
      validate_engine(params);
    } catch (const StatusError&) {
      // build_domain checks the particles (validate_flat) before these
      validate_particles_exact(sys, id_range(sys));
      throw;
    }
    mark("validate params");
    // The per-particle checks (id range, then validate_flat's checks on the
    // host threads; the exact serial pass only to name the reference's first
    // error) run on a helper thread while the device is set up and the
    // particle upload is enqueued: joined before anything reads their result,
    // and before any other error is reported, so a bad particle is still the
    // ConfigError the reference raises (a failing device init included).
    IdRange idr;
    std::exception_ptr verr;
    bool ids_iota = false;  // ids[k] == lo + k: generated on the device, not uploaded
    bool defer_vm = false;  // velocities / masses placed after the setup pass
    std::thread vthread([&] {
      try {
        idr = id_range(sys);
        if (!particles_ok_fast(sys, idr)) validate_particles_exact(sys, idr);
        if (idr.dense && sys->n > 0) {
          std::atomic<bool> iota{true};
          parallel_chunks(sys->n, [&](int, int64_t b, int64_t e) {
            for (int64_t k = b; k < e; ++k) {
              if (sys->id[k] != idr.lo + k) {
                iota = false;
                return;
              }
            }
          });
          ids_iota = iota;
        }
      } catch (...) {
        verr = std::current_exception();
      }
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{vthread};
    auto join_validation = [&] {
      if (vthread.joinable()) vthread.join();
      if (verr) {
        // (the upload reads the caller's arrays)
        if (c->stream) cudaStreamSynchronize(c->stream);
        if (c->side) cudaStreamSynchronize(c->side);
        std::rethrow_exception(verr);
      }
    };
    try {  // device setup (a particle error found meanwhile takes precedence)
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    mark("device count");
    if (ndev < 1) throw CudaFail{"no CUDA device"};
    if (params->device >= 0) {
      ck(cudaSetDevice(params->device), "cudaSetDevice");
    }
    ck(cudaGetDevice(&c->device), "cudaGetDevice");
    int major = 0;  // (cudaGetDeviceProperties costs tens of ms: only on failure)
    ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c->device),
       "cudaDeviceGetAttribute");
    if (major != 10) {
      cudaDeviceProp prop;
      ck(cudaGetDeviceProperties(&prop, c->device), "cudaGetDeviceProperties");
      throw CudaFail{std::string("device ") + prop.name +
                     " is not sm_100 (this build targets sm_100a only)"};
    }
    mark("device check");
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking),
       "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "cudaStreamCreate");
    mark("streams");
    c->ls = c->stream;
    c->use_graphs = params->reserved[2] == 0;  // reserved[2] = 1 disables CUDA graphs
    // TMD_GRAPHS=0: eager launches for profilers (ncu cannot profile the kernel
    // nodes of graphs holding conditional nodes); results are bitwise the same
    if (const char* e = std::getenv("TMD_GRAPHS")) {
      if (e[0] == '0') c->use_graphs = false;
    }
    ck(cudaEventCreate(&c->t0), "cudaEventCreate");
    ck(cudaEventCreate(&c->t1), "cudaEventCreate");
    mark("device + streams");
    } catch (...) {
      join_validation();
      throw;
    }
    if (slab) join_validation();  // (the slab selection reads the particles)

    // Slab mode: keep the particles whose wrapped position lies in this
    // rank's z layers (exact host wrap + cell, bit-identical to the device's).
    // Slab mode: the whole system goes to a device scratch block, where the
    // particles whose wrapped position lies in this rank's z layers are
    // selected (exact wrap + cell, bit-identical to the host's rule) and
    // compacted in input order; they are unpacked into the slot arrays once
    // those exist (below).
    int64_t n_keep = sys->n;
    SlabStage stage;
    if (slab) {
      make_slab(c, rank, nranks);
      stage_slab_selection(c, sys, stage);
      n_keep = stage.n_keep;
      mark("slab selection");
    }
    c->my_rank = rank;
    c->nranks = nranks;
    // slot capacity: the whole system, or in slab mode room for the owned
    // particles to double plus both ghost layers (checked at every exchange)
    c->n_cap = sys->n;
    c->n_total = sys->n;
    if (slab) {
      c->n_cap = std::min<int64_t>(2 * sys->n, 2 * n_keep + 65536);
      if (c->n_cap > kMaxSlots) {
        throw StatusError{TMD_ERR_CONFIG, "slab too large for one GPU context"};
      }
    }
    c->n = n_keep;
    c->stride = static_cast<int>((c->n_cap + 31) / 32 * 32);
    c->nblk = std::max(1, blocks_for(c->n, kBlock));  // (an empty system keeps a grid)
    c->dt = params->dt;
    c->half_dt = 0.5 * params->dt;
    c->r_skin = params->r_skin;
    c->r_cut = lj->r_cut;
    c->timers_on = params->section_timers != 0;
    c->th.on = params->thermostat != 0;
    c->th.gamma = params->gamma;
    c->th.temperature = params->temperature;
    c->th.dt = params->dt;
    c->th.seed = params->seed;
    c->lj.fcap = params->force_cap;
    c->variant = (params->reserved[0] >= 1 && params->reserved[0] <= 3) ? params->reserved[0]
                                                                       : kDefaultVariant;
    if (slab) c->variant = 3;  // slab mode runs the brick build + global-slot forces
    if (sys->n_bonds > 0 && c->variant == 2) c->variant = 3;  // bonds: global-slot kernels
    if (params->force_cap > 0.0) {
      if (slab) throw StatusError{TMD_ERR_CONFIG, "force cap: single-GPU warm-up only"};
      c->variant = 1;  // the capped pair force lives in the thread-per-particle kernel
    }
    c->unroll = params->reserved[1] > 0 ? params->reserved[1] : 1;
    c->unroll_auto = params->reserved[1] <= 0;
    {
      const int l = params->reserved[4];
      c->lanes_auto = !(l == 1 || l == 2 || l == 4 || l == 8);
      c->lanes = c->lanes_auto ? 1 : l;
    }
    // auto: double the lanes per particle while the force grid holds fewer
    // than kLanesTargetThreads threads; fixed for the context's life
    // (captured graphs keep their grids)
    if (c->lanes_auto) {
      while (c->lanes < kLanesAutoMax && c->n * c->lanes < kLanesTargetThreads) c->lanes *= 2;
    }
    c->if_nodes = c->n > kChainMaxParticles;
    // speculative blocks (no IF node per step) for systems up to 4M particles
    // in the kernels that honour the halt word; the IF-node graphs above
    c->spec_mode = !slab && c->n <= kSpecMaxParticles;
    if (const char* e = std::getenv("TMD_SPEC")) c->spec_mode = !slab && e[0] == '1';
    if (const char* e = std::getenv("TMD_IF_NODES")) c->if_nodes = e[0] == '1';
    c->build_kind = params->reserved[3];
    c->build_auto = c->build_kind != 3 && c->build_kind != 5 && c->build_kind != 6;
    if (c->build_auto) c->build_kind = 6;  // decided at the first binning (setup_pass)
    setup_bricks(c, static_cast<double>(sys->n), lj->r_cut + params->r_skin);
    mark("bricks");
    if (slab) {  // groups of the owned particles only (+ migration headroom)
      const int64_t want = c->n + c->n / 4 + 1024;
      c->ngroups_max = static_cast<int>(want / 32) + c->bg.nbricks + 1;
    }
    // lj_prepare (potentials.hpp:49-61)
    c->lj.sigma2 = lj->sigma * lj->sigma;
    c->lj.rc2 = lj->r_cut * lj->r_cut;
    c->lj.eps4 = 4.0 * lj->epsilon;
    c->lj.eps24 = 24.0 * lj->epsilon;
    c->lj.shift = 0.0;
    if (lj->energy_shifted) {
      const double s2 = c->lj.sigma2 / c->lj.rc2;
      const double s6 = s2 * s2 * s2;
      c->lj.shift = c->lj.eps4 * (s6 * s6 - s6);
    }

    const size_t n = static_cast<size_t>(c->n_cap);  // capacity
    // Per-slot arrays: one allocation carved into 256-B aligned arrays
    // (cudaMalloc costs ~0.25 ms a call whatever the size); slab contexts
    // allocate them one by one, since they regrow them (grow_capacity).
    std::vector<std::pair<void**, size_t>> plan;
    auto want = [&](auto*& p, size_t count) {
      plan.emplace_back(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(*p));
    };
    // slot n_cap of both buffers: far-away sentinel (variant 3 list padding)
    want(c->posb[0], n + 1);
    want(c->posb[1], n + 1);
    want(c->pos2, n);
    want(c->snap, n);
    want(c->vx, n); want(c->vy, n); want(c->vz, n);
    want(c->vx2, n); want(c->vy2, n); want(c->vz2, n);
    want(c->fx, n); want(c->fy, n); want(c->fz, n);
    want(c->mass, n); want(c->mass2, n);
    want(c->id, n); want(c->id2, n);
    want(c->cell, n); want(c->cell2, n);
    want(c->rank, n); want(c->perm, n);
    want(c->nnbr, n);
    want(c->ck_pos, n);
    want(c->ck_vx, n); want(c->ck_vy, n); want(c->ck_vz, n);
    want(c->ck_mass, n);
    want(c->ck_id, n);
    if (params->thermostat) {
      want(c->ck_fx, n);
      want(c->ck_fy, n);
      want(c->ck_fz, n);
    }
    if (!slab) want(c->dl, 11 * n);  // download / upload scratch
    // the context's small arrays: in the arena too for a whole-box context
    // (slab contexts re-cut and regrow them, so they keep their own)
    c->nparts = std::max({blocks_for(c->n_cap, kBlock), blocks_for(c->n_cap, kLanesPPB),
                          c->bg.nbricks});
    const size_t nscan = static_cast<size_t>(blocks_for(std::max(c->g.ncells, c->bg.nbricks), kScanTile) + 1);
    if (!slab) {
      want(c->count, static_cast<size_t>(c->g.ncells));
      want(c->start, static_cast<size_t>(c->g.ncells) + 1);
      want(c->part_e, static_cast<size_t>(c->nparts));
      want(c->part_w, static_cast<size_t>(c->nparts));
      want(c->part_ke, static_cast<size_t>(c->nparts));
      want(c->scalars, 4);
      want(c->ctrl, 1);
      want(c->rebuild_log, static_cast<size_t>(kChunk));
      if (c->timers_on) want(c->ticks, static_cast<size_t>(kTickSteps * kTickPhases + 1));
      want(c->cell_rank, static_cast<size_t>(c->g.ncells));
      want(c->brick_rank_off, static_cast<size_t>(c->bg.nbricks) + 1);
      want(c->scan_tmp, nscan);
    }
    mark("plan");
    if (!slab) {
      size_t tot = 0;
      for (const auto& e : plan) tot += (e.second + 255) / 256 * 256;
      c->arena = static_cast<char*>(big_alloc(tot, &c->arena_bytes));
      mark("arena");
      size_t off = 0;
      for (const auto& e : plan) {
        *e.first = c->arena + off;
        off += (e.second + 255) / 256 * 256;
      }
    } else {
      for (const auto& e : plan) *e.first = sized_alloc(e.second);  // (cached: a slab regrows them)
    }
    c->cur = 0;
    c->pos = c->posb[0];
    if (slab) {
      c->count = dalloc<int>(c->g.ncells);
      c->start = dalloc<int>(static_cast<size_t>(c->g.ncells) + 1);
      c->part_e = dalloc<double>(c->nparts);
      c->part_w = dalloc<double>(c->nparts);
      c->part_ke = dalloc<double>(c->nparts);
      c->scalars = dalloc<double>(4);
      c->ctrl = dalloc<Ctrl>(1);
      c->rebuild_log = dalloc<int>(static_cast<size_t>(kChunk));
      if (c->timers_on) c->ticks = dalloc<long long>(kTickSteps * kTickPhases + 1);
    }
    mark("device arrays");
    upload_bricks(c);  // (small, pageable: before the particle upload takes the copy engine)
    mark("upload bricks");
    c->h_ctrl = static_cast<Ctrl*>(pinned_small(sizeof(Ctrl)));
    c->h_scalars = static_cast<double*>(pinned_small(4 * sizeof(double)));
    mark("pinned");
    std::memset(c->h_ctrl, 0, sizeof(Ctrl));
    ck(cudaMemsetAsync(c->ctrl, 0, sizeof(Ctrl), c->stream), "memset ctrl");
    ck(cudaMemsetAsync(c->count, 0, sizeof(int) * c->g.ncells, c->stream),
       "memset count");
    ck(cudaMemsetAsync(c->fx, 0, n * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(c->fy, 0, n * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(c->fz, 0, n * sizeof(double), c->stream), "memset");

    mark("allocate");
    // upload the kept particles (input order; the first resort sorts by cell)
    const size_t m = static_cast<size_t>(n_keep);
    const double4 far = make_double4(kFarD, kFarD, kFarD, 0.0);
    if (!slab) {
      // the caller's arrays as they are, unpacked on the device (double4
      // positions, SoA velocities); ids a dense range -> device download
      // positions first on the context stream; velocities and masses behind
      // them on the side stream (one copy at a time over PCIe), so that with
      // ids lo, lo + 1, ... in input order they arrive while the setup pass
      // (resort, list build, first forces — none of which reads them) runs
      // and are placed by id afterwards
      if (m > 0) {
        ck(cudaMemcpyAsync(c->dl, sys->pos, 3 * m * sizeof(double), cudaMemcpyHostToDevice,
                           c->stream), "H2D pos");
        ck(cudaEventCreateWithFlags(&c->ev_up[0], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&c->ev_up[1], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(c->ev_up[0], c->stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->side, c->ev_up[0], 0), "cudaStreamWaitEvent");
        if (sys->vel) {
          ck(cudaMemcpyAsync(c->dl + 3 * m, sys->vel, 3 * m * sizeof(double),
                             cudaMemcpyHostToDevice, c->side), "H2D vel");
        }
        if (sys->mass) {
          ck(cudaMemcpyAsync(c->dl + 6 * m, sys->mass, m * sizeof(double),
                             cudaMemcpyHostToDevice, c->side), "H2D mass");
        }
        ck(cudaEventRecord(c->ev_up[1], c->side), "cudaEventRecord");
      }
      mark("upload enqueued");
      join_validation();  // (overlapped with the upload)
      mark("validated");
      if (m > 0) {
        if (ids_iota) {  // ids lo, lo + 1, ... in input order: no 8 B per particle over PCIe
          c->launches += 1;
          k_iota_i64<<<blocks_for(static_cast<int64_t>(m), kBlock), kBlock, 0, c->stream>>>(
              static_cast<int>(m), idr.lo, c->id);
        } else {
          ck(cudaMemcpyAsync(c->id, sys->id, m * sizeof(long long), cudaMemcpyHostToDevice,
                             c->stream), "H2D id");
        }
        // (the Langevin bath's first force reads velocities and masses)
        defer_vm = ids_iota && !c->th.on && (sys->vel || sys->mass);
        if (!defer_vm) ck(cudaStreamWaitEvent(c->stream, c->ev_up[1], 0), "cudaStreamWaitEvent");
        k_upload<<<blocks_for(static_cast<int64_t>(m), kBlock), kBlock, 0, c->stream>>>(
            static_cast<int>(m), c->dl,
            (sys->vel && !defer_vm) ? c->dl + 3 * m : nullptr,
            (sys->mass && !defer_vm) ? c->dl + 6 * m : nullptr, c->posb[0], c->vx, c->vy, c->vz,
            c->mass);
        ck(cudaGetLastError(), "k_upload");
        c->ids_dense = static_cast<unsigned long long>(idr.hi - idr.lo) ==
                       static_cast<unsigned long long>(m - 1);
        c->dl_lo = idr.lo;
      }
    } else {
      if (m > 0) {
        k_slab_unpack<<<blocks_for(static_cast<int64_t>(m), kBlock), kBlock, 0, c->stream>>>(
            static_cast<int>(m), stage.sel, stage.pos, stage.vel, stage.mass, stage.id,
            c->posb[0], c->vx, c->vy, c->vz, c->mass, c->id);
        ck(cudaGetLastError(), "k_slab_unpack");
      }
      ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
      stage.release();
      mark("upload");
    }
    set_type_table(c, sys, idr);
    k_set_far<<<1, 1, 0, c->stream>>>(c->posb[0] + n, c->posb[1] + n, far);  // list padding slot
    if (slab) alloc_slab(c);
    if (sys->n_bonds > 0) setup_bonds(c, sys, fene);

    c->auto_cap = params->nbr_capacity <= 0;
    // Initial capacity: the expected count at this density (27 cells worth
    // within a sphere of r_verlet) with generous headroom; refined after the
    // first build.
    int cap0 = params->nbr_capacity;
    if (c->auto_cap) {
      const double vol = c->g.L[0] * c->g.L[1] * c->g.L[2];
      const double rho = static_cast<double>(c->n_total) / vol;
      const double rverlet = lj->r_cut + params->r_skin;
      const double expect = rho * 4.18879020478639 * rverlet * rverlet * rverlet;
      cap0 = static_cast<int>(expect * 1.5) + 16;
    }
    alloc_list(c, cap0);
    // slab mode: the owner of the decomposition finishes the setup after the
    // first migration/ghost exchange (tmd_gpu_slab_*); whole box: now
    mark("list alloc");
    if (!slab) setup_pass(c);
    if (defer_vm) {  // velocities / masses placed by id into the slots the setup pass chose
      ck(cudaStreamWaitEvent(c->stream, c->ev_up[1], 0), "cudaStreamWaitEvent");
      c->launches += 1;
      k_place_vm<<<blocks_for(c->n, kBlock), kBlock, 0, c->stream>>>(
          static_cast<int>(c->n), c->id, c->dl_lo, sys->vel ? c->dl + 3 * c->n : nullptr,
          sys->mass ? c->dl + 6 * c->n : nullptr, c->vx, c->vy, c->vz, c->mass);
      ck(cudaGetLastError(), "k_place_vm");
    }
    mark("setup pass");
    c->step = 0;
    c->rebuilds = 0;
    c->ke_fresh = false;
  });
  if (rc != TMD_OK) {
    g_create_error = c->err;
    free_all(c);
    delete c;
    return rc;
  }
  *out = c;
  return TMD_OK;
}

}  // namespace

extern "C" {

int tmd_gpu_create(const tmd_system* sys, const tmd_lj_params* lj,
                   const tmd_fene_params* fene, const tmd_engine_params* params,
                   tmd_gpu_ctx** out) {
  return create_impl(sys, lj, fene, params, 0, 1, false, out);
}

int tmd_gpu_create_slab(const tmd_system* sys, const tmd_lj_params* lj,
                        const tmd_fene_params* fene, const tmd_engine_params* params,
                        int rank, int nranks, tmd_gpu_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    if (out) *out = nullptr;
    g_create_error = "invalid rank / nranks";
    return TMD_ERR_CONFIG;
  }
  return create_impl(sys, lj, fene, params, rank, nranks, true, out);
}

}  // extern "C"

namespace {

struct HostState {
  std::vector<long long> id;
  std::vector<double4> pos;
  std::vector<double> v[3], f[3], mass;
  std::vector<int> cell;
  std::vector<size_t> order;  // slots sorted by id
};

// The current list in global-index ELL-transposed form (variant 1 already
// is; variant 2 is decoded from brick-local indices on the device).
const uint32_t* decoded_list(tmd_gpu_ctx* c) {
  if (c->variant == 1) return c->nbr;
  const size_t words = static_cast<size_t>(c->cap) * c->stride;
  if (c->decoded_words < words) {
    if (c->decoded) cudaFree(c->decoded);
    c->decoded = dalloc<uint32_t>(words);
    c->decoded_words = words;
  }
  c->launches += 1;
  if (c->variant == 3) {
    k_decode_chunked<<<c->nblk, 128, 0, c->ls>>>(static_cast<int>(c->n), c->nbr, c->nnbr,
                                                     c->cap, c->decoded, c->stride);
    return c->decoded;
  }
  k_decode_list<<<c->bg.nbricks, 128, 0, c->ls>>>(
      c->cell_rank, c->brick_rank_off, c->start, c->g, c->bg, c->nbr, c->nnbr, c->decoded,
      c->stride);
  return c->decoded;
}

HostState fetch(tmd_gpu_ctx* c, bool pos, bool vel, bool frc, bool cell, bool mass = false) {
  HostState h;
  const size_t n = static_cast<size_t>(c->n);
  h.id.resize(n);
  ck(cudaMemcpyAsync(h.id.data(), c->id, n * sizeof(long long),
                     cudaMemcpyDeviceToHost, c->stream), "D2H id");
  if (pos) {
    h.pos.resize(n);
    ck(cudaMemcpyAsync(h.pos.data(), c->pos, n * sizeof(double4),
                       cudaMemcpyDeviceToHost, c->stream), "D2H pos");
  }
  double* vs[3] = {c->vx, c->vy, c->vz};
  double* fs[3] = {c->fx, c->fy, c->fz};
  for (int k = 0; k < 3; ++k) {
    if (vel) {
      h.v[k].resize(n);
      ck(cudaMemcpyAsync(h.v[k].data(), vs[k], n * sizeof(double),
                         cudaMemcpyDeviceToHost, c->stream), "D2H vel");
    }
    if (frc) {
      h.f[k].resize(n);
      ck(cudaMemcpyAsync(h.f[k].data(), fs[k], n * sizeof(double),
                         cudaMemcpyDeviceToHost, c->stream), "D2H force");
    }
  }
  if (cell) {
    h.cell.resize(n);
    ck(cudaMemcpyAsync(h.cell.data(), c->cell, n * sizeof(int),
                       cudaMemcpyDeviceToHost, c->stream), "D2H cell");
  }
  if (mass) {
    h.mass.resize(n);
    ck(cudaMemcpyAsync(h.mass.data(), c->mass, n * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream), "D2H mass");
  }
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  h.order.resize(n);
  if (n > 0) {
    // ids filling a dense range: order by direct placement, else sort
    const long long lo = *std::min_element(h.id.begin(), h.id.end());
    const long long hi = *std::max_element(h.id.begin(), h.id.end());
    if (static_cast<unsigned long long>(hi - lo) == static_cast<unsigned long long>(n - 1)) {
      for (size_t s = 0; s < n; ++s) h.order[static_cast<size_t>(h.id[s] - lo)] = s;
    } else {
      std::iota(h.order.begin(), h.order.end(), size_t{0});
      std::sort(h.order.begin(), h.order.end(),
                [&](size_t a, size_t b) { return h.id[a] < h.id[b]; });
    }
  }
  return h;
}

}  // namespace

extern "C" {

const char* tmd_gpu_last_error(const tmd_gpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int tmd_gpu_compute_forces(tmd_gpu_ctx* c, double* pe, double* virial) {
  return guard(c, [&] {
    c->ck_valid = false;
    c->obs_fresh = false;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    launch_forces(c);
    launch_reduce_pe(c);
    ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 2 * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    sync_ctrl(c);
    raise_physics(c, false);
    if (pe) *pe = c->h_scalars[0];
    if (virial) *virial = c->h_scalars[1];
  });
}

}  // extern "C"

namespace {

void free_pair_list(tmd_gpu_ctx* c) {
  for (void* p : {static_cast<void*>(c->pl_pairs), static_cast<void*>(c->pl_off),
                  static_cast<void*>(c->pl_jstart), static_cast<void*>(c->pl_jpairs),
                  static_cast<void*>(c->pl_fp), static_cast<void*>(c->pl_part)}) {
    if (p) cudaFree(p);
  }
  c->pl_pairs = nullptr;
  c->pl_off = nullptr;
  c->pl_jstart = nullptr;
  c->pl_jpairs = nullptr;
  c->pl_fp = nullptr;
  c->pl_part = nullptr;
  c->pl_m = 0;
}

// Slots move at every resort: a pair list holds for one layout generation.
uint64_t layout_gen(const tmd_gpu_ctx* c) { return c->rebuilds * 1000003ull + c->setups; }

void need_pair_list(const tmd_gpu_ctx* c) {
  if (!c->pl_pairs) throw StatusError{TMD_ERR_STATE, "no pair index list built"};
  if (c->pl_layout != layout_gen(c)) {
    throw StatusError{TMD_ERR_STATE, "pair index list is stale: the particles were re-sorted "
                                     "since it was built"};
  }
}

// build_pair_index_list (neighbor_list.hpp:196-247) from the current list.
void build_pair_list(tmd_gpu_ctx* c) {
  free_pair_list(c);
  const int n = static_cast<int>(c->n);
  const uint32_t* gl = decoded_list(c);
  c->pl_off = dalloc<int>(static_cast<size_t>(n) + 1);
  int* cnt = dalloc<int>(static_cast<size_t>(n) + 1);
  ck(cudaMemsetAsync(cnt, 0, sizeof(int) * (static_cast<size_t>(n) + 1), c->stream), "memset");
  c->launches += 1;
  if (n > 0) k_pl_count<<<blocks_for(n, kBlock), kBlock, 0, c->stream>>>(n, gl, c->nnbr, c->stride, cnt);
  size_t tb = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, c->pl_off, n + 1, c->stream), "cub scan");
  void* tmp = dalloc<char>(tb);
  ck(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, c->pl_off, n + 1, c->stream), "cub scan");
  int m = 0;
  ck(cudaMemcpyAsync(&m, c->pl_off + n, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  cudaFree(tmp);
  cudaFree(cnt);
  c->pl_m = m;
  const size_t um = std::max<size_t>(static_cast<size_t>(m), 1);
  c->pl_pairs = dalloc<uint2>(um);
  c->pl_jpairs = dalloc<uint32_t>(um);
  c->pl_fp = dalloc<double>(3 * um);
  c->pl_jstart = dalloc<long long>(static_cast<size_t>(n) + 1);
  c->pl_part = dalloc<double>(2 * static_cast<size_t>(std::max(1, blocks_for(m, kBlock))));
  uint32_t* jkey = dalloc<uint32_t>(um);
  uint32_t* jsorted = dalloc<uint32_t>(um);
  uint32_t* vals = dalloc<uint32_t>(um);
  c->launches += 3;
  if (n > 0) {
    k_pl_fill<<<blocks_for(n, kBlock), kBlock, 0, c->stream>>>(n, gl, c->nnbr, c->stride,
                                                               c->pl_off, c->pl_pairs, jkey);
  }
  if (m > 0) k_pl_iota<<<blocks_for(m, kBlock), kBlock, 0, c->stream>>>(m, vals);
  int bits = 1;
  while ((int64_t{1} << bits) <= c->n_cap) ++bits;
  tb = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, jkey, jsorted, vals, c->pl_jpairs, m, 0, bits,
                                     c->stream), "cub sort");
  tmp = dalloc<char>(tb);
  // stable: each j's pair numbers stay ascending (a fixed summation order)
  ck(cub::DeviceRadixSort::SortPairs(tmp, tb, jkey, jsorted, vals, c->pl_jpairs, m, 0, bits,
                                     c->stream), "cub sort");
  k_pl_jstart<<<blocks_for(n + 1, kBlock), kBlock, 0, c->stream>>>(n, m, jsorted, c->pl_jstart);
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  cudaFree(tmp);
  cudaFree(jkey);
  cudaFree(jsorted);
  cudaFree(vals);
}

// compute_pair_forces(const PairIndexList&, ...) (neighbor_list.hpp:250-268)
void launch_pair_forces(tmd_gpu_ctx* c) {
  const int n = static_cast<int>(c->n);
  const int nb = std::max(1, blocks_for(c->pl_m, kBlock));
  c->launches += 4;
  k_pl_forces<<<nb, kBlock, 0, c->stream>>>(c->pl_m, c->pl_pairs, c->pos, c->g, c->lj, c->pl_fp,
                                           c->pl_part, c->pl_part + nb, c->id, c->ctrl);
  if (n > 0) {
    k_pl_gather<<<blocks_for(n, kBlock), kBlock, 0, c->stream>>>(
        n, c->pl_off, c->pl_jstart, c->pl_jpairs, c->pl_fp, c->fx, c->fy, c->fz);
  }
  k_reduce<<<1, kRedThreads, 0, c->stream>>>(c->pl_part, nb, 1.0, c->scalars + 0);
  k_reduce<<<1, kRedThreads, 0, c->stream>>>(c->pl_part + nb, nb, 1.0, c->scalars + 1);
}

}  // namespace

extern "C" {

int tmd_gpu_build_pair_index_list(tmd_gpu_ctx* c, int64_t* n_pairs) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    build_pair_list(c);
    c->pl_layout = layout_gen(c);
    if (n_pairs) *n_pairs = c->pl_m;
  });
}

int tmd_gpu_pair_index_list(tmd_gpu_ctx* c, int64_t* pairs, size_t cap, size_t* n_out) {
  return guard(c, [&] {
    if (!n_out) throw StatusError{TMD_ERR_CONFIG, "n_out is required"};
    need_pair_list(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    *n_out = static_cast<size_t>(c->pl_m);
    if (!pairs || cap == 0) return;
    const size_t m = std::min(cap, static_cast<size_t>(c->pl_m));
    std::vector<uint2> pr(m);
    std::vector<long long> ids(static_cast<size_t>(c->n_cap));
    ck(cudaMemcpyAsync(pr.data(), c->pl_pairs, m * sizeof(uint2), cudaMemcpyDeviceToHost,
                       c->stream), "D2H pairs");
    ck(cudaMemcpyAsync(ids.data(), c->id, ids.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                       c->stream), "D2H ids");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    for (size_t k = 0; k < m; ++k) {
      pairs[2 * k] = ids[pr[k].x];
      pairs[2 * k + 1] = ids[pr[k].y & kIdxMask];
    }
  });
}

int tmd_gpu_compute_forces_pairs(tmd_gpu_ctx* c, double* pe, double* virial) {
  return guard(c, [&] {
    need_pair_list(c);
    c->ck_valid = false;
    c->obs_fresh = false;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    launch_pair_forces(c);
    ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream), "D2H scalars");
    sync_ctrl(c);
    raise_physics(c, false);
    if (pe) *pe = c->h_scalars[0];
    if (virial) *virial = c->h_scalars[1];
  });
}

int tmd_gpu_time_pair_traversal(tmd_gpu_ctx* c, int reps, double* ms) {
  return guard(c, [&] {
    need_pair_list(c);
    if (reps < 1) throw StatusError{TMD_ERR_CONFIG, "reps must be >= 1"};
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->ck_valid = false;
    c->obs_fresh = false;
    launch_pair_forces(c);  // warm
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    for (int r = 0; r < reps; ++r) launch_pair_forces(c);
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    ck(cudaEventSynchronize(c->t1), "cudaEventSynchronize");
    float t = 0.f;
    ck(cudaEventElapsedTime(&t, c->t0, c->t1), "cudaEventElapsedTime");
    ck(cudaGetLastError(), "kernel launch");
    *ms = static_cast<double>(t) / reps;
  });
}

int tmd_gpu_step(tmd_gpu_ctx* c, int64_t nsteps) {
  return guard(c, [&] {
    if (nsteps < 0) throw StatusError{TMD_ERR_CONFIG, "step count must be non-negative"};
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->h_ctrl->status != 0) {
      throw StatusError{TMD_ERR_STATE,
                        "engine is in an error state from an earlier step"};
    }
    do_run(c, nsteps);
  });
}

int tmd_gpu_run_observed(tmd_gpu_ctx* c, int64_t nsteps, int64_t stride, tmd_observables* out,
                         int64_t cap, int64_t* n_out) {
  return guard(c, [&] {
    if (nsteps < 0) throw StatusError{TMD_ERR_CONFIG, "step count must be non-negative"};
    if (stride < 1) throw StatusError{TMD_ERR_CONFIG, "observable stride must be at least 1"};
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->h_ctrl->status != 0) {
      throw StatusError{TMD_ERR_STATE, "engine is in an error state from an earlier step"};
    }
    if (!c->obs_host) {
      c->obs_host = static_cast<double*>(pinned_small(sizeof(double) * 4 * kObsRows));
      ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->obs_dev), c->obs_host, 0),
         "cudaHostGetDevicePointer");
    }
    const int64_t s0 = c->step;
    c->obs_rows.clear();
    c->obs_stride = static_cast<int>(std::min<int64_t>(stride, 1 << 30));
    try {
      do_run(c, nsteps);
    } catch (...) {
      c->obs_stride = 0;
      throw;
    }
    c->obs_stride = 0;
    // rows by step (a rollback replays and re-records steps: keep the last)
    std::vector<std::array<double, 4>> rows;
    for (const auto& r : c->obs_rows) {
      const int64_t st = static_cast<int64_t>(r[0]);
      if (st <= s0 || st > s0 + nsteps) continue;
      while (!rows.empty() && static_cast<int64_t>(rows.back()[0]) >= st) rows.pop_back();
      rows.push_back(r);
    }
    *n_out = static_cast<int64_t>(rows.size());
    for (size_t k = 0; k < rows.size() && static_cast<int64_t>(k) < cap; ++k) {
      out[k].step = static_cast<int64_t>(rows[k][0]);
      out[k].kinetic = rows[k][1];
      out[k].potential = rows[k][2];
      out[k].virial = rows[k][3];
      out[k].temperature = (c->n > 0 ? 2.0 * rows[k][1] / (3.0 * static_cast<double>(c->n)) : 0.0);
    }
  });
}

int tmd_gpu_observe(tmd_gpu_ctx* c, tmd_observables* out) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->obs_fresh) {  // the run's graph already delivered them
      out->step = c->step;
      out->potential = c->h_scalars[0];
      out->virial = c->h_scalars[1];
      out->kinetic = c->h_scalars[2];
      out->temperature = (c->n > 0 ? 2.0 * out->kinetic / (3.0 * static_cast<double>(c->n)) : 0.0);
      return;
    }
    // after a run the closing half-kick already left the kinetic partials of
    // the current velocities (the force kernel's blocks: 128 particles, or 32
    // for the small-system lanes kernel — the same sum to rounding as
    // k_kinetic's, and what run_observed recorded); the brick variant's
    // partials are per brick
    if (!(c->ke_fresh && c->variant != 2)) {
      c->launches += 1;
      launch_kinetic(c);
    }
    launch_reduce_ke(c);
    ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 3 * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "kernel launch");
    out->step = c->step;
    out->potential = c->h_scalars[0];
    out->virial = c->h_scalars[1];
    out->kinetic = c->h_scalars[2];
    // KineticResult::temperature (soa_store.hpp:200-204)
    out->temperature = (c->n > 0 ? 2.0 * out->kinetic / (3.0 * static_cast<double>(c->n)) : 0.0);
  });
}

int tmd_gpu_download(tmd_gpu_ctx* c, int64_t* id, double* pos, double* vel,
                     double* force, int32_t* type, double* mass) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t nn = static_cast<size_t>(c->n);
    std::vector<long long> ids_tmp;
    long long* ids_out = reinterpret_cast<long long*>(id);
    if (!ids_out && type && !c->type_val.empty()) {  // ids needed for the type lookup
      ids_tmp.resize(nn);
      ids_out = ids_tmp.data();
    }
    if (c->ids_dense && !c->g.zslab && nn > 0) {
      // id order by direct placement on the device, positions wrapped there
      // (wrap1, box.hpp:47-51), one copy per array into the
      // caller's buffers
      double* dpos = c->dl;
      double* dvel = c->dl + 3 * nn;
      double* dfrc = c->dl + 6 * nn;
      long long* did = reinterpret_cast<long long*>(c->dl + 9 * nn);
      double* dmass = c->dl + 10 * nn;
      k_download<<<blocks_for(c->n, kBlock), kBlock, 0, c->stream>>>(
          static_cast<int>(nn), c->pos, c->vx, c->vy, c->vz, c->fx, c->fy, c->fz, c->mass, c->id,
          c->dl_lo, c->g, pos ? dpos : nullptr, vel ? dvel : nullptr, force ? dfrc : nullptr,
          mass ? dmass : nullptr, did);
      ck(cudaGetLastError(), "k_download");
      (void)did;  // (dense ids in id order are lo, lo + 1, ...: written by the host below)
      if (pos) {
        ck(cudaMemcpyAsync(pos, dpos, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), "D2H pos");
      }
      if (vel) {
        ck(cudaMemcpyAsync(vel, dvel, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), "D2H vel");
      }
      if (force) {
        ck(cudaMemcpyAsync(force, dfrc, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), "D2H force");
      }
      if (mass) {
        ck(cudaMemcpyAsync(mass, dmass, nn * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
           "D2H mass");
      }
      if (ids_out) {  // while the copies run
        const long long lo = c->dl_lo;
        parallel_chunks(static_cast<int64_t>(nn), [&](int, int64_t b, int64_t e) {
          for (int64_t k = b; k < e; ++k) ids_out[k] = lo + k;
        });
      }
      ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    } else if (nn > 0) {
      // ids of any shape (slab contexts, sparse ids): a device sort of the
      // ids gives the slot order, one gather kernel writes id-ordered arrays
      const int n = static_cast<int>(nn);
      size_t tb = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, static_cast<const long long*>(nullptr),
                                         static_cast<long long*>(nullptr),
                                         static_cast<const int*>(nullptr),
                                         static_cast<int*>(nullptr), n, 0, 64, c->stream),
         "cub sort size");
      const size_t words = 11 * nn;  // pos 3, vel 3, force 3, mass 1 doubles + sorted ids
      const size_t bytes = words * sizeof(double) + 2 * nn * sizeof(int) + tb + 256;
      size_t got = 0;
      char* scratch = static_cast<char*>(big_alloc(bytes, &got));
      double* dpos = reinterpret_cast<double*>(scratch);
      double* dvel = dpos + 3 * nn;
      double* dfrc = dpos + 6 * nn;
      double* dmass = dpos + 9 * nn;
      long long* did = reinterpret_cast<long long*>(dpos + 10 * nn);
      int* vin = reinterpret_cast<int*>(dpos + 11 * nn);
      int* vout = vin + nn;
      void* tmp = reinterpret_cast<char*>(vout + nn);
      try {
        k_iota_int<<<blocks_for(n, kBlock), kBlock, 0, c->stream>>>(n, vin);
        ck(cub::DeviceRadixSort::SortPairs(tmp, tb, c->id, did, vin, vout, n, 0, 64, c->stream),
           "cub sort ids");
        k_download_gather<<<blocks_for(n, kBlock), kBlock, 0, c->stream>>>(
            n, vout, c->pos, c->vx, c->vy, c->vz, c->fx, c->fy, c->fz, c->mass, c->g,
            pos ? dpos : nullptr, vel ? dvel : nullptr, force ? dfrc : nullptr,
            mass ? dmass : nullptr);
        ck(cudaGetLastError(), "k_download_gather");
        if (ids_out) {
          ck(cudaMemcpyAsync(ids_out, did, nn * sizeof(long long), cudaMemcpyDeviceToHost,
                             c->stream), "D2H id");
        }
        if (pos) {
          ck(cudaMemcpyAsync(pos, dpos, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream), "D2H pos");
        }
        if (vel) {
          ck(cudaMemcpyAsync(vel, dvel, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream), "D2H vel");
        }
        if (force) {
          ck(cudaMemcpyAsync(force, dfrc, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream), "D2H force");
        }
        if (mass) {
          ck(cudaMemcpyAsync(mass, dmass, nn * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream), "D2H mass");
        }
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
      } catch (...) {
        cudaStreamSynchronize(c->stream);
        big_free(scratch, got);
        throw;
      }
      big_free(scratch, got);
    }
    if (type) {
      if (c->type_val.empty()) {
        std::fill(type, type + nn, 0);
      } else {
        for (size_t r = 0; r < nn; ++r) type[r] = type_of(c, ids_out[r]);
      }
    }
  });
}

int tmd_gpu_set_velocities(tmd_gpu_ctx* c, const int64_t* id, const double* vel) {
  return guard(c, [&] {
    c->ck_valid = false;
    c->ke_fresh = false;
    c->obs_fresh = false;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    HostState h = fetch(c, false, false, false, false);
    const size_t n = h.order.size();
    std::vector<std::pair<int64_t, size_t>> in(n);
    for (size_t k = 0; k < n; ++k) in[k] = {id[k], k};
    std::sort(in.begin(), in.end());
    std::vector<double> v[3];
    for (int k = 0; k < 3; ++k) v[k].resize(n);
    for (size_t r = 0; r < n; ++r) {
      const size_t slot = h.order[r];
      if (in[r].first != h.id[slot]) {
        throw StatusError{TMD_ERR_CONFIG, "set_velocities: id set differs from the engine's"};
      }
      for (int k = 0; k < 3; ++k) v[k][slot] = vel[3 * in[r].second + k];
    }
    double* vs[3] = {c->vx, c->vy, c->vz};
    for (int k = 0; k < 3; ++k) {
      ck(cudaMemcpyAsync(vs[k], v[k].data(), n * sizeof(double),
                         cudaMemcpyHostToDevice, c->stream), "H2D vel");
    }
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  });
}

int tmd_gpu_cell_of(tmd_gpu_ctx* c, int64_t* id, int32_t* cell) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    HostState h = fetch(c, false, false, false, true);
    for (size_t r = 0; r < h.order.size(); ++r) {
      id[r] = h.id[h.order[r]];
      cell[r] = h.cell[h.order[r]];
    }
  });
}

int tmd_gpu_pairs(tmd_gpu_ctx* c, int64_t* pairs, size_t cap, size_t* n_out) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    HostState h = fetch(c, false, false, false, false);
    const size_t n = h.order.size();
    if (c->n_ghost > 0) {  // slab mode: neighbours may be ghost slots
      h.id.resize(n + static_cast<size_t>(c->n_ghost));
      ck(cudaMemcpy(h.id.data() + n, c->id + n, static_cast<size_t>(c->n_ghost) * sizeof(long long),
                    cudaMemcpyDeviceToHost), "D2H ghost ids");
    }
    const int rows = std::min(c->cap, std::max(c->h_ctrl->max_count, 0));
    std::vector<int> cnt(n);
    std::vector<uint32_t> list(static_cast<size_t>(rows) * c->stride);
    const uint32_t* glist = decoded_list(c);
    ck(cudaMemcpyAsync(cnt.data(), c->nnbr, n * sizeof(int),
                       cudaMemcpyDeviceToHost, c->stream), "D2H nnbr");
    if (!list.empty()) {
      ck(cudaMemcpyAsync(list.data(), glist, list.size() * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost, c->stream), "D2H nbr");
    }
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    std::vector<std::pair<int64_t, int64_t>> out;
    out.reserve(static_cast<size_t>(c->h_ctrl->entries / 2 + 1));
    for (size_t i = 0; i < n; ++i) {
      const int64_t a = h.id[i];
      for (int k = 0; k < cnt[i]; ++k) {
        const uint32_t ent = list[static_cast<size_t>(k) * c->stride + i];
        const int64_t b = h.id[ent & kIdxMask];
        if (a < b) out.emplace_back(a, b);
      }
    }
    std::sort(out.begin(), out.end());
    *n_out = out.size();
    for (size_t k = 0; k < std::min(cap, out.size()); ++k) {
      pairs[2 * k] = out[k].first;
      pairs[2 * k + 1] = out[k].second;
    }
  });
}

int tmd_gpu_timers(tmd_gpu_ctx* c, double sec[5], double* elapsed) {
  for (int k = 0; k < 5; ++k) sec[k] = c->sec[k];
  if (elapsed) *elapsed = c->elapsed;
  return TMD_OK;
}

uint64_t tmd_gpu_rebuild_count(const tmd_gpu_ctx* c) { return c->rebuilds; }
int64_t tmd_gpu_step_count(const tmd_gpu_ctx* c) { return c->step; }
int64_t tmd_gpu_size(const tmd_gpu_ctx* c) { return c->n; }

int tmd_gpu_list_stats(tmd_gpu_ctx* c, tmd_list_stats* out) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    unsigned long long* d = dalloc<unsigned long long>(1);
    ck(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream), "memset");
    c->launches += 1;
    k_count_incut<<<c->nblk, kBlock, 0, c->ls>>>(
        static_cast<int>(c->n), c->pos, decoded_list(c), c->nnbr, c->stride, c->g,
        c->lj.rc2, d);
    unsigned long long h = 0;
    ck(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream), "D2H");
    sync_ctrl(c);
    cudaFree(d);
    out->n = c->n;
    out->entries = c->h_ctrl->entries;
    out->in_cut = static_cast<int64_t>(h);
    out->max_count = c->h_ctrl->max_count;
    out->capacity = c->cap;
    for (int k = 0; k < 3; ++k) {
      out->dims[k] = c->g.dims[k];
      out->cell_len[k] = c->g.cell_len[k];
    }
  });
}

int tmd_gpu_time_force_kernel(tmd_gpu_ctx* c, int reps, double* ms) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (reps < 1) throw StatusError{TMD_ERR_CONFIG, "reps must be >= 1"};
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    for (int r = 0; r < reps; ++r) launch_forces(c);
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    ck(cudaEventSynchronize(c->t1), "cudaEventSynchronize");
    float t = 0.f;
    ck(cudaEventElapsedTime(&t, c->t0, c->t1), "cudaEventElapsedTime");
    ck(cudaGetLastError(), "kernel launch");
    *ms = static_cast<double>(t) / reps;
  });
}

// The kernel a production step runs: forces + the fused velocity-Verlet
// epilogue (kFused: closing half-kick, next opening half-kick + drift into
// the other position buffer, displacement max). Each launch advances the
// state by one step without rebuild checks, so the state is checkpointed
// first and restored afterwards (positions, velocities; the list is rebuilt
// and the forces recomputed at the restored positions, as after a rollback).
int tmd_gpu_time_step_kernel(tmd_gpu_ctx* c, int reps, double* ms) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (reps < 1) throw StatusError{TMD_ERR_CONFIG, "reps must be >= 1"};
    if (c->nranks > 1 || c->g.zslab) {
      throw StatusError{TMD_ERR_STATE, "step-kernel timing needs a whole-box context"};
    }
    if (c->th.on) {  // the restored forces would need the checkpoint's Langevin kick
      throw StatusError{TMD_ERR_CONFIG, "step-kernel timing needs an NVE context"};
    }
    sync_ctrl(c);
    const Ctrl before = *c->h_ctrl;
    checkpoint(c);
    launch_forces(c, kForcesOnly);  // warm (same list, same positions)
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    for (int r = 0; r < reps; ++r) launch_forces(c, kFused);
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    ck(cudaEventSynchronize(c->t1), "cudaEventSynchronize");
    float t = 0.f;
    ck(cudaEventElapsedTime(&t, c->t0, c->t1), "cudaEventElapsedTime");
    ck(cudaGetLastError(), "kernel launch");
    *ms = static_cast<double>(t) / reps;
    restore(c, before);
    c->ck_valid = false;
    setup_pass(c);
    enqueue_observables(c);
    sync_ctrl(c);
  });
}

// Captures the CUDA graphs a run will launch (blocks of kGraphSteps and
// single steps at the current buffer parity; with obs_stride > 0 the
// observed family as run_observed(stride) launches it), so that no capture
// falls inside a later timed run.
int tmd_gpu_prepare_graphs(tmd_gpu_ctx* c, int64_t obs_stride) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (!c->use_graphs || c->nranks > 1 || c->g.zslab) return;
    if (c->graph_dirty) drop_graphs(c);
    if (c->spec_mode && c->variant >= 2) {  // the blocks a run of this system will launch
      const int keep = c->obs_stride;
      for (int pass = 0; pass < (obs_stride > 0 ? 2 : 1); ++pass) {
        c->obs_stride = pass == 0 ? 0 : static_cast<int>(std::min<int64_t>(obs_stride, 1 << 30));
        if (pass == 1 && c->sgo_stride != c->obs_stride) {
          drop_spec_graphs(c, true);
          c->sgo_stride = c->obs_stride;
        }
        try {
          for (int par = 0; par < 2; ++par) {
            for (int slot = 0; slot < 2; ++slot) {
              for (int K = 0; K <= 12; ++K) spec_graph(c, K, slot, par);
            }
          }
        } catch (...) {
          c->obs_stride = keep;
          throw;
        }
      }
      c->obs_stride = keep;
      return;
    }
    for (int kind = 0; kind < 2; ++kind) {
      auto& sgr = c->sg[kind][c->cur];
      if (!sgr.exec) capture_graph(c, kind == 0 ? kGraphSteps : 1, sgr);
    }
    if (obs_stride > 0) {
      const int stride = static_cast<int>(std::min<int64_t>(obs_stride, 1 << 30));
      if (c->sgo_stride != stride) {
        for (auto& row : c->sgo) {
          for (auto& sg : row) {
            if (sg.exec) cudaGraphExecDestroy(sg.exec);
            if (sg.graph) cudaGraphDestroy(sg.graph);
            sg = tmd_gpu_ctx::StepGraph{};
          }
        }
        c->sgo_stride = stride;
      }
      const int keep = c->obs_stride;
      c->obs_stride = stride;
      try {
        for (int kind = 0; kind < 2; ++kind) {
          auto& sgr = c->sgo[kind][c->cur];
          if (!sgr.exec) capture_graph(c, kind == 0 ? kGraphSteps : 1, sgr);
        }
      } catch (...) {
        c->obs_stride = keep;
        throw;
      }
      c->obs_stride = keep;
    }
  });
}

int tmd_gpu_time_list_build(tmd_gpu_ctx* c, int reps, double* ms) {
  return guard(c, [&] {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (reps < 1) throw StatusError{TMD_ERR_CONFIG, "reps must be >= 1"};
    set_force_rebuild(c);
    launch_decide(c, false);  // rebuild = 1 until the next decision
    ck(cudaEventRecord(c->t0, c->stream), "cudaEventRecord");
    for (int r = 0; r < reps; ++r) launch_build(c);
    ck(cudaEventRecord(c->t1, c->stream), "cudaEventRecord");
    ck(cudaEventSynchronize(c->t1), "cudaEventSynchronize");
    float t = 0.f;
    ck(cudaEventElapsedTime(&t, c->t0, c->t1), "cudaEventElapsedTime");
    sync_ctrl(c);
    *ms = static_cast<double>(t) / reps;
  });
}

void* tmd_gpu_stream(tmd_gpu_ctx* c) { return c->stream; }

uint64_t tmd_gpu_launch_count(const tmd_gpu_ctx* c) { return c->launches; }

void tmd_gpu_kernel_config(const tmd_gpu_ctx* c, int* variant, int* lanes, int* build_kind) {
  if (variant) *variant = c->variant;
  if (lanes) *lanes = c->variant == 3 ? c->lanes : 1;
  if (build_kind) *build_kind = c->variant >= 2 ? c->build_kind : 0;
}

int tmd_gpu_fp64_peak(int device, double* tflops) {
  tmd_gpu_ctx tmp;
  return guard(&tmp, [&] {
    if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
    int dev = 0, sms = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    double* out = dalloc<double>(static_cast<size_t>(sms) * 8 * 256);
    const int blocks = sms * 8, iters = 1 << 14;
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "ev");
    ck(cudaEventCreate(&b), "ev");
    k_dfma_peak<<<blocks, 256>>>(out, iters);  // warm-up
    ck(cudaEventRecord(a), "ev");
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_dfma_peak<<<blocks, 256>>>(out, iters);
    ck(cudaEventRecord(b), "ev");
    ck(cudaEventSynchronize(b), "sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
    ck(cudaGetLastError(), "k_dfma_peak");
    const double flops = 2.0 * kDfmaChains * static_cast<double>(iters) * blocks * 256 * reps;
    *tflops = flops / (1e-3 * ms) / 1e12;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
  });
}

// ---------------------------------------------------------------------------
// z-slab decomposition entry points (multi-GPU). The caller (one
// process per GPU, paper_2109_10876_b200/decomp.py) drives every rank through
// the same sequence and moves the byte buffers between ranks itself (NCCL,
// or device copies when all ranks live in one process):
//
//   setup / rebuild:  decide(rebuild=1) -> migrate_out -> [records to their
//                     destination ranks] -> migrate_in -> commit -> border(0/1)
//                     -> [boundary layers to the lower/upper neighbour]
//                     -> ghost_in -> [counts, ids, positions] -> ghosts_ready
//   per step:         forces(fused) -> halo -> [positions] -> max_d2 ->
//                     [max over ranks] -> decide(rebuild) -> ...
//
// Every call returns with the context's stream drained, so the caller may
// move the returned device buffers on any stream.

namespace {

void need_slab(const tmd_gpu_ctx* c) {
  if (!c->g.zslab) {
    throw StatusError{TMD_ERR_STATE, "not a slab context (use tmd_gpu_create_slab)"};
  }
}

// Keeps the list's group capacity ahead of the owned count (migration can
// grow a slab's population).
void ensure_groups(tmd_gpu_ctx* c) {
  const int need = static_cast<int>(c->n / 32) + c->bg.nbricks + 1;
  if (need > c->ngroups_max) {
    c->ngroups_max = need + need / 8 + 64;
    alloc_list(c, c->cap);
  }
}


// Commit of a migration, device side (no host round trip): arrivals
// unpacked, the normal resort, then the lowest and highest owned layers
// exported (per-cell counts, their scan, ids and positions, slots). The
// border sizes are left on the device at boff[s] + dxy.
void slab_commit_launch(tmd_gpu_ctx* c) {
  if (c->mig_nrecv > 0) {
    c->launches += 1;
    k_mig_unpack<<<blocks_for(c->mig_nrecv, kBlock), kBlock, 0, c->ls>>>(
        static_cast<int>(c->mig_nrecv), c->mig_recv, static_cast<int>(c->n), c->pos, c->vx,
        c->vy, c->vz, c->mass, c->id);
  }
  c->n += c->mig_nrecv;
  c->mig_nrecv = 0;
  c->nblk = std::max(1, blocks_for(c->n, kBlock));
  ensure_groups(c);
  launch_resort(c);  // requires the rebuild decision (decide(rebuild=1))
  const int dxy = c->g.dims[0] * c->g.dims[1];
  const int qb = blocks_for(dxy, kBlock);
  for (int s = 0; s < 2; ++s) {
    const int lz = s == 0 ? 1 : c->g.zown;  // lowest / highest owned layer
    c->launches += 3;
    k_layer_counts<<<qb, kBlock, 0, c->ls>>>(lz, c->g, c->cell_rank, c->start, c->count);
    launch_scan(c, dxy, c->count, c->boff[s]);  // leaves count zeroed
    k_layer_counts<<<qb, kBlock, 0, c->ls>>>(lz, c->g, c->cell_rank, c->start, c->bcnt[s]);
    k_layer_gather<<<qb, kBlock, 0, c->ls>>>(lz, c->g, c->cell_rank, c->start, c->boff[s],
                                             c->pos, c->id, c->bidx[s], c->bids[s],
                                             c->bpos[s]);
  }
  c->fused_ready = false;  // the layout changed: remote ghost addresses are re-derived
}

// The border sizes on the host: the fused halo's export map (slot -> index
// in each side's export).
void slab_commit_finish(tmd_gpu_ctx* c, int64_t nb0, int64_t nb1) {
  c->nb[0] = nb0;
  c->nb[1] = nb1;
  c->launches += 3;
  k_fill_int2<<<c->nblk, kBlock, 0, c->ls>>>(static_cast<int>(c->n), c->exp, make_int2(-1, -1));
  for (int s = 0; s < 2; ++s) {
    if (c->nb[s] == 0) continue;
    k_export_map<<<blocks_for(c->nb[s], kBlock), kBlock, 0, c->ls>>>(
        static_cast<int>(c->nb[s]), c->bidx[s], s, c->exp);
  }
}

}  // namespace

int tmd_gpu_slab_info(tmd_gpu_ctx* c, int64_t info[11]) {
  return guard(c, [&] {
    info[0] = c->my_rank;
    info[1] = c->nranks;
    info[2] = c->g.z0;
    info[3] = c->g.zown;
    info[4] = c->n;
    info[5] = c->n_ghost_lo;
    info[6] = c->n_ghost_hi;
    info[7] = static_cast<int64_t>(c->g.dims[0]) * c->g.dims[1];
    info[8] = c->n_cap;
    info[9] = static_cast<int64_t>(sizeof(MigRec));
    info[10] = c->recuts;
  });
}

int tmd_gpu_slab_layer_counts(tmd_gpu_ctx* c, int64_t* counts) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const int dz = c->g.dims[2];
    if (static_cast<size_t>(dz) * sizeof(unsigned int) > 96 * 1024) {
      throw StatusError{TMD_ERR_CONFIG, "too many z layers for the layer histogram"};
    }
    unsigned long long* d = dalloc<unsigned long long>(static_cast<size_t>(dz));
    ck(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * dz, c->stream), "memset");
    if (c->n > 0) {
      c->launches += 1;
      const int blocks = std::min(c->nblk, 148 * 8);
      const size_t smem = static_cast<size_t>(dz) * sizeof(unsigned int);
      if (smem > 48 * 1024) {
        ck(cudaFuncSetAttribute(k_layer_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)), "smem attr hist");
      }
      k_layer_hist<<<blocks, kBlock, smem, c->ls>>>(static_cast<int>(c->n), c->pos, c->g, d);
    }
    std::vector<unsigned long long> h(static_cast<size_t>(dz));
    ck(cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * dz, cudaMemcpyDeviceToHost,
                       c->stream), "D2H hist");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "k_layer_hist");
    cudaFree(d);
    for (int z = 0; z < dz; ++z) counts[z] = static_cast<int64_t>(h[static_cast<size_t>(z)]);
  });
}

int tmd_gpu_slab_recut(tmd_gpu_ctx* c, const int32_t* cuts) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const int R = c->nranks, dz = c->g.dims[2];
    std::vector<int> v(cuts, cuts + R + 1);
    if (v[0] != 0 || v[static_cast<size_t>(R)] != dz) {
      throw StatusError{TMD_ERR_CONFIG, "cut planes must start at 0 and end at dims_z"};
    }
    for (int r = 0; r < R; ++r) {
      if (v[static_cast<size_t>(r) + 1] <= v[static_cast<size_t>(r)]) {
        throw StatusError{TMD_ERR_CONFIG, "every slab needs at least one z layer"};
      }
    }
    recut(c, v);
  });
}

int tmd_gpu_slab_max_d2(tmd_gpu_ctx* c, double* local_max_d2) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    sync_ctrl(c);
    raise_physics(c, true);
    if (c->h_ctrl->status & kStatStray) throw CudaFail{"slab: particle outside its slab"};
    c->step = c->h_ctrl->step;
    c->rebuilds = static_cast<uint64_t>(c->h_ctrl->rebuilds);
    double m = 0.0;
    std::memcpy(&m, &c->h_ctrl->max_d2, sizeof m);
    *local_max_d2 = m;
  });
}

int tmd_gpu_slab_decide(tmd_gpu_ctx* c, int rebuild, int advance) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (rebuild) set_force_rebuild(c);
    launch_decide(c, advance != 0);
  });
}

int tmd_gpu_slab_migrate_out(tmd_gpu_ctx* c, int64_t* counts, void** send) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const int R = c->nranks;
    const int n = static_cast<int>(c->n);
    ck(cudaMemsetAsync(c->mig_count, 0, 2 * sizeof(int) * R, c->stream), "memset");
    ck(cudaMemsetAsync(c->mig_keep, 0, sizeof(int), c->stream), "memset");
    c->launches += 2;
    if (n > 0) {
      k_mig_classify<<<c->nblk, kBlock, 0, c->ls>>>(n, c->pos, c->id, c->owner_of_z,
                                                    c->my_rank, c->g, c->mig_dest,
                                                    c->mig_count, c->ctrl);
    }
    std::vector<int> h(static_cast<size_t>(R));
    ck(cudaMemcpyAsync(h.data(), c->mig_count, sizeof(int) * R, cudaMemcpyDeviceToHost,
                       c->stream), "D2H mig counts");
    sync_ctrl(c);
    raise_physics(c, true);
    std::vector<int> off(static_cast<size_t>(R) + 1, 0);
    for (int r = 0; r < R; ++r) off[r + 1] = off[r] + h[r];
    ck(cudaMemcpyAsync(c->mig_off, off.data(), sizeof(int) * (R + 1), cudaMemcpyHostToDevice,
                       c->stream), "H2D mig offsets");
    if (n > 0) {
      k_mig_pack<<<c->nblk, kBlock, 0, c->ls>>>(
          n, c->pos, c->vx, c->vy, c->vz, c->mass, c->id, c->mig_dest, c->my_rank,
          c->mig_off, c->mig_count + R, c->mig_send, c->mig_keep, c->pos2, c->vx2, c->vy2,
          c->vz2, c->mass2, c->id2);
    }
    int keep = 0;
    ck(cudaMemcpyAsync(&keep, c->mig_keep, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
       "D2H keep");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    const size_t k = static_cast<size_t>(keep);
    auto cp = [&](void* d, const void* s, size_t bytes) {
      if (bytes) ck(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, c->stream), "copy");
    };
    cp(c->pos, c->pos2, k * sizeof(double4));
    cp(c->vx, c->vx2, k * sizeof(double));
    cp(c->vy, c->vy2, k * sizeof(double));
    cp(c->vz, c->vz2, k * sizeof(double));
    cp(c->mass, c->mass2, k * sizeof(double));
    cp(c->id, c->id2, k * sizeof(long long));
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "kernel launch");
    c->n = keep;
    c->n_ghost = c->n_ghost_lo = c->n_ghost_hi = 0;
    for (int r = 0; r < R; ++r) counts[r] = h[r];
    *send = c->mig_send;
  });
}

int tmd_gpu_slab_migrate_in(tmd_gpu_ctx* c, int64_t nrecv, void** recv) {
  return guard(c, [&] {
    need_slab(c);
    if (nrecv < 0) throw StatusError{TMD_ERR_CONFIG, "negative record count"};
    grow_capacity(c, c->n + nrecv);
    c->mig_nrecv = nrecv;
    *recv = c->mig_recv;
  });
}

int tmd_gpu_slab_commit(tmd_gpu_ctx* c, int64_t nb_out[2]) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    slab_commit_launch(c);
    const int dxy = c->g.dims[0] * c->g.dims[1];
    int tot[2] = {0, 0};
    for (int s = 0; s < 2; ++s) {
      ck(cudaMemcpyAsync(&tot[s], c->boff[s] + dxy, sizeof(int), cudaMemcpyDeviceToHost,
                         c->stream), "D2H border size");
    }
    sync_ctrl(c);
    raise_physics(c, true);
    if (c->h_ctrl->status & kStatStray) throw CudaFail{"slab: particle outside its slab"};
    slab_commit_finish(c, tot[0], tot[1]);
    nb_out[0] = tot[0];
    nb_out[1] = tot[1];
  });
}

int tmd_gpu_slab_border(tmd_gpu_ctx* c, int side, void** counts, void** ids, void** pos) {
  return guard(c, [&] {
    need_slab(c);
    if (side != 0 && side != 1) throw StatusError{TMD_ERR_CONFIG, "side must be 0 or 1"};
    *counts = c->bcnt[side];
    *ids = c->bids[side];
    *pos = c->bpos[side];
  });
}

int tmd_gpu_slab_ghost_in(tmd_gpu_ctx* c, int64_t n_lo, int64_t n_hi, void* lo[3],
                          void* hi[3]) {
  return guard(c, [&] {
    need_slab(c);
    if (n_lo < 0 || n_hi < 0) throw StatusError{TMD_ERR_CONFIG, "negative ghost count"};
    grow_capacity(c, c->n + n_lo + n_hi);
    c->n_ghost_lo = n_lo;
    c->n_ghost_hi = n_hi;
    c->n_ghost = n_lo + n_hi;
    lo[0] = c->gcnt[0];
    lo[1] = c->id + c->n;
    lo[2] = c->pos + c->n;
    hi[0] = c->gcnt[1];
    hi[1] = c->id + c->n + n_lo;
    hi[2] = c->pos + c->n + n_lo;
  });
}

int tmd_gpu_slab_ghosts_ready(tmd_gpu_ctx* c) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->launches += 1;
    k_ghost_starts<<<1, 1024, 0, c->ls>>>(c->g, static_cast<int>(c->n), c->gcnt[0], c->gcnt[1],
                                         c->start);
    for (;;) {
      launch_build(c);
      sync_ctrl(c);
      raise_physics(c, true);
      if (c->h_ctrl->status & kOverflowBits) {
        const Ctrl h = *c->h_ctrl;
        reset_status(c);
        grow_after_overflow(c, h);
        if (c->variant != 3) {
          throw StatusError{TMD_ERR_CONFIG, "slab mode: brick halo exceeds shared memory"};
        }
        continue;
      }
      if (c->auto_cap) {
        const int want = round8(c->h_ctrl->max_count + c->h_ctrl->max_count / 4 + 8);
        if (want > c->cap) {
          alloc_list(c, want);
          continue;
        }
      }
      break;
    }
  });
}

int tmd_gpu_slab_kick_drift(tmd_gpu_ctx* c) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (c->n > 0) launch_kick_drift(c);
  });
}

// mode: 0 forces only, 1 forces + closing half-kick, 2 closing half-kick +
// next opening half-kick + drift (the position buffers swap).
int tmd_gpu_slab_forces(tmd_gpu_ctx* c, int mode) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    launch_forces(c, mode == 2 ? kFused : (mode == 1 ? kKick2 : kForcesOnly));
    if (mode == 0) launch_thermo_init(c);  // setup evaluation (step-0 noise)
  });
}

int tmd_gpu_slab_halo(tmd_gpu_ctx* c, void* send[2], void* recv[2]) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    for (int s = 0; s < 2; ++s) {
      if (c->nb[s] == 0) continue;
      c->launches += 1;
      k_pack_border<<<blocks_for(c->nb[s], kBlock), kBlock, 0, c->ls>>>(
          static_cast<int>(c->nb[s]), c->bidx[s], c->pos, c->bpos[s], c->ctrl);
    }
    send[0] = c->bpos[0];
    send[1] = c->bpos[1];
    recv[0] = c->pos + c->n;
    recv[1] = c->pos + c->n + c->n_ghost_lo;
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "kernel launch");
  });
}

int tmd_gpu_slab_sums(tmd_gpu_ctx* c, double out[3]) {
  return guard(c, [&] {
    need_slab(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->launches += 1;
    launch_kinetic(c);
    launch_reduce_ke(c);
    launch_reduce_pe(c);
    ck(cudaMemcpyAsync(c->h_scalars, c->scalars, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "kernel launch");
    for (int k = 0; k < 3; ++k) out[k] = c->h_scalars[k];
  });
}

int tmd_gpu_brute_force(const tmd_system* sys, const tmd_lj_params* lj, double r_verlet,
                        int device, double* force, double* pe, int64_t* pairs, size_t cap,
                        size_t* n_pairs) {
  tmd_gpu_ctx tmp;
  const int rc = guard(&tmp, [&] {
    if (!sys || !lj || sys->n < 1 || !sys->pos || !sys->id) {
      throw StatusError{TMD_ERR_CONFIG, "brute force: empty system"};
    }
    if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
    const size_t n = static_cast<size_t>(sys->n);
    LjConst c{};
    c.sigma2 = lj->sigma * lj->sigma;
    c.rc2 = lj->r_cut * lj->r_cut;
    c.eps4 = 4.0 * lj->epsilon;
    c.eps24 = 24.0 * lj->epsilon;
    if (lj->energy_shifted) {
      const double s2 = c.sigma2 / c.rc2, s6 = s2 * s2 * s2;
      c.shift = c.eps4 * (s6 * s6 - s6);
    }
    const int blocks = blocks_for(static_cast<int64_t>(n), kBlock);
    double* dpos = dalloc<double>(3 * n);
    long long* did = dalloc<long long>(n);
    double* dforce = dalloc<double>(3 * n);
    double* dpart = dalloc<double>(static_cast<size_t>(blocks));
    unsigned long long* dn = dalloc<unsigned long long>(1);
    int* dover = dalloc<int>(1);
    const size_t pcap = std::max<size_t>(cap, 1);
    long long* dpairs = dalloc<long long>(2 * pcap);
    ck(cudaMemcpy(dpos, sys->pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(did, sys->id, n * sizeof(long long), cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemset(dn, 0, sizeof(unsigned long long)), "memset");
    ck(cudaMemset(dover, 0, sizeof(int)), "memset");
    k_brute<<<blocks, kBlock>>>(static_cast<int>(n), dpos, did, sys->box[0], sys->box[1],
                                sys->box[2], c, r_verlet * r_verlet, dforce, dpart, dn, dpairs,
                                static_cast<unsigned long long>(cap), dover);
    ck(cudaGetLastError(), "k_brute");
    std::vector<double> part(static_cast<size_t>(blocks));
    unsigned long long np = 0;
    int over = 0;
    ck(cudaMemcpy(part.data(), dpart, part.size() * sizeof(double), cudaMemcpyDeviceToHost),
       "D2H");
    ck(cudaMemcpy(&np, dn, sizeof np, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(&over, dover, sizeof over, cudaMemcpyDeviceToHost), "D2H");
    if (force) {
      ck(cudaMemcpy(force, dforce, 3 * n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    }
    if (pairs && np > 0) {
      const size_t m = std::min<size_t>(cap, static_cast<size_t>(np));
      std::vector<long long> h(2 * m);
      ck(cudaMemcpy(h.data(), dpairs, 2 * m * sizeof(long long), cudaMemcpyDeviceToHost),
         "D2H");
      std::vector<std::pair<int64_t, int64_t>> v(m);
      for (size_t k = 0; k < m; ++k) v[k] = {h[2 * k], h[2 * k + 1]};
      std::sort(v.begin(), v.end());
      for (size_t k = 0; k < m; ++k) {
        pairs[2 * k] = v[k].first;
        pairs[2 * k + 1] = v[k].second;
      }
    }
    void* ptrs[] = {dpos, did, dforce, dpart, dn, dover, dpairs};
    for (void* q : ptrs) cudaFree(q);
    if (over) throw StatusError{TMD_ERR_PHYSICS, "brute force: overlapping particles"};
    if (pe) {
      double t = 0.0;
      for (double v : part) t += v;
      *pe = t;
    }
    if (n_pairs) *n_pairs = static_cast<size_t>(np);
  });
  if (rc != TMD_OK) g_create_error = tmp.err;
  return rc;
}

void release_nccl_cache();

void tmd_gpu_release_cache(void) {
  release_nccl_cache();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (const CachedBlock& b : g_cache) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(b.device);
    cudaFree(b.p);
    cudaSetDevice(cur);
  }
  g_cache.clear();
}

void tmd_gpu_destroy(tmd_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
}

}  // extern "C"

#include "tmd_slab_nccl.cuh"

void release_nccl_cache() {
#ifndef TMD_NO_NCCL
  nccl_cache_release_all();
#endif
}

namespace {
void free_comm(tmd_gpu_ctx* c) {
  for (auto& e : c->ipc_open) cudaIpcCloseMemHandle(e.second);
  c->ipc_open.clear();
  delete comm(c);
  c->comm = nullptr;
}
}  // namespace
