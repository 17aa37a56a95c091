/*
 * tmd_gpu.h — C ABI of the B200 LJ short-range engine (libtmd_gpu.so).
 *
 * Drop-in boundary for the reference `taskmd` engine's hot path
 * (/root/reference/proj/include/taskmd/). There is no plugin/FFI layer in the
 * reference: its path sits behind inline C++ APIs, so each entry point below
 * names the reference interface it replaces. A header-only C++ wrapper with
 * the taskmd::Engine surface sits on top (include/taskmd_gpu/engine.hpp), and
 * the Python mirror binds the same symbols with ctypes
 * (paper_2109_10876_b200/engine.py).
 *
 * Conventions
 *  - plain pointers and sizes only; host arrays are copied, never retained;
 *  - every call returns a status (TMD_OK = 0) except the getters noted;
 *  - statuses map 1:1 onto the reference's exception types
 *    (errors.hpp:19-43) and, through them, onto the CLI exit codes
 *    (md_cli.cpp:333-352);
 *  - a context owns one GPU's device memory and one CUDA stream; it is NOT
 *    thread-safe (one host thread drives it, like taskmd::Engine,
 *    task_pool.hpp:15-24);
 *  - there is no CPU fallback: without a usable sm_100 device, create fails
 *    with TMD_ERR_CUDA.
 */
#ifndef TMD_GPU_H_
#define TMD_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMD_GPU_ABI_VERSION 4

/* Status codes. */
#define TMD_OK 0
#define TMD_ERR_CONFIG 1  /* taskmd::ConfigError  */
#define TMD_ERR_PHYSICS 2 /* taskmd::PhysicsError */
#define TMD_ERR_VERIFY 3  /* taskmd::VerifyError  */
#define TMD_ERR_STATE 4   /* taskmd::StateError   */
#define TMD_ERR_CUDA 5    /* device / driver failure (no reference analog) */

/* Timer sections, in the order of taskmd::Section (timers.hpp:11-17). */
#define TMD_SECTION_FORCES 0
#define TMD_SECTION_COMM 1
#define TMD_SECTION_INTEGRATE 2
#define TMD_SECTION_NEIGH 3
#define TMD_SECTION_RESORT 4

typedef struct tmd_gpu_ctx tmd_gpu_ctx;

/* taskmd::FlatConfig (flat_config.hpp:18-40) as plain arrays. pos/vel are
 * xyz-interleaved [3*n]; type and mass may be NULL (0 and 1.0). vel may be
 * NULL (zero). Topology::bonds (topology.hpp:14-31) as n_bonds (a, b) id pairs
 * (bonds[2*k], bonds[2*k+1]); angles are not on the GPU path. Bonded systems
 * need ids in a dense range (max - min < 4 n + 1024) and at most 8 bonds per
 * particle. */
typedef struct tmd_system {
  double box[3];
  int64_t n;
  const int64_t* id;
  const int32_t* type;
  const double* mass;
  const double* pos;
  const double* vel;
  int64_t n_bonds;
  const int64_t* bonds;
} tmd_system;

/* taskmd::LjParams (potentials.hpp:21-26). */
typedef struct tmd_lj_params {
  double epsilon;
  double sigma;
  double r_cut;
  int energy_shifted;
} tmd_lj_params;

/* taskmd::FeneParams (potentials.hpp:77-104): Interactions::fene, NULL when
 * absent. Bonds need it, and r_max <= r_cut + r_skin (domain.hpp:151-159). */
typedef struct tmd_fene_params {
  double k;
  double r_max;
} tmd_fene_params;

/* taskmd::EngineConfig (engine.hpp:19-26) minus the CPU-only knobs
 * (n_sub / worker_threads have no GPU meaning), plus r_skin (the
 * build_domain argument, domain.hpp:134) and device selection. */
typedef struct tmd_engine_params {
  double dt;
  double r_skin;
  int device;        /* CUDA ordinal; -1 = current device */
  int section_timers; /* 1: fill the five SectionTimers with CUDA-event
                         times per phase; 0: only `elapsed` */
  int nbr_capacity;  /* 0 = auto (sized from the first build); else fixed
                        entries per particle (rounded up to a multiple of 8) */
  int reserved[5];   /* [0] kernel variant: 0 = default (3), 1 = thread-per-
                        particle ELL list, 2 = brick-staged shared memory,
                        3 = sector-chunked list + 256-bit gathers;
                        [1] variant-3 gathers in flight (1/2/4/8, 0 = 4);
                        [2] 1 = no CUDA graphs;
                        [3] variant-3 list build: 0 = by cell occupancy,
                        3 = warp per cell, 5 = thread per particle,
                        6 = warp per cell over a culled candidate stream;
                        [4] variant-3 threads per particle (1/2/4/8, 0 = by
                        particle count: small systems get more) */
  /* EngineConfig::thermostat (optional<LangevinParams>, potentials.hpp:174-178):
   * thermostat = 0 is NVE. The Langevin force of thermostat_and_half_kick
   * (engine.hpp:209-239) with counter_normal3(seed, kThermostat, step, id). */
  int thermostat;
  double gamma;
  double temperature;
  uint64_t seed;
  /* > 0: cap every LJ pair force at |F| <= force_cap (energies uncapped) —
   * the overlap warm-up of a freshly generated polymer melt (BASELINE
   * configs[2]); runs the thread-per-particle kernel. 0 = off. */
  double force_cap;
} tmd_engine_params;

/* taskmd::StepObservables (engine.hpp:43-48) plus the virial
 * W = sum over in-cut pairs of ff * r^2 (absent from the reference). */
typedef struct tmd_observables {
  int64_t step;
  double kinetic;
  double potential;
  double virial;
  double temperature;
} tmd_observables;

/* Neighbour-list statistics of the last build (roofline accounting). */
typedef struct tmd_list_stats {
  int64_t n;          /* owned particles */
  int64_t entries;    /* unpadded full-list entries (E) */
  int64_t in_cut;     /* entries with r < r_cut at the last force call (2P) */
  int32_t max_count;  /* largest per-particle entry count */
  int32_t capacity;   /* allocated entries per particle */
  int32_t dims[3];    /* cell grid */
  double cell_len[3];
} tmd_list_stats;

/* Replaces build_domain(flat, inter, r_skin, n_sub) (domain.hpp:134-189) +
 * Engine::Engine(Domain, EngineConfig) (engine.hpp:68-77): validates like the
 * reference (validate_flat / validate_lj / build_cell_grid), uploads, bins,
 * builds the list and runs the initial untimed force evaluation
 * (compute_forces_untimed, engine.hpp:244-278). */
int tmd_gpu_create(const tmd_system* sys, const tmd_lj_params* lj,
                   const tmd_fene_params* fene /* NULL: no bonds */,
                   const tmd_engine_params* params, tmd_gpu_ctx** out);

/* Message of the last failed call on ctx (or of the last failed create when
 * ctx is NULL). Getter: never fails. */
const char* tmd_gpu_last_error(const tmd_gpu_ctx* ctx);

/* One force evaluation at the current positions with the current list:
 * compute_subnode_forces + reduce_potential (engine.hpp:191-207) ==
 * compute_pair_forces (neighbor_list.hpp:150) over the whole system. */
int tmd_gpu_compute_forces(tmd_gpu_ctx* ctx, double* pe, double* virial);

/* Engine::step / Engine::run (engine.hpp:80-130). PhysicsError messages carry
 * "(at step N)" like run_phase (engine.hpp:167-170). */
int tmd_gpu_step(tmd_gpu_ctx* ctx, int64_t nsteps);

/* Engine::run with an observable row every `stride` steps (the CLI's
 * observable_stride loop, md_cli.cpp:110-126, without a host round trip per
 * row): each recorded step's (step, KE, PE, W, T) is written by the device
 * into mapped pinned host memory as the step completes. Rows for the steps
 * s with s % stride == 0 in (start, start + nsteps], in order; at most cap
 * written to out, *n_out = the count. */
int tmd_gpu_run_observed(tmd_gpu_ctx* ctx, int64_t nsteps, int64_t stride, tmd_observables* out,
                         int64_t cap, int64_t* n_out);

/* Engine::observe (engine.hpp:132-140) + virial. */
int tmd_gpu_observe(tmd_gpu_ctx* ctx, tmd_observables* out);

/* flatten_domain (domain.hpp:193-207): arrays of n entries sorted by id,
 * positions wrapped into the box, each particle's type and mass as created
 * (ParticleRec, flat_config.hpp:18-40); forces are the last evaluation's.
 * Any output pointer may be NULL. */
int tmd_gpu_download(tmd_gpu_ctx* ctx, int64_t* id, double* pos, double* vel,
                     double* force, int32_t* type, double* mass);

/* Overwrite velocities by id (ids sorted or not; every owned id exactly once).
 * The analog of tests poking Domain stores (test_engine.cpp:174-184). */
int tmd_gpu_set_velocities(tmd_gpu_ctx* ctx, const int64_t* id,
                           const double* vel);

/* Parity tap: CellGrid::cell_of of every particle at the last resort
 * (distribute_records, domain.hpp:56-65), sorted by id. */
int tmd_gpu_cell_of(tmd_gpu_ctx* ctx, int64_t* id, int32_t* cell);

/* Parity tap: every listed pair as (min id, max id), sorted — the same
 * multiset as the reference's half lists (test_neighbor.cpp:49-65). Writes at
 * most cap pairs to pairs[2*cap]; *n receives the total. */
int tmd_gpu_pairs(tmd_gpu_ctx* ctx, int64_t* pairs, size_t cap, size_t* n);

/* PairIndexList (neighbor_list.hpp:193-268): the reference's classical
 * Verlet list of explicit (i, j) pairs and its Newton-3 traversal, the
 * baseline of its traversal microbenchmark (bench_traversal.cpp).
 * tmd_gpu_build_pair_index_list = build_pair_index_list (196-247): from the
 * current neighbour list, each unordered pair (and periodic image) once;
 * *n_pairs = its length. It holds until the particles are next re-sorted
 * (a rebuild): later calls fail with TMD_ERR_STATE. */
int tmd_gpu_build_pair_index_list(tmd_gpu_ctx* ctx, int64_t* n_pairs);
/* Parity tap: the pair list as (id_i, id_j), list order; at most cap pairs,
 * *n = the total. */
int tmd_gpu_pair_index_list(tmd_gpu_ctx* ctx, int64_t* pairs, size_t cap, size_t* n);
/* compute_pair_forces(const PairIndexList&, ...) (250-268): one force
 * evaluation at the current positions over the pair list (per-pair forces,
 * then per-particle sums in a fixed order: no floating-point atomics);
 * forces stored as by tmd_gpu_compute_forces. */
int tmd_gpu_compute_forces_pairs(tmd_gpu_ctx* ctx, double* pe, double* virial);
/* Benchmark hook: mean ms per pair-list traversal (bench_traversal.cpp). */
int tmd_gpu_time_pair_traversal(tmd_gpu_ctx* ctx, int reps, double* ms_per_traversal);

/* Engine::timers (engine.hpp:145): seconds per section + elapsed. */
int tmd_gpu_timers(tmd_gpu_ctx* ctx, double sec[5], double* elapsed);

/* Getters (never fail on a valid ctx). */
uint64_t tmd_gpu_rebuild_count(const tmd_gpu_ctx* ctx); /* engine.hpp:148 */
int64_t tmd_gpu_step_count(const tmd_gpu_ctx* ctx);     /* engine.hpp:146 */
int64_t tmd_gpu_size(const tmd_gpu_ctx* ctx);

int tmd_gpu_list_stats(tmd_gpu_ctx* ctx, tmd_list_stats* out);

/* Benchmark hook: launches the force kernel `reps` times back to back on the
 * context's stream between two CUDA events recorded on that stream and
 * returns the mean milliseconds per launch. Results are left in place. */
int tmd_gpu_time_force_kernel(tmd_gpu_ctx* ctx, int reps, double* ms_per_launch);

/* Benchmark hook: the kernel a production step runs (forces + the fused
 * velocity-Verlet epilogue: closing half-kick, next opening half-kick + drift,
 * displacement max), `reps` launches back to back between CUDA events on the
 * context's stream; mean milliseconds per launch. The launches advance the
 * state, so positions and velocities are checkpointed before and restored
 * after (list rebuilt, forces recomputed). Whole-box NVE contexts only. */
int tmd_gpu_time_step_kernel(tmd_gpu_ctx* ctx, int reps, double* ms_per_launch);

/* Captures the CUDA graphs the next run will launch (15-step blocks and
 * single steps at the current buffer parity; obs_stride > 0: also the family
 * tmd_gpu_run_observed(stride) launches) without running them, so that no
 * capture falls inside a timed run. No-op with section timers or in slab
 * mode. */
int tmd_gpu_prepare_graphs(tmd_gpu_ctx* ctx, int64_t obs_stride);

/* Benchmark hook: rebuilds the neighbour list `reps` times at the current
 * positions (no resort) between CUDA events; mean milliseconds per build. */
int tmd_gpu_time_list_build(tmd_gpu_ctx* ctx, int reps, double* ms_per_build);

/* Raw stream handle (cudaStream_t) of the context, for callers that want to
 * order their own work after the engine's. */
void* tmd_gpu_stream(tmd_gpu_ctx* ctx);

/* The kernels this context runs (no reference counterpart; bench and test
 * accounting): force/list variant (1-3), variant-3 threads per particle
 * (1/2/4/8) and list build kind (3/5/6). Getter; null outputs are skipped. */
void tmd_gpu_kernel_config(const tmd_gpu_ctx* ctx, int* variant, int* lanes, int* build_kind);

/* Kernels this context has enqueued so far (bench accounting). Getter. */
uint64_t tmd_gpu_launch_count(const tmd_gpu_ctx* ctx);

/* Measured FP64 FMA throughput of the device in TFLOP/s (2 FLOP per DFMA),
 * the FLOP-side roofline denominator. device = -1: current device. */
int tmd_gpu_fp64_peak(int device, double* tflops);

/* Frees the context. Its two large device blocks (per-slot arrays, list)
 * go to a process-wide cache for the next context of the process (at most
 * 16 GiB per device, reused at <= 1.5x the request). */
void tmd_gpu_destroy(tmd_gpu_ctx* ctx);

/* Returns every cached block of the process to the driver (e.g. before
 * handing the memory to another library). */
void tmd_gpu_release_cache(void);

/* ---- z-slab decomposition (one context per GPU) --------------
 * Replaces the reference's in-process subnode decomposition
 * (decomp.hpp:47-118 make_subnode_decomposition / make_subnode_layouts,
 * domain.hpp:54-92 distribute_records, decomp.hpp:142-200 build_ghost_plan /
 * update_ghost_positions) for one process per GPU: the box is cut into slabs
 * of whole z cell layers (range rule i*dims/s, decomp.hpp:87-93); a slab owns
 * its layers plus one ghost layer per side. With a full neighbour list there
 * is no reverse force pass (collect_ghost_forces, decomp.hpp:202-224).
 *
 * The caller moves the buffers between ranks (NCCL or device copies); every
 * call returns with the context's stream drained. Sequence:
 *   rebuild:  slab_decide(1, adv) -> slab_migrate_out -> [records to their
 *             destinations] -> slab_migrate_in -> slab_commit ->
 *             slab_border(0/1) -> [lower layer to rank-1's upper ghost, upper
 *             layer to rank+1's lower ghost] -> slab_ghost_in -> [counts,
 *             ids, positions] -> slab_ghosts_ready
 *   step:     slab_forces(2) -> slab_halo -> [positions] -> slab_max_d2 ->
 *             [max over ranks > 0.25 skin^2 ?] -> slab_decide(r, 1) -> ...
 * Buffers: counts int32[dx*dy] (cells x-fastest), ids int64[n],
 * positions double4[n] (x, y, z, unused), records info[9] bytes each. */

/* Slab `rank` of `nranks` (1 <= nranks <= z cell layers, >= 3 layers; with
 * nranks = 1 the slab's ghost layers are its own boundary layers); every
 * rank passes the same whole system and keeps the particles in its layers.
 * The context is not usable for forces before the first rebuild sequence. */
int tmd_gpu_create_slab(const tmd_system* sys, const tmd_lj_params* lj,
                        const tmd_fene_params* fene, const tmd_engine_params* params,
                        int rank, int nranks, tmd_gpu_ctx** out);

/* info: rank, nranks, first owned z layer, owned layers, owned particles,
 * lower ghosts, upper ghosts, cells per layer, slot capacity, record bytes,
 * re-cuts of the native loop. */
int tmd_gpu_slab_info(tmd_gpu_ctx* ctx, int64_t info[11]);

/* Native step loop of the decomposition (one process or thread per GPU):
 * the same protocol driven from C++ with NCCL on the context's stream.
 * tmd_nccl_unique_id fills 128 bytes on one rank (ncclGetUniqueId), which the
 * caller broadcasts; every rank then attaches its slab context
 * (ncclCommInitRank with the context's rank / nranks), runs the first
 * migration / ghost exchange + forces (tmd_gpu_slab_setup), and steps
 * (tmd_gpu_slab_run: collective, the same nsteps on every rank; per step one
 * NCCL group of halo sends/receives, one MAX all-reduce and an 8-byte read
 * for the rebuild decision). flags bit 0: load-aware cut planes
 * re-evaluated at every rebuild (tmd_gpu_slab_layer_counts summed with an
 * NCCL all-reduce); bit 1: fused halo — the force kernel's epilogue stores
 * boundary particles' new positions straight into the neighbours' ghost
 * slots (CUDA IPC peer memory over NVLink), replacing the per-step pack +
 * NCCL point-to-point. tmd_gpu_slab_observe all-reduces PE, W, KE. */
int tmd_nccl_unique_id(void* id);
int tmd_gpu_slab_attach_nccl(tmd_gpu_ctx* ctx, const void* unique_id, int flags);
/* The same loop with every rank's context in ONE process, one host thread per
 * rank (R slabs on one GPU, or several GPUs of one process): a collective is a
 * rendezvous of the rank threads exchanging stream events and device
 * pointers, after which each rank's stream copies / reduces its peers'
 * buffers — stream-ordered like NCCL, no kernel waits on another rank's
 * kernel. Create one group per decomposition, attach each rank's context
 * (flags as above), then call tmd_gpu_slab_setup / _run / _run_observed /
 * _observe on every rank concurrently from its own thread. A rank that fails
 * releases the others (they fail with "a peer rank failed"). The group may be
 * destroyed once every context is attached (contexts hold a reference).
 * Replaces the reference's in-process subnode decomposition driven by its
 * TaskPool (decomp.hpp:47-224, task_pool.hpp:15-106). */
int tmd_local_group_create(int nranks, void** group);
void tmd_local_group_destroy(void* group);
int tmd_gpu_slab_attach_local(tmd_gpu_ctx* ctx, void* group, int flags);
/* One process per rank whose collectives and messages are staged through host
 * memory shared by mapping the file `path` (every rank passes the same path;
 * the file is created and sized on first use and should start empty). Each
 * operation synchronises the context stream first, so no kernel ever waits on
 * another rank: several ranks can share ONE GPU. The fused halo's peer
 * buffers are CUDA IPC mappings as with NCCL. The multi-process test path of
 * the native loop (NCCL needs a GPU per rank); not a production transport. */
int tmd_gpu_slab_attach_host(tmd_gpu_ctx* ctx, const char* path, int flags);
int tmd_gpu_slab_setup(tmd_gpu_ctx* ctx);
int tmd_gpu_slab_run(tmd_gpu_ctx* ctx, int64_t nsteps);
/* tmd_gpu_slab_run recording every `stride`-th step's observables as the
 * device computes them (the slab form of tmd_gpu_run_observed): rows hold
 * this rank's LOCAL kinetic / potential / virial sums (temperature 0); the
 * caller sums them over ranks (one reduction of the whole table, no per-step
 * host round trip). */
int tmd_gpu_slab_run_observed(tmd_gpu_ctx* ctx, int64_t nsteps, int64_t stride,
                              tmd_observables* rows, int64_t cap, int64_t* n_rows);
int tmd_gpu_slab_observe(tmd_gpu_ctx* ctx, int64_t n_total, tmd_observables* out);

/* Load-aware cuts: owned particles per global z layer
 * (counts[dims_z], wrapped positions) — the caller sums them over ranks and
 * picks cut planes; tmd_gpu_slab_recut then moves this slab to layers
 * [cuts[rank], cuts[rank+1]) (cuts[0] = 0, cuts[nranks] = dims_z, every slab
 * >= 1 layer; all ranks pass the same cuts, right before slab_migrate_out).
 * Replaces the reference's static range rule (decomp.hpp:87-93) for
 * inhomogeneous systems, the role autotune_subnodes + work stealing play on
 * the CPU (engine.hpp:293-373, task_pool.hpp:85-106). */
int tmd_gpu_slab_layer_counts(tmd_gpu_ctx* ctx, int64_t* counts);
/* The cut planes the native loop picks from summed layer counts: contiguous
 * slabs minimising the largest population, each >= 1 layer (host only). */
int tmd_balanced_cuts(const int64_t* counts, int dims_z, int nranks, int32_t* cuts);
int tmd_gpu_slab_recut(tmd_gpu_ctx* ctx, const int32_t* cuts);

/* Largest squared displacement since the last build over the owned particles
 * (needs_rebuild's per-subnode max, neighbor_list.hpp:114-145). Raises any
 * pending physics error. */
int tmd_gpu_slab_max_d2(tmd_gpu_ctx* ctx, double* local_max_d2);

/* Sets this step's rebuild decision (rebuild != 0 forces it); advance != 0
 * counts a step (and a rebuild). */
int tmd_gpu_slab_decide(tmd_gpu_ctx* ctx, int rebuild, int advance);

/* Wraps every owned particle and moves the ones whose z layer another rank
 * owns into a record buffer grouped by destination: counts[nranks] records
 * per destination, *send the device buffer (destination-major). */
int tmd_gpu_slab_migrate_out(tmd_gpu_ctx* ctx, int64_t* counts, void** send);

/* Device buffer for nrecv incoming records (any source order). */
int tmd_gpu_slab_migrate_in(tmd_gpu_ctx* ctx, int64_t nrecv, void** recv);

/* Appends the received records, resorts the owned particles (cell-sorted,
 * brick-major) and exports both boundary layers; nb[0] / nb[1] = particles
 * in the lowest / highest owned layer. */
int tmd_gpu_slab_commit(tmd_gpu_ctx* ctx, int64_t nb[2]);

/* Device buffers of boundary layer `side` (0 lowest, 1 highest): per-cell
 * counts, ids, positions. */
int tmd_gpu_slab_border(tmd_gpu_ctx* ctx, int side, void** counts, void** ids,
                        void** pos);

/* Destination buffers (counts, ids, positions) of the lower ghost layer
 * (n_lo particles, from rank-1's highest layer) and the upper one (n_hi,
 * from rank+1's lowest layer). */
int tmd_gpu_slab_ghost_in(tmd_gpu_ctx* ctx, int64_t n_lo, int64_t n_hi, void* lo[3],
                          void* hi[3]);

/* Ghost layers complete: cell ranges + neighbour-list build (grows on
 * overflow). */
int tmd_gpu_slab_ghosts_ready(tmd_gpu_ctx* ctx);

/* Opening half-kick + drift of the owned particles (Engine::half_kick_and_drift,
 * engine.hpp:174-189). */
int tmd_gpu_slab_kick_drift(tmd_gpu_ctx* ctx);

/* Forces on the owned particles; mode 0 forces only, 1 + closing half-kick,
 * 2 + closing half-kick + next opening half-kick and drift. */
int tmd_gpu_slab_forces(tmd_gpu_ctx* ctx, int mode);

/* Packs both boundary layers' current positions: send[0/1] -> rank-1 / rank+1
 * (slab_commit's nb[] positions each); recv[0/1] <- rank-1 / rank+1 (the
 * n_lo / n_hi ghost positions). */
int tmd_gpu_slab_halo(tmd_gpu_ctx* ctx, void* send[2], void* recv[2]);

/* This slab's potential energy, virial (of the last force call) and kinetic
 * energy; the caller sums them over ranks. */
int tmd_gpu_slab_sums(tmd_gpu_ctx* ctx, double out[3]);

/* Brute-force check for the CLI's `verify` (the reference uses
 * oracle_forces_energy / oracle_pair_set, oracle.hpp:31-160, md_cli.cpp:
 * 205-306): O(N^2) LJ forces and energy under the minimum-image convention
 * plus every pair within r_verlet, on the GPU, without cells or lists.
 * force[3n] in input order; pairs sorted (min id, max id), at most cap;
 * *n_pairs = the total. Errors: tmd_gpu_last_error(NULL). */
int tmd_gpu_brute_force(const tmd_system* sys, const tmd_lj_params* lj, double r_verlet,
                        int device, double* force, double* pe, int64_t* pairs, size_t cap,
                        size_t* n_pairs);

/* ---- host-side setup helpers (no GPU needed) ----------------------------
 * Synthetic inputs of the BASELINE.json shapes. FCC is absent from the
 * reference (generators.hpp has only simple cubic), see SURVEY §8(d). */

/* FCC lattice: cells^3 unit cells x 4 basis sites, cubic box
 * L = cbrt(4 cells^3 / rho), a = L / cells, positions
 * (i + b_k + offset) * a, ids in z, y, x, basis order. Arrays sized
 * 4*cells^3. */
int tmd_gen_fcc(int cells, double rho, double offset, int64_t* id, double* pos,
                double box[3]);

/* The reference's generators (generators.hpp), restated for the run-config
 * front end: gen_lattice (47-81), gen_spherical (83-135; call with id = NULL
 * first for the count), gen_random (212-258; TMD_ERR_VERIFY = placement
 * gave up). Velocities thermal at T with zero net momentum. */
int tmd_gen_lattice(int64_t n, double rho, double temperature, uint64_t seed, int64_t* id,
                    double* pos, double* vel, double box[3]);
int tmd_gen_spherical(double box_length, double diameter_fraction, double rho_in, double alpha,
                      double temperature, uint64_t seed, int64_t* id, double* pos, double* vel,
                      int64_t* n_out, double box[3]);
int tmd_gen_random(int64_t n, double rho, double min_distance, double temperature,
                   uint64_t seed, int64_t* id, double* pos, double* vel, double box[3]);

/* Kremer-Grest melt (BASELINE configs[2]; new — the reference generates
 * only ring melts, generators.hpp:137-210): n_chains linear random-walk
 * chains of chain_len beads, bond length `bond`, no immediate back-folding,
 * cubic box L = (N/rho)^(1/3), ids chain-major, bonds[2*(n_chains*(chain_len-1))]
 * as consecutive (i, i+1) pairs. Velocities are left to the caller. */
int tmd_gen_chains(int64_t n_chains, int64_t chain_len, double rho, double bond, uint64_t seed,
                   int64_t* id, double* pos, int64_t* bonds, double box[3]);

/* gen_detail::thermal_velocities + zero_net_momentum (generators.hpp:19-39):
 * v = sqrt(T/m) * counter_normal3(seed, kVelocityInit, 0, id), then the
 * mass-weighted net momentum is removed. mass may be NULL (1.0). */
void tmd_thermal_velocities(int64_t n, const int64_t* id, const double* mass,
                            double temperature, uint64_t seed, double* vel);

/* counter_uniform3 / counter_normal3 (random.hpp:53-81), context ids as
 * taskmd::RngContext (1 thermostat, 2 velocity init, 3 placement). */
void tmd_counter_uniform3(uint64_t seed, uint64_t ctx, uint64_t step,
                          uint64_t id, double out[3]);
void tmd_counter_normal3(uint64_t seed, uint64_t ctx, uint64_t step,
                         uint64_t id, double out[3]);

int tmd_gpu_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TMD_GPU_H_ */
