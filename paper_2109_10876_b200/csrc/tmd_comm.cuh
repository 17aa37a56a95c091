// Transport of the native slab loop (tmd_slab_nccl.cuh): the collectives and
// point-to-point messages of the z-slab decomposition behind one small
// interface, stream-ordered like NCCL (nothing in a step waits for the host).
//
//   NcclComm   one process (or thread) per GPU, NCCL on the context stream.
//   HostFileComm  one process per rank, collectives and messages staged through
//              host memory shared by a file mapping (every op synchronises the
//              stream first): slow, but it runs the multi-process path — CUDA
//              IPC peer buffers of the fused halo included — with several
//              ranks on ONE GPU without any kernel waiting on another rank
//              (the test of the cross-process protocol; NCCL needs one GPU per
//              rank).
//   LocalComm  every rank's context in one process, one host thread per rank
//              (R slabs on one GPU, or several GPUs of one process): a
//              collective is a host rendezvous of the rank threads that
//              publishes stream events and device pointers; each rank's stream
//              then waits on its peers' events and copies / reduces their
//              buffers on its own stream, and every rank's later work waits
//              until all copies out of its buffers ran. No kernel ever waits
//              on another rank's kernel — only on events of finished work.
//
// Point-to-point messages of a group between a pair of ranks match in
// posting order (NCCL's rule); LocalComm also checks sizes and that every
// message was matched, which turns a protocol bug into an error instead of a
// hang.
#pragma once

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#ifndef TMD_NO_NCCL
#include <nccl.h>
#endif

namespace {

enum class CType { kI32, kI64, kU64, kF64 };
enum class COp { kSum, kMax };

inline size_t ctype_bytes(CType t) { return t == CType::kI32 ? 4 : 8; }

struct SlabComm {
  virtual ~SlabComm() = default;
  // in place over `count` elements of every rank's buf
  virtual void allreduce(void* buf, size_t count, CType t, COp op, cudaStream_t s) = 0;
  // recv[q * bytes, (q + 1) * bytes) = rank q's send (send and recv disjoint)
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  virtual void group_start() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void group_end(cudaStream_t s) = 0;
  virtual void abort() {}  // a rank failed: release peers blocked in a collective
  virtual bool in_process() const = 0;  // every rank's buffers are this process's pointers
};

#ifndef TMD_NO_NCCL
inline void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw CudaFail{std::string(what) + ": " + ncclGetErrorString(r)};
  }
}

// Communicators outlive their engines: a closed context hands its
// communicator to a process-wide cache keyed by (device, ranks, rank), and
// the next context of the process with the same key takes it instead of
// paying ncclCommInitRank again (hundreds of ms). Every rank of an SPMD job
// creates and closes its engines in the same sequence, so all hit or all
// miss together. TMD_NCCL_CACHE=0 turns it off; tmd_gpu_release_cache
// destroys the cached ones.
struct NcclCached {
  int device, nranks, rank;
  ncclComm_t comm;
};
inline std::mutex& nccl_cache_mu() {
  static std::mutex m;
  return m;
}
inline std::vector<NcclCached>& nccl_cache() {
  static std::vector<NcclCached> v;
  return v;
}
inline bool nccl_cache_on() {
  const char* e = std::getenv("TMD_NCCL_CACHE");
  return !(e && e[0] == '0');
}
inline ncclComm_t nccl_cache_take(int device, int nranks, int rank) {
  if (!nccl_cache_on()) return nullptr;
  std::lock_guard<std::mutex> lk(nccl_cache_mu());
  auto& v = nccl_cache();
  for (size_t k = 0; k < v.size(); ++k) {
    if (v[k].device == device && v[k].nranks == nranks && v[k].rank == rank) {
      ncclComm_t c = v[k].comm;
      v[k] = v.back();
      v.pop_back();
      return c;
    }
  }
  return nullptr;
}
inline void nccl_cache_release_all() {
  std::lock_guard<std::mutex> lk(nccl_cache_mu());
  for (auto& e : nccl_cache()) ncclCommDestroy(e.comm);
  nccl_cache().clear();
}

struct NcclComm final : SlabComm {
  ncclComm_t nc = nullptr;
  int device = 0, nranks = 1, rank = 0;
  ~NcclComm() override {
    if (!nc) return;
    if (nccl_cache_on()) {
      std::lock_guard<std::mutex> lk(nccl_cache_mu());
      nccl_cache().push_back({device, nranks, rank, nc});
    } else {
      ncclCommDestroy(nc);
    }
  }
  static ncclDataType_t dt(CType t) {
    switch (t) {
      case CType::kI32: return ncclInt32;
      case CType::kI64: return ncclInt64;
      case CType::kU64: return ncclUint64;
      default: return ncclFloat64;
    }
  }
  void allreduce(void* buf, size_t count, CType t, COp op, cudaStream_t s) override {
    nck(ncclAllReduce(buf, buf, count, dt(t), op == COp::kSum ? ncclSum : ncclMax, nc, s),
        "ncclAllReduce");
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    nck(ncclAllGather(send, recv, bytes, ncclUint8, nc, s), "ncclAllGather");
  }
  void group_start() override { nck(ncclGroupStart(), "ncclGroupStart"); }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nck(ncclSend(buf, bytes, ncclUint8, peer, nc, s), "ncclSend");
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nck(ncclRecv(buf, bytes, ncclUint8, peer, nc, s), "ncclRecv");
  }
  void group_end(cudaStream_t) override { nck(ncclGroupEnd(), "ncclGroupEnd"); }
  bool in_process() const override { return false; }
};
#endif

// ---- in-process transport -----------------------------------------------------

// Shared by the R rank threads of one decomposition (reference-counted: the
// creator's handle plus one per attached context).
struct LocalGroup {
  explicit LocalGroup(int nranks) : R(nranks), slot(static_cast<size_t>(nranks)) {}
  const int R;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<char> taken = std::vector<char>(static_cast<size_t>(R), 0);
  struct Msg {
    int peer;
    const void* p;
    size_t bytes;
  };
  struct Slot {
    cudaEvent_t ready = nullptr, done = nullptr;  // created by the owning rank
    const void* src = nullptr;                     // all-gather / all-reduce source
    std::vector<Msg> sends;                        // this group's sends, in posting order
  };
  std::vector<Slot> slot;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw CudaFail{"slab loop: a peer rank failed"};
    const uint64_t g = gen;
    if (++arrived == R) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (gen == g) throw CudaFail{"slab loop: a peer rank failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

template <class T>
__global__ void k_local_reduce(const T* __restrict__ g, int R, size_t count, int op,
                               T* __restrict__ out) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  T acc = g[i];
  for (int q = 1; q < R; ++q) {  // fixed rank order: deterministic sums
    const T v = g[static_cast<size_t>(q) * count + i];
    acc = op == 0 ? acc + v : (v > acc ? v : acc);
  }
  out[i] = acc;
}

struct LocalComm final : SlabComm {
  std::shared_ptr<LocalGroup> grp;
  int r = 0;
  char* stage = nullptr;   // this rank's copy of an all-reduce input
  char* gather = nullptr;  // every rank's copy, rank-major
  size_t cap = 0;          // bytes per rank of stage / gather
  std::vector<LocalGroup::Msg> recvs;

  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : grp(std::move(g)), r(rank) {
    auto& me = grp->slot[static_cast<size_t>(r)];
    ck(cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming), "cudaEventCreate");
    reserve(4096);
  }
  ~LocalComm() override {
    auto& me = grp->slot[static_cast<size_t>(r)];
    if (me.ready) cudaEventDestroy(me.ready);
    if (me.done) cudaEventDestroy(me.done);
    me.ready = me.done = nullptr;
    std::lock_guard<std::mutex> lk(grp->mu);
    grp->taken[static_cast<size_t>(r)] = 0;
    cudaFree(stage);
    cudaFree(gather);
  }
  void reserve(size_t bytes) {
    if (bytes <= cap) return;
    ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");  // no peer still reads the old stage
    cudaFree(stage);
    cudaFree(gather);
    cap = std::max<size_t>(bytes, 2 * cap);
    void* a = nullptr;
    void* b = nullptr;
    ck(cudaMalloc(&a, cap), "cudaMalloc(stage)");
    ck(cudaMalloc(&b, cap * static_cast<size_t>(grp->R)), "cudaMalloc(gather)");
    stage = static_cast<char*>(a);
    gather = static_cast<char*>(b);
  }
  LocalGroup::Slot& slot(int q) { return grp->slot[static_cast<size_t>(q)]; }
  void wait_all(cudaStream_t s, bool ready) {
    for (int q = 0; q < grp->R; ++q) {
      ck(cudaStreamWaitEvent(s, ready ? slot(q).ready : slot(q).done, 0), "cudaStreamWaitEvent");
    }
  }
  // publish (sources ready) -> rendezvous -> copy in -> rendezvous -> later
  // work on this stream waits until every rank's copies out of this rank's
  // buffers ran
  template <class F>
  void exchange(cudaStream_t s, F&& copy_in) {
    ck(cudaEventRecord(slot(r).ready, s), "cudaEventRecord");
    grp->barrier();
    wait_all(s, true);
    copy_in();
    ck(cudaEventRecord(slot(r).done, s), "cudaEventRecord");
    grp->barrier();
    wait_all(s, false);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    slot(r).src = send;
    exchange(s, [&] {
      for (int q = 0; q < grp->R; ++q) {
        ck(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(q) * bytes, slot(q).src,
                           bytes, cudaMemcpyDefault, s), "allgather copy");
      }
    });
  }
  void allreduce(void* buf, size_t count, CType t, COp op, cudaStream_t s) override {
    const size_t bytes = count * ctype_bytes(t);
    reserve(bytes);
    ck(cudaMemcpyAsync(stage, buf, bytes, cudaMemcpyDeviceToDevice, s), "allreduce stage");
    slot(r).src = stage;
    exchange(s, [&] {
      for (int q = 0; q < grp->R; ++q) {
        ck(cudaMemcpyAsync(gather + static_cast<size_t>(q) * bytes, slot(q).src, bytes,
                           cudaMemcpyDefault, s), "allreduce gather");
      }
      const int blocks = static_cast<int>((count + 255) / 256);
      const int o = op == COp::kSum ? 0 : 1;
      if (blocks == 0) return;
      switch (t) {
        case CType::kI32:
          k_local_reduce<int><<<blocks, 256, 0, s>>>(reinterpret_cast<const int*>(gather), grp->R,
                                                     count, o, static_cast<int*>(buf));
          break;
        case CType::kI64:
          k_local_reduce<long long><<<blocks, 256, 0, s>>>(
              reinterpret_cast<const long long*>(gather), grp->R, count, o,
              static_cast<long long*>(buf));
          break;
        case CType::kU64:
          k_local_reduce<unsigned long long><<<blocks, 256, 0, s>>>(
              reinterpret_cast<const unsigned long long*>(gather), grp->R, count, o,
              static_cast<unsigned long long*>(buf));
          break;
        default:
          k_local_reduce<double><<<blocks, 256, 0, s>>>(reinterpret_cast<const double*>(gather),
                                                        grp->R, count, o, static_cast<double*>(buf));
      }
      ck(cudaGetLastError(), "k_local_reduce");
    });
  }
  void group_start() override {
    slot(r).sends.clear();
    recvs.clear();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t) override {
    slot(r).sends.push_back({peer, buf, bytes});
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t) override {
    recvs.push_back({peer, buf, bytes});
  }
  void group_end(cudaStream_t s) override {
    std::string err;
    exchange(s, [&] {
      // the k-th receive from q takes q's k-th send to this rank
      std::vector<size_t> next(static_cast<size_t>(grp->R), 0);
      for (const auto& m : recvs) {
        const auto& theirs = slot(m.peer).sends;
        size_t& k = next[static_cast<size_t>(m.peer)];
        while (k < theirs.size() && theirs[k].peer != r) ++k;
        if (k == theirs.size()) {
          err = "receive from rank " + std::to_string(m.peer) + " has no matching send";
          return;
        }
        if (theirs[k].bytes != m.bytes) {
          err = "message size mismatch from rank " + std::to_string(m.peer) + ": " +
                std::to_string(theirs[k].bytes) + " vs " + std::to_string(m.bytes) + " bytes";
          return;
        }
        ck(cudaMemcpyAsync(const_cast<void*>(m.p), theirs[k].p, m.bytes, cudaMemcpyDefault, s),
           "p2p copy");
        ++k;
      }
      for (int q = 0; q < grp->R; ++q) {  // every send to this rank was received
        const auto& theirs = slot(q).sends;
        for (size_t k = next[static_cast<size_t>(q)]; k < theirs.size(); ++k) {
          if (theirs[k].peer == r) {
            err = "unmatched send from rank " + std::to_string(q);
            return;
          }
        }
      }
    });
    // (raised after the second rendezvous, so no peer is left waiting in it)
    if (!err.empty()) throw CudaFail{"slab loop: " + err};
  }
  void abort() override { grp->abort(); }
  bool in_process() const override { return true; }
};

// Cross-process transport over a shared file mapping (test path, see the
// header). Layout: a 4 KB header {arrivals, generation, abort}, one 1 MB slot
// per rank for collectives, one mailbox per ordered rank pair for point-to-
// point messages (a message table, then the payloads in posting order).
struct HostFileComm final : SlabComm {
  static constexpr size_t kHeader = 4096;
  static constexpr size_t kSlot = size_t{1} << 20;
  static constexpr size_t kBox = size_t{32} << 20;
  static constexpr int kMaxMsgs = 64;
  struct Pending {
    void* p;
    size_t bytes;
    int peer;
  };
  int rank = 0, nranks = 1;
  char* base = nullptr;
  size_t mapped = 0;
  std::vector<Pending> sends, recvs;

  HostFileComm(const char* path, int r, int R) : rank(r), nranks(R) {
    mapped = kHeader + static_cast<size_t>(R) * kSlot + static_cast<size_t>(R) * R * kBox;
    const int fd = ::open(path, O_RDWR | O_CREAT, 0600);
    if (fd < 0) throw CudaFail{std::string("host transport: cannot open ") + path};
    struct stat st {};
    if (::fstat(fd, &st) != 0 ||
        (static_cast<size_t>(st.st_size) < mapped && ::ftruncate(fd, static_cast<off_t>(mapped)) != 0)) {
      ::close(fd);
      throw CudaFail{"host transport: cannot size the mapping"};
    }
    void* m = ::mmap(nullptr, mapped, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (m == MAP_FAILED) throw CudaFail{"host transport: mmap failed"};
    base = static_cast<char*>(m);
  }
  ~HostFileComm() override {
    if (base) ::munmap(base, mapped);
  }
  int* word(int k) { return reinterpret_cast<int*>(base) + k; }  // 0 arrivals, 1 gen, 2 abort
  char* slot(int q) { return base + kHeader + static_cast<size_t>(q) * kSlot; }
  char* box(int src, int dst) {
    return base + kHeader + static_cast<size_t>(nranks) * kSlot +
           (static_cast<size_t>(src) * nranks + dst) * kBox;
  }
  void barrier() {
    const int g = __atomic_load_n(word(1), __ATOMIC_ACQUIRE);
    if (__atomic_add_fetch(word(0), 1, __ATOMIC_ACQ_REL) == nranks) {
      __atomic_store_n(word(0), 0, __ATOMIC_RELAXED);
      __atomic_add_fetch(word(1), 1, __ATOMIC_RELEASE);
      return;
    }
    while (__atomic_load_n(word(1), __ATOMIC_ACQUIRE) == g) {
      if (__atomic_load_n(word(2), __ATOMIC_ACQUIRE)) throw CudaFail{"a peer rank failed"};
      sched_yield();
    }
  }
  static void sync(cudaStream_t s) { ck(cudaStreamSynchronize(s), "cudaStreamSynchronize"); }
  // Copies on the context stream, completed before returning (the shared
  // pages are pageable host memory: a plain cudaMemcpy H2D may return before
  // its DMA lands, and the context stream does not order after it).
  static void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind k, cudaStream_t s,
                   const char* what) {
    ck(cudaMemcpyAsync(dst, src, bytes, k, s), what);
    sync(s);
  }
  void allreduce(void* buf, size_t count, CType t, COp op, cudaStream_t s) override {
    const size_t bytes = count * ctype_bytes(t);
    if (bytes > kSlot) throw CudaFail{"host transport: all-reduce too large"};
    sync(s);
    copy(slot(rank), buf, bytes, cudaMemcpyDeviceToHost, s, "D2H all-reduce");
    barrier();
    std::vector<char> acc(slot(0), slot(0) + bytes);
    for (int q = 1; q < nranks; ++q) {  // fixed rank order
      const char* v = slot(q);
      for (size_t k = 0; k < count; ++k) {
        switch (t) {
          case CType::kI32: {
            auto* a = reinterpret_cast<int32_t*>(acc.data()) + k;
            const int32_t b = reinterpret_cast<const int32_t*>(v)[k];
            *a = op == COp::kSum ? *a + b : std::max(*a, b);
            break;
          }
          case CType::kI64: {
            auto* a = reinterpret_cast<int64_t*>(acc.data()) + k;
            const int64_t b = reinterpret_cast<const int64_t*>(v)[k];
            *a = op == COp::kSum ? *a + b : std::max(*a, b);
            break;
          }
          case CType::kU64: {
            auto* a = reinterpret_cast<uint64_t*>(acc.data()) + k;
            const uint64_t b = reinterpret_cast<const uint64_t*>(v)[k];
            *a = op == COp::kSum ? *a + b : std::max(*a, b);
            break;
          }
          default: {
            auto* a = reinterpret_cast<double*>(acc.data()) + k;
            const double b = reinterpret_cast<const double*>(v)[k];
            *a = op == COp::kSum ? *a + b : std::max(*a, b);
          }
        }
      }
    }
    copy(buf, acc.data(), bytes, cudaMemcpyHostToDevice, s, "H2D all-reduce");
    barrier();  // the slots are free again
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (bytes > kSlot) throw CudaFail{"host transport: all-gather too large"};
    sync(s);
    copy(slot(rank), send, bytes, cudaMemcpyDeviceToHost, s, "D2H all-gather");
    barrier();
    for (int q = 0; q < nranks; ++q) {
      ck(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(q) * bytes, slot(q),
                         bytes, cudaMemcpyHostToDevice, s), "H2D all-gather");
    }
    sync(s);
    barrier();
  }
  void group_start() override {
    sends.clear();
    recvs.clear();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t) override {
    sends.push_back({const_cast<void*>(buf), bytes, peer});
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t) override {
    recvs.push_back({buf, bytes, peer});
  }
  // mailbox (src -> dst): int count, size_t sizes[kMaxMsgs], payloads in order
  static size_t* sizes_of(char* b) { return reinterpret_cast<size_t*>(b + 64); }
  static char* data_of(char* b) { return b + 64 + kMaxMsgs * sizeof(size_t); }
  void group_end(cudaStream_t s) override {
    sync(s);
    for (int d = 0; d < nranks; ++d) *reinterpret_cast<int*>(box(rank, d)) = 0;
    std::vector<size_t> fill(static_cast<size_t>(nranks), 0);
    for (const Pending& m : sends) {
      char* b = box(rank, m.peer);
      int& n = *reinterpret_cast<int*>(b);
      size_t& f = fill[static_cast<size_t>(m.peer)];
      if (n >= kMaxMsgs || 64 + kMaxMsgs * sizeof(size_t) + f + m.bytes > kBox) {
        throw CudaFail{"host transport: mailbox full"};
      }
      sizes_of(b)[n++] = m.bytes;
      if (m.bytes) {
        ck(cudaMemcpyAsync(data_of(b) + f, m.p, m.bytes, cudaMemcpyDeviceToHost, s),
           "D2H message");
      }
      f += m.bytes;
    }
    sync(s);
    barrier();
    std::string err;
    std::vector<int> next(static_cast<size_t>(nranks), 0);
    std::vector<size_t> off(static_cast<size_t>(nranks), 0);
    for (const Pending& m : recvs) {
      char* b = box(m.peer, rank);
      const int n = *reinterpret_cast<int*>(b);
      int& k = next[static_cast<size_t>(m.peer)];
      if (k >= n) {
        err = "receive from rank " + std::to_string(m.peer) + " has no matching send";
        break;
      }
      if (sizes_of(b)[k] != m.bytes) {
        err = "message size mismatch from rank " + std::to_string(m.peer);
        break;
      }
      if (m.bytes) {
        ck(cudaMemcpyAsync(m.p, data_of(b) + off[static_cast<size_t>(m.peer)], m.bytes,
                           cudaMemcpyHostToDevice, s), "H2D message");
      }
      off[static_cast<size_t>(m.peer)] += m.bytes;
      ++k;
    }
    sync(s);
    for (int q = 0; q < nranks && err.empty(); ++q) {
      if (next[static_cast<size_t>(q)] != *reinterpret_cast<int*>(box(q, rank))) {
        err = "unmatched send from rank " + std::to_string(q);
      }
    }
    barrier();  // (errors raised after it: no peer is left waiting)
    if (!err.empty()) throw CudaFail{"slab loop: " + err};
  }
  void abort() override { __atomic_store_n(word(2), 1, __ATOMIC_RELEASE); }
  bool in_process() const override { return false; }
};

}  // namespace
