// Multi-GPU combine of the per-restart partials (DESIGN.md §7 "Multi-GPU").
//
// Each rank evaluates its shard (FFT engine: a contiguous slice of the (restart, channel, bin) units;
// Chebyshev engine: a contiguous slice of the (restart, transmit channel) rows) and reduces it locally
// to (m_r, S_r, keys, normalised gradient partial g_r).  ONE grouped collective per evaluation then
// combines the ranks:
//   SUM over ranks of  [ wS_r | wG_r g_r ]   (fp64, per restart: 1 + 2 M N values)
//   MAX over ranks of  [ key_auto | key_cross | bits(m_r) ]   (u64)
// with the weights taken against a reference shift m_ref that every rank holds identically (the
// previous evaluation's global maximum):
//   LSE:    wS_r = wG_r = e^{beta (m_r - m_ref)} S_r,                  g = sum wG g / sum wS
//   p-norm: wS_r = (m_r / m_ref)^p S_r, wG_r = (m_r / m_ref)^{p-1} S_r^{1-1/p},
//           g = (sum wS)^{1/p - 1} sum wG g
// The fp64 weights cannot overflow for beta |m_r - m_ref| < 700, so the combine is exact (no second
// round); the restart's loss is m_ref + ln(sum wS) / beta (LSE) or m_ref (sum wS)^{1/p}.
//
// Backends: PEER (below: the collective as one kernel of this library over NVLink peer memory, selected by
// sqngd_peer_export / sqngd_peer_attach; world_peer.cuh fuses pack and unpack into it),
// NCCL (dlopen'ed torch-bundled libnccl.so.2; one ncclGroupStart/End around the SUM and the
// MAX all-reduce; capturable into the step's CUDA graph), and a single-device LOOPBACK group for tests:
// the W contexts of one process, each driven by its own host thread, meet in a host barrier; the last
// to arrive makes its stream wait for every rank's event, sums / maxes the W buffers in one kernel
// (fixed rank order) and records an event that every rank's stream waits on.  No kernel waits on
// another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#ifndef SQNGD_NCCL_PATH
#define SQNGD_NCCL_PATH "libnccl.so.2"
#endif

namespace sq {

struct WorldArgs;  // misc_kernels.cuh

struct Comm {
  virtual ~Comm() {}
  // In-place grouped all-reduce: SUM of nsum doubles, MAX of nmax u64, as one collective call.
  virtual bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                         std::string* why) = 0;
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
  // Optional: the whole combine (pack, all-reduce, unpack) as ONE kernel (world_peer.cuh).
  virtual bool has_fused() const { return false; }
  virtual bool fused(const WorldArgs*, cudaStream_t, std::string*) { return false; }
  virtual void destroy() {}
};

struct NcclComm : Comm {
  void* lib = nullptr;
  void* comm = nullptr;
  int (*allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  int (*destroy_fn)(void*) = nullptr;
  const char* (*errstr)(int) = nullptr;
  enum { kUint64 = 5, kFloat64 = 8, kSum = 0, kMax = 2 };
  struct UniqueId { char internal[128]; };

  bool init(const void* uid, int rank, int nranks, std::string* why) {
    lib = dlopen(SQNGD_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) { *why = "dlopen libnccl.so.2 failed"; return false; }
    typedef int (*fn_init_v)(void**, int, UniqueId, int);
    fn_init_v initr = (fn_init_v)dlsym(lib, "ncclCommInitRank");
    allreduce_fn = (decltype(allreduce_fn))dlsym(lib, "ncclAllReduce");
    group_start = (decltype(group_start))dlsym(lib, "ncclGroupStart");
    group_end = (decltype(group_end))dlsym(lib, "ncclGroupEnd");
    destroy_fn = (decltype(destroy_fn))dlsym(lib, "ncclCommDestroy");
    errstr = (decltype(errstr))dlsym(lib, "ncclGetErrorString");
    if (!initr || !allreduce_fn || !group_start || !group_end || !destroy_fn) { *why = "missing NCCL symbols"; return false; }
    UniqueId id;
    memcpy(&id, uid, sizeof(id));
    const int rc = initr(&comm, nranks, id, rank);
    if (rc != 0) { *why = errstr ? errstr(rc) : "ncclCommInitRank"; return false; }
    return true;
  }
  bool check(int rc, std::string* why) {
    if (rc != 0) { *why = errstr ? errstr(rc) : "nccl error"; return false; }
    return true;
  }
  bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                 std::string* why) override {
    if (!check(group_start(), why)) return false;
    if (nsum && !check(allreduce_fn(sum, sum, nsum, kFloat64, kSum, comm, st), why)) return false;
    if (nmax && !check(allreduce_fn(mx, mx, nmax, kUint64, kMax, comm, st), why)) return false;
    return check(group_end(), why);
  }
  bool capturable() const override { return true; }
  void destroy() override {
    if (comm && destroy_fn) destroy_fn(comm);
    comm = nullptr;
  }
};

// ------------------------------------------------------------------------------- peer memory
// The same grouped all-reduce as ONE kernel of our own over NVLink peer memory (SURVEY §8(f) NEXT-4,
// DESIGN.md §7 "In-kernel all-reduce").  Every rank owns a WINDOW (one cudaMalloc, exported with
// cudaIpcGetMemHandle and mapped by its peers):
//   [ epoch[kPeerBlocks] | flag[kPeerMax][kPeerBlocks] | stage[2][cap_sum doubles + cap_max u64] ]
// Block b of k_peer_allreduce owns slice b of the payload on every rank (same grid on every rank):
//   phase A  e = epoch[b] + 1;  copy slice b of (sum, mx) into the own stage[e & 1];  fence;  store e
//            into flag[rank][b] of EVERY rank's window (st.release.sys over NVLink);
//   phase B  wait until the own flag[r][b] >= e for every r (ld.acquire.sys, clock watchdog);  read slice b
//            of every rank's stage[e & 1] (own rank locally, peers over NVLink, ld.global.cg) and write
//            sum_r / max_r in RANK ORDER into the caller's buffers (bit-identical on every rank);
//            epoch[b] = e.
// A peer can be at most one epoch ahead (its epoch e + 1 wait needs this rank's e + 1 signal), so the two
// stage parities suffice and the flags only grow.  No host-side argument changes between calls (the
// epoch lives in the window), so the launch replays inside the step's CUDA graph.  A block waits only on
// the same-numbered block of its peers, never on a block of its own grid.
constexpr int kPeerMax = 8;
constexpr int kPeerBlocks = 128;
constexpr int kPeerThreads = 512;  // 128 x 512 threads x 4 loads in flight cover the HBM latency-bandwidth product
struct PeerArgs {
  unsigned char* win[kPeerMax];  // every rank's window, as mapped into this process
  int world, rank;
  size_t cap_sum, cap_max;       // stage capacity (elements), identical on every rank
  int* status;                   // the context's latched device status (bit 16: peer wait timed out)
};
__host__ __device__ inline size_t peer_flags_bytes() { return sizeof(unsigned long long) * (size_t)(1 + kPeerMax) * kPeerBlocks; }
__host__ __device__ inline size_t peer_stage_bytes(size_t cap_sum, size_t cap_max) { return 8 * (cap_sum + cap_max); }
__host__ __device__ inline size_t peer_window_bytes(size_t cap_sum, size_t cap_max) {
  return peer_flags_bytes() + 2 * peer_stage_bytes(cap_sum, cap_max);
}
constexpr int kPeerPhaseA = 1, kPeerPhaseB = 2;
constexpr int kPeerTimeoutBit = 1 << 16;

__device__ __forceinline__ void peer_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long peer_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kPeerThreads) k_peer_allreduce(PeerArgs a, double* sum, size_t nsum, unsigned long long* mx,
                                                        size_t nmax, int phases, unsigned long long timeout_ns) {
  typedef unsigned long long u64;
  const int b = blockIdx.x, nb = gridDim.x, t = threadIdx.x;
  u64* own = reinterpret_cast<u64*>(a.win[a.rank]);
  const u64 e = own[b] + 1;  // epoch[b]: written only by this block's previous launch
  const size_t stage_off = peer_flags_bytes() + (size_t)(e & 1) * peer_stage_bytes(a.cap_sum, a.cap_max);
  const size_t cs = (nsum + nb - 1) / nb, cm = (nmax + nb - 1) / nb;
  const size_t s0 = min(nsum, (size_t)b * cs), s1 = min(nsum, s0 + cs);
  const size_t m0 = min(nmax, (size_t)b * cm), m1 = min(nmax, m0 + cm);
  if (phases & kPeerPhaseA) {
    u64* st_sum = reinterpret_cast<u64*>(a.win[a.rank] + stage_off);
    u64* st_max = st_sum + a.cap_sum;
    const u64* src = reinterpret_cast<const u64*>(sum);
#pragma unroll 4
    for (size_t i = s0 + t; i < s1; i += blockDim.x) st_sum[i] = src[i];
    for (size_t i = m0 + t; i < m1; i += blockDim.x) st_max[i] = mx[i];
    // the block's stage writes happen-before the barrier; the signalling threads' release at system
    // scope is cumulative over them (the pattern of a grid barrier: bar.sync, then one fence + flag)
    __syncthreads();
    if (t < a.world)
      peer_st_release(reinterpret_cast<u64*>(a.win[t]) + (size_t)(1 + a.rank) * kPeerBlocks + b, e);
  }
  if (phases & kPeerPhaseB) {
    __shared__ int timed_out;
    if (t == 0) timed_out = 0;
    __syncthreads();
    if (t < a.world) {
      const u64* f = own + (size_t)(1 + t) * kPeerBlocks + b;
      u64 t0 = 0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (peer_ld_acquire(f) < e) {
        u64 t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > timeout_ns) {  // a peer never signalled: latch the error, do not hang the GPU
          timed_out = 1;
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
    if (timed_out) {
      if (t == 0) atomicOr(a.status, kPeerTimeoutBit);
      return;  // epoch[b] is not advanced: the context is unusable after a timeout (sqngd_sync reports it)
    }
    // (the acquires above, then the barrier, order these loads after the peers' stage writes; .cg: L2)
#pragma unroll 4
    for (size_t i = s0 + t; i < s1; i += blockDim.x) {
      double s = 0.0;
      for (int r = 0; r < a.world; ++r)  // fixed rank order
        s += __ldcg(reinterpret_cast<const double*>(a.win[r] + stage_off) + i);
      sum[i] = s;
    }
    for (size_t i = m0 + t; i < m1; i += blockDim.x) {
      u64 m = 0ull;
      for (int r = 0; r < a.world; ++r) {
        const u64 v = __ldcg(reinterpret_cast<const u64*>(a.win[r] + stage_off) + a.cap_sum + i);
        m = v > m ? v : m;
      }
      mx[i] = m;
    }
    __syncthreads();
    if (t == 0) own[b] = e;
  }
}

inline int peer_grid(size_t nsum, size_t nmax) {
  const size_t n = nsum > nmax ? nsum : nmax;
  const size_t g = (n + 1023) / 1024;  // >= 4 elements per thread before another block is worth its flags
  return (int)(g < 1 ? 1 : (g > (size_t)kPeerBlocks ? (size_t)kPeerBlocks : g));
}

// One rank's window: allocated zeroed (epoch 0, flags 0), exported / attached through CUDA IPC.
struct PeerWindow {
  unsigned char* base = nullptr;
  size_t cap_sum = 0, cap_max = 0;
  cudaError_t alloc(size_t cs, size_t cm) {
    cap_sum = cs;
    cap_max = cm;
    cudaError_t e = cudaMalloc(&base, peer_window_bytes(cs, cm));
    if (e != cudaSuccess) return e;
    return cudaMemset(base, 0, peer_window_bytes(cs, cm));
  }
  void release() {
    if (base) cudaFree(base);
    base = nullptr;
  }
};

struct PeerComm : Comm {
  PeerWindow own;
  PeerArgs args{};
  bool opened[kPeerMax] = {};
  unsigned long long timeout_ns = 30ull * 1000000000ull;
  bool use_fused = true;  // fixed at attach: the fused and the 3-launch form must not share a window
  bool has_fused() const override { return use_fused; }
  bool fused(const WorldArgs* wa, cudaStream_t st, std::string* why) override;  // world_peer.cuh
  // handles: world x CUDA_IPC_HANDLE_SIZE bytes, rank-major, every rank's exported window (this rank's
  // own entry is ignored: the local pointer is used).
  bool attach(const void* handles, int rank, int world, int* status, std::string* why) {
    if (world < 1 || world > kPeerMax || !own.base) { *why = "peer attach: world outside 1..8 or no window"; return false; }
    args.world = world;
    args.rank = rank;
    args.cap_sum = own.cap_sum;
    args.cap_max = own.cap_max;
    args.status = status;
    for (int r = 0; r < world; ++r) {
      if (r == rank) { args.win[r] = own.base; continue; }
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)handles + (size_t)r * sizeof(h), sizeof(h));
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) { *why = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e); return false; }
      args.win[r] = (unsigned char*)p;
      opened[r] = true;
    }
    return true;
  }
  bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                 std::string* why) override {
    if (nsum > own.cap_sum || nmax > own.cap_max) { *why = "peer all-reduce: payload larger than the window"; return false; }
    k_peer_allreduce<<<peer_grid(nsum, nmax), kPeerThreads, 0, st>>>(args, sum, nsum, mx, nmax, kPeerPhaseA | kPeerPhaseB, timeout_ns);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { *why = cudaGetErrorString(e); return false; }
    return true;
  }
  bool capturable() const override { return true; }
  void destroy() override {
    for (int r = 0; r < kPeerMax; ++r)
      if (opened[r]) { cudaIpcCloseMemHandle(args.win[r]); opened[r] = false; }
    own.release();
  }
};

// ------------------------------------------------------------------------------- loopback
constexpr int kLoopMax = 8;
struct LoopPtrs {
  double* sum[kLoopMax];
  unsigned long long* mx[kLoopMax];
};
__global__ void k_loop_reduce(LoopPtrs p, int world, size_t nsum, size_t nmax) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nsum; i += stride) {
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += p.sum[r][i];  // fixed rank order
    for (int r = 0; r < world; ++r) p.sum[r][i] = s;
  }
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nmax; i += stride) {
    unsigned long long m = 0ull;
    for (int r = 0; r < world; ++r) m = p.mx[r][i] > m ? p.mx[r][i] : m;
    for (int r = 0; r < world; ++r) p.mx[r][i] = m;
  }
}

struct LoopGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  LoopPtrs ptrs{};
  cudaEvent_t ready[kLoopMax] = {};
  cudaEvent_t done = nullptr;
  size_t nsum = 0, nmax = 0;
  std::string err;
  // peer mode (sqngd_loopback_set_peer): the reduction is k_peer_allreduce itself, phase A for every
  // rank and then phase B for every rank on one stream (every wait is already satisfied: no kernel waits
  // on another rank's kernel), over windows of the W contexts on this device.
  bool peer = false;
  bool peer_fused = false;                   // (peer) the whole combine in k_world_peer, phase by phase
  const WorldArgs* wargs[kLoopMax] = {};     // (peer_fused) every rank's combine arguments
  int drop_signal_rank = -1;                 // (tests) this rank's phase A is not launched: the watchdog path
  PeerWindow win[kLoopMax];
  int* status[kLoopMax] = {};
  size_t cap_sum = 0, cap_max = 0;  // window capacity: the contexts' largest payload
  bool init(int w) {
    world = w;
    for (int r = 0; r < w; ++r)
      if (cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming) != cudaSuccess) return false;
    return cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess;
  }
  ~LoopGroup() {
    for (int r = 0; r < world; ++r)
      if (ready[r]) cudaEventDestroy(ready[r]);
    if (done) cudaEventDestroy(done);
    for (int r = 0; r < world; ++r) win[r].release();
  }
};

struct LoopComm : Comm {
  LoopGroup* g = nullptr;
  int rank = 0;
  int* status = nullptr;
  size_t cap_sum = 0, cap_max = 0;
  bool has_fused() const override { return g->peer && g->peer_fused; }
  bool fused(const WorldArgs* wa, cudaStream_t st, std::string* why) override;  // world_peer.cuh
  bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                 std::string* why) override {
    std::unique_lock<std::mutex> lk(g->mu);
    if (cap_sum > g->cap_sum) g->cap_sum = cap_sum;
    if (cap_max > g->cap_max) g->cap_max = cap_max;
    if (g->arrived == 0) {
      g->nsum = nsum;
      g->nmax = nmax;
      g->err.clear();
    } else if (g->nsum != nsum || g->nmax != nmax) {
      g->err = "loopback: ranks called the collective with different sizes";
    }
    g->ptrs.sum[rank] = sum;
    g->ptrs.mx[rank] = mx;
    g->status[rank] = status;
    cudaEventRecord(g->ready[rank], st);
    const long long gen = g->generation;
    if (++g->arrived == g->world) {  // last to arrive: reduce on this stream, release the others
      if (g->err.empty()) {
        for (int r = 0; r < g->world; ++r) cudaStreamWaitEvent(st, g->ready[r], 0);
        const size_t n = nsum > nmax ? nsum : nmax;
        const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
        if (g->peer) {
          for (int r = 0; r < g->world && g->err.empty(); ++r)
            if (!g->win[r].base && g->win[r].alloc(g->cap_sum, g->cap_max) != cudaSuccess)
              g->err = "loopback: peer window allocation";
          if (g->err.empty() && (nsum > g->win[0].cap_sum || nmax > g->win[0].cap_max))
            g->err = "loopback: payload larger than the peer windows";
          for (int ph = kPeerPhaseA; ph <= kPeerPhaseB && g->err.empty(); ph <<= 1)
            for (int r = 0; r < g->world; ++r) {
              PeerArgs a{};
              for (int q = 0; q < g->world; ++q) a.win[q] = g->win[q].base;
              a.world = g->world;
              a.rank = r;
              a.cap_sum = g->win[0].cap_sum;
              a.cap_max = g->win[0].cap_max;
              a.status = g->status[r];
              k_peer_allreduce<<<peer_grid(nsum, nmax), kPeerThreads, 0, st>>>(a, g->ptrs.sum[r], nsum, g->ptrs.mx[r], nmax, ph,
                                                                       2000000000ull);
            }
        } else {
          k_loop_reduce<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(g->ptrs, g->world, nsum, nmax);
        }
        cudaEventRecord(g->done, st);
      }
      g->arrived = 0;
      ++g->generation;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->generation != gen; });
      if (g->err.empty()) cudaStreamWaitEvent(st, g->done, 0);
    }
    if (!g->err.empty()) { *why = g->err; return false; }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { *why = cudaGetErrorString(e); return false; }
    return true;
  }
  bool capturable() const override { return false; }
};

}  // namespace sq
