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
// Backends: NCCL (dlopen'ed torch-bundled libnccl.so.2; one ncclGroupStart/End around the SUM and the
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

struct Comm {
  virtual ~Comm() {}
  // In-place grouped all-reduce: SUM of nsum doubles, MAX of nmax u64, as one collective call.
  virtual bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                         std::string* why) = 0;
  virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
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
  }
};

struct LoopComm : Comm {
  LoopGroup* g = nullptr;
  int rank = 0;
  bool allreduce(double* sum, size_t nsum, unsigned long long* mx, size_t nmax, cudaStream_t st,
                 std::string* why) override {
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->arrived == 0) {
      g->nsum = nsum;
      g->nmax = nmax;
      g->err.clear();
    } else if (g->nsum != nsum || g->nmax != nmax) {
      g->err = "loopback: ranks called the collective with different sizes";
    }
    g->ptrs.sum[rank] = sum;
    g->ptrs.mx[rank] = mx;
    cudaEventRecord(g->ready[rank], st);
    const long long gen = g->generation;
    if (++g->arrived == g->world) {  // last to arrive: reduce on this stream, release the others
      if (g->err.empty()) {
        for (int r = 0; r < g->world; ++r) cudaStreamWaitEvent(st, g->ready[r], 0);
        const size_t n = nsum > nmax ? nsum : nmax;
        const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
        k_loop_reduce<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(g->ptrs, g->world, nsum, nmax);
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
