// Multi-GPU combine of the per-restart partials: each rank evaluates a
// contiguous slice of the (restart, channel, Doppler-chunk) groups; the library then
// runs, per evaluation,
//   1. grouped all-reduce MAX of {shift m (f64), packed max keys (u64)}   [R x 3]
//   2. local rescale S <- S e^{beta (m_local - m)} (or (m_local/m)^p)     (tiny kernel)
//   3. all-reduce SUM of S                                                 [R]
//   4. (gradients) all-reduce SUM of the normalized gradient partial      [R][M][N] c64
// NCCL is dlopen'ed (the torch-bundled libnccl.so.2, same process as torch's own), so the
// library links and runs on one GPU without it.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <string>

#ifndef SQNGD_NCCL_PATH
#define SQNGD_NCCL_PATH "libnccl.so.2"
#endif

namespace sq {

struct RedRescale {  // mirrors Red (misc_kernels.cuh) for the S rescale kernel
  double m, S;
  unsigned long long key_a, key_c;
};

__global__ void k_red_pack(int R, const RedRescale* red, double* mbuf, unsigned long long* kbuf) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  mbuf[r] = red[r].m;
  kbuf[2 * r] = red[r].key_a;
  kbuf[2 * r + 1] = red[r].key_c;
}

__global__ void k_red_rescale(int R, int mode, double bp, RedRescale* red, const double* mglob,
                              const unsigned long long* kglob, double* sbuf) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double ml = red[r].m, mg = mglob[r];
  double S = red[r].S;
  if (!(S > 0.0) || !(ml > -INFINITY)) S = 0.0;
  else S *= (mode == 1) ? exp(bp * (ml - mg)) : pow(ml / mg, bp);
  sbuf[r] = S;
  red[r].m = mg;
  red[r].key_a = kglob[2 * r];
  red[r].key_c = kglob[2 * r + 1];
}

__global__ void k_red_unpack(int R, RedRescale* red, const double* sbuf) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) red[r].S = sbuf[r];
}

struct Comm {
  typedef int (*fn_init)(void**, int, const void*, int);  // ncclCommInitRank(comm*, nranks, id (by value), rank)
  void* lib = nullptr;
  void* comm = nullptr;
  int world = 1;
  // ncclResult_t ncclAllReduce(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t)
  int (*allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  int (*destroy_fn)(void*) = nullptr;
  const char* (*errstr)(int) = nullptr;
  double* mbuf = nullptr;              // [R]
  unsigned long long* kbuf = nullptr;  // [R][2]
  double* sbuf = nullptr;              // [R]
  int cap = 0;

  enum { kUint64 = 5, kFloat32 = 7, kFloat64 = 8, kSum = 0, kMax = 2 };
  struct UniqueId { char internal[128]; };

  bool init(const void* uid, int rank, int nranks, std::string* why) {
    world = nranks;
    lib = dlopen(SQNGD_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) { *why = "dlopen libnccl.so.2 failed"; return false; }
    typedef int (*fn_init_v)(void**, int, UniqueId, int);
    fn_init_v initr = (fn_init_v)dlsym(lib, "ncclCommInitRank");
    allreduce = (decltype(allreduce))dlsym(lib, "ncclAllReduce");
    group_start = (decltype(group_start))dlsym(lib, "ncclGroupStart");
    group_end = (decltype(group_end))dlsym(lib, "ncclGroupEnd");
    destroy_fn = (decltype(destroy_fn))dlsym(lib, "ncclCommDestroy");
    errstr = (decltype(errstr))dlsym(lib, "ncclGetErrorString");
    if (!initr || !allreduce || !group_start || !group_end || !destroy_fn) { *why = "missing NCCL symbols"; return false; }
    UniqueId id;
    memcpy(&id, uid, sizeof(id));
    int rc = initr(&comm, nranks, id, rank);
    if (rc != 0) { *why = errstr ? errstr(rc) : "ncclCommInitRank"; return false; }
    return true;
  }
  bool ensure(int R) {
    if (R <= cap) return true;
    if (mbuf) { cudaFree(mbuf); cudaFree(kbuf); cudaFree(sbuf); }
    if (cudaMalloc(&mbuf, sizeof(double) * R) || cudaMalloc(&kbuf, sizeof(unsigned long long) * 2 * R) ||
        cudaMalloc(&sbuf, sizeof(double) * R))
      return false;
    cap = R;
    return true;
  }
  bool check(int rc, std::string* why) {
    if (rc != 0) { *why = errstr ? errstr(rc) : "nccl error"; return false; }
    return true;
  }
  template <class RedT>
  bool reduce_red(RedT* red, int R, int mode, double bp, cudaStream_t st, std::string* why) {
    if (!ensure(R)) { *why = "alloc"; return false; }
    RedRescale* rr = reinterpret_cast<RedRescale*>(red);
    k_red_pack<<<(R + 127) / 128, 128, 0, st>>>(R, rr, mbuf, kbuf);
    if (!check(group_start(), why)) return false;
    if (!check(allreduce(mbuf, mbuf, R, kFloat64, kMax, comm, st), why)) return false;
    if (!check(allreduce(kbuf, kbuf, 2 * R, kUint64, kMax, comm, st), why)) return false;
    if (!check(group_end(), why)) return false;
    k_red_rescale<<<(R + 127) / 128, 128, 0, st>>>(R, mode, bp, rr, mbuf, kbuf, sbuf);
    if (!check(allreduce(sbuf, sbuf, R, kFloat64, kSum, comm, st), why)) return false;
    k_red_unpack<<<(R + 127) / 128, 128, 0, st>>>(R, rr, sbuf);
    return cudaGetLastError() == cudaSuccess;
  }
  bool sum_f32(float* buf, size_t n, cudaStream_t st, std::string* why) {
    return check(allreduce(buf, buf, n, kFloat32, kSum, comm, st), why);
  }
  void destroy() {
    if (comm && destroy_fn) destroy_fn(comm);
    comm = nullptr;
    if (mbuf) { cudaFree(mbuf); cudaFree(kbuf); cudaFree(sbuf); }
    mbuf = nullptr;
  }
};

}  // namespace sq
