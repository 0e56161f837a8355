// Microbenchmark + layout check of the tcgen05 pieces the Chebyshev contraction needs on sm_100a:
//   1. D[128 x N] = A[128 x K] . B[N x K]^T, kind::tf32, A and B in shared memory (K-major, no swizzle,
//      core matrices of 8 rows x 16 B: element (r, k) at (r % 8) * 16 + (r / 8) * SBO + (k / 4) * LBO +
//      (k % 4) * 4), D in TMEM; checked against a CPU product.
//   2. the same with A in TMEM (written by tcgen05.st: lane = row, column = k).
//   3. tcgen05.ld / tcgen05.st throughput with 16 warps (bytes per SM cycle).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tcgen05 tools/ubench_tcgen05.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e = (x);                                                                           \
    if (e != cudaSuccess) {                                                                        \
      printf("CUDA %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__);                      \
      exit(1);                                                                                     \
    }                                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

constexpr int M = 128, K = 32, NN = 32;

// mode 0: A, B in smem; mode 1: A in TMEM (columns 64..64+K), B in smem.
__global__ void k_check(const float* A, const float* B, float* D, int mode) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[NN * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical K-major no-swizzle: LBO = 128 B (next 4 k), SBO = (K / 4) * 128 B (next 8 rows)
  const uint32_t LBO = 128, SBO_A = (K / 4) * 128, SBO_B = (K / 4) * 128;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sA[((r % 8) * 16 + (r / 8) * SBO_A + (k / 4) * LBO + (k % 4) * 4) / 4] = A[i];
  }
  for (int i = tid; i < NN * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sB[((r % 8) * 16 + (r / 8) * SBO_B + (k / 4) * LBO + (k % 4) * 4) / 4] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  if (mode == 1) {  // A into TMEM columns 64..64+K: warp w writes lanes 32 w.. (4 warps)
    float v[16];
    for (int c = 0; c < K; c += 16) {
      for (int i = 0; i < 16; ++i) v[i] = A[(32 * warp + lane) * K + c + i];
      st16(tb + ((uint32_t)(32 * warp) << 16) + 64 + c, v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, NN);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t bd = desc_kmajor(smem_u32(sB) + ks * 2 * LBO, LBO, SBO_B);
      if (mode == 0) {
        const uint64_t ad = desc_kmajor(smem_u32(sA) + ks * 2 * LBO, LBO, SBO_A);
        mma_ss(tb, ad, bd, id, ks > 0);
      } else {
        mma_ts(tb, tb + 64 + ks * 8, bd, id, ks > 0);
      }
    }
    commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  float v[16];
  for (int c = 0; c < NN; c += 16) {
    ld16(tb + ((uint32_t)(32 * warp) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[(32 * warp + lane) * NN + c + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

// TMEM load / store throughput: every warp repeatedly loads (or stores) 16 columns of its lane quarter.
__global__ void k_tput(int iters, int store, float* sink, long long* cyc) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase + ((uint32_t)(32 * (warp % 4)) << 16) + 16 * (warp / 4);
  float v[16], acc = 0.f;
  for (int i = 0; i < 16; ++i) v[i] = (float)i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = tb + 128 * (it & 1);
    if (store) {
      v[0] = (float)it;
      st16(a, v);
    } else {
      ld16(a, v);
      acc += v[it & 15];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + tid] = acc + v[3];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  std::vector<float> A(M * K), B(NN * K), D(M * NN), ref(M * NN);
  srand(3);
  for (auto& x : A) x = (float)(rand() % 17 - 8) * 0.25f;  // exact in tf32
  for (auto& x : B) x = (float)(rand() % 13 - 6) * 0.5f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      ref[m * NN + n] = (float)s;
    }
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  for (int mode = 0; mode < 2; ++mode) {
    CK(cudaMemset(dD, 0, D.size() * 4));
    k_check<<<1, 128>>>(dA, dB, dD, mode);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    int bad = 0;
    for (int i = 0; i < M * NN; ++i) {
      err = fmax(err, fabs(D[i] - ref[i]));
      bad += fabs(D[i] - ref[i]) > 1e-3;
    }
    printf("check mode %d (%s): max err %.3g, bad %d  D[0]=%g ref %g D[1][3]=%g ref %g\n", mode,
           mode ? "A in TMEM" : "A, B in smem", err, bad, D[0], ref[0], D[NN + 3], ref[NN + 3]);
  }
  float* sink;
  long long* cyc;
  CK(cudaMalloc(&sink, 148 * 512 * 4));
  CK(cudaMalloc(&cyc, 148 * 8));
  for (int store = 0; store < 2; ++store)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096;
      k_tput<<<148, 32 * warps>>>(iters, store, sink, cyc);
      CK(cudaDeviceSynchronize());
      long long c;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      const double bytes = (double)iters * warps * 32 * 16 * 4;
      printf("%s x16, %2d warps/SM: %.1f B/cycle/SM (%.0f cycles)\n", store ? "tcgen05.st" : "tcgen05.ld", warps,
             bytes / c, (double)c);
    }
  return 0;
}
