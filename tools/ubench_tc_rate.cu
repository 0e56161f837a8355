// tcgen05.mma issue-rate microbenchmark (sm_100a): cycles per MMA for the shapes k_lrt5 uses.
//   SS : A, B in shared memory (K-major, no swizzle), kind::tf32, M = 128, N in {16, 32, 64, 128}
//   TS : A in TMEM, B in shared memory
// One CTA per SM, one thread issues `iters` MMAs into one (or two alternating) accumulators, then
// commits and waits.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tc_rate tools/ubench_tc_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__global__ void k(int mode, int N, int iters, int chains, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  float* A = reinterpret_cast<float*>(sm);          // 128 x 32 K-major image (16 KB)
  float* B = reinterpret_cast<float*>(sm + 16384);  // 256 x 32 image (32 KB)
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 7);
  (void)A;
  (void)B;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tb;
  if (mode >= 2 && threadIdx.x < 32) {  // converged warp, elect inside the asm, unrolled x4
    const uint64_t da = desc_k(smem_u32(sm), 128, 1024), db = desc_k(smem_u32(sm + 16384), 128, 1024);
    const uint32_t id = idesc_tf32(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t acc = (i + j) >= 1;
        if (mode == 4)
          asm volatile(
              "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
              "l"(da), "l"(db), "r"(id), "r"(acc));
        else if (mode == 5)
          asm volatile(
              "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
              "l"(da), "l"(db), "r"(id & ~(0x3Fu << 7)), "r"(acc));
        else if (mode == 2)
          asm volatile(
              "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
              "l"(da + 16 * j), "l"(db + 16 * j), "r"(id), "r"(acc));
        else
          asm volatile(
              "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
              "r"(t + 384 + 8 * j), "l"(db + 16 * j), "r"(id), "r"(acc));
      }
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(
          smem_u32(&bar)));
      long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  }
  if (mode < 2 && threadIdx.x == 0) {
    const uint64_t da = desc_k(smem_u32(sm), 128, 1024), db = desc_k(smem_u32(sm + 16384), 128, 1024);
    const uint32_t id = idesc_tf32(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = t + 128 * (i % chains);
      const uint32_t acc = i >= chains;
      if (mode == 0)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                d),
            "l"(da + 16 * (i & 3)), "l"(db + 16 * (i & 3)), "r"(id), "r"(acc));
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(
                d),
            "r"(t + 384 + 8 * (i & 3)), "l"(db + 16 * (i & 3)), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
        smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}
int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int mode = 2; mode < 6; ++mode)
    for (int N : {16, 64, 256})
      for (int chains : {1}) {
        const int iters = 4096;
        k<<<148, 128, 65536>>>(mode, N, iters, chains, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%s N=%3d chains=%d: %.1f cycles/MMA (floor N/2 = %d) %s\n", mode == 5 ? "SS-f16-const" : mode == 4 ? "SS-tf32-const" : (mode & 1) ? (mode >= 2 ? "TS-warp" : "TS") : (mode >= 2 ? "SS-warp" : "SS"), N, chains,
               (double)c / iters, N / 2, e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
