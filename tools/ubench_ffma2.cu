// Throughput of packed FP32 (FFMA2 / FADD2 / FMUL2, PTX fma.rn.f32x2 on sm_100a) against scalar FFMA:
// every thread runs NC independent dependency chains; reports FP32 lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
template <int NC>
__global__ void k_scalar(float* out, int iters, float b, float c) {
  float x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fmaf(x[i], b, c);
  float s = 0; for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
template <int NC>
__global__ void k_pair(float* out, int iters, float b, float c) {
  u64 x[NC];
  u64 bb, cc;
  asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b), "f"(b));
  asm("mov.b64 %0, {%1,%2};" : "=l"(cc) : "f"(c), "f"(c));
#pragma unroll
  for (int i = 0; i < NC; ++i) { float v = threadIdx.x + i; asm("mov.b64 %0, {%1,%2};" : "=l"(x[i]) : "f"(v), "f"(v)); }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fma2(x[i], bb, cc);
  float s = 0;
  for (int i = 0; i < NC; ++i) { float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x[i])); s += p + q; }
  if (s == 1.2345f) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; cudaMalloc(&o, 4);
  const int iters = 1 << 14, threads = 1024, blocks = sms * 2;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) k_scalar<8><<<blocks, threads>>>(o, iters, 0.999f, 0.001f);
      else k_pair<8><<<blocks, threads>>>(o, iters, 0.999f, 0.001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double lane_fma = (double)blocks * threads * iters * 8 * (mode ? 2 : 1);
      const double per_clk_sm = lane_fma / (ms * 1e-3) / sms / (clk * 1e3);
      printf("%s: %.3f ms, %.1f lane-FMA/clk/SM (at %d MHz boost), %.2f TFLOP/s\n", mode ? "FFMA2" : "FFMA ",
             ms, per_clk_sm, clk / 1000, 2 * lane_fma / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
