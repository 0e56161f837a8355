// Microbenchmark: legacy warp-level mma.sync throughput on sm_100a (TF32 m16n8k8, F16 m16n8k16).
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 2048
template <int KIND>
__global__ void kern(float* out, int n) {
  float d[8][4];
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  b[0] = a[1]; b[1] = a[2];
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[t][i] = 0.f;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[t][0]), "+f"(d[t][1]), "+f"(d[t][2]), "+f"(d[t][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[t][0]), "+f"(d[t][1]), "+f"(d[t][2]), "+f"(d[t][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[t][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND>
void run(const char* name, float* out, int sms, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<KIND><<<sms, threads>>>(out, 16);
  cudaEventRecord(e0);
  kern<KIND><<<sms, threads>>>(out, ITER);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops_per = KIND == 0 ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16;
  double mmas = (double)sms * (threads / 32) * ITER * 8;
  printf("%-14s threads/SM=%4d  %.1f TFLOP/s  %.3f mma/clk/SM (1965 MHz)\n", name, threads, mmas * flops_per / ms / 1e9,
         mmas / sms / (ms * 1e-3 * 1965e6));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 1024 * 4);
  for (int th : {128, 256, 512, 1024}) {
    run<0>("tf32 m16n8k8", out, sms, th);
    run<1>("f16 m16n8k16", out, sms, th);
  }
  return 0;
}
