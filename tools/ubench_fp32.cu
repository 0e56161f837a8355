// Microbenchmark: FP32 issue rates of FADD / FMUL / FFMA (3-reg, imm) on one SM pipe set.
// Each thread runs 8 independent dependency chains, unrolled; 32 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 4096
template <int KIND>
__global__ void kern(float* out, const float* in, int n) {
  float a[8], b = in[threadIdx.x & 7] , c = in[(threadIdx.x + 3) & 7];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[i] + threadIdx.x;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 0) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
        if (KIND == 1) asm volatile("mul.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
        if (KIND == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
        if (KIND == 3) asm volatile("fma.rn.f32 %0, %0, %1, 0f3F800001;" : "+f"(a[i]) : "f"(b));
        if (KIND == 4) { // alternate add / 3-reg fma
          if (i & 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
          else asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
        }
        if (KIND == 5) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[i]) : "f"(a[(i+1)&7]), "f"(c));
        if (KIND == 6) asm volatile("add.f32 %0, %1, %0;" : "+f"(a[i]) : "f"(a[(i+3)&7]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND>
void run(const char* name, float* out, float* in, int sms, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<KIND><<<sms, threads>>>(out, in, 16);
  cudaEventRecord(e0);
  kern<KIND><<<sms, threads>>>(out, in, ITER);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double instr = (double)sms * (threads / 32) * ITER * 16 * 8;  // warp-instructions
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * 1965e6;
  printf("%-22s threads/SM=%4d  warp-instr per SMSP-cycle (at 1965 MHz) = %.3f  (%.3f ms)\n", name, threads,
         instr / (sms * 4.0) / cyc, ms);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out, *in; cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&in, 64 * 4);
  float h[16]; for (int i = 0; i < 16; ++i) h[i] = 1.0f + i * 1e-7f; cudaMemcpy(in, h, 64, cudaMemcpyHostToDevice);
  for (int th : {256, 512, 1024}) {
    run<0>("FADD", out, in, sms, th);
    run<1>("FMUL", out, in, sms, th);
    run<2>("FFMA 3reg", out, in, sms, th);
    run<3>("FFMA imm", out, in, sms, th);
    run<4>("FADD/FFMA alt", out, in, sms, th);
    run<5>("FFMA 3reg distinct", out, in, sms, th);
    run<6>("FADD 2 distinct", out, in, sms, th);
  }
  return 0;
}
