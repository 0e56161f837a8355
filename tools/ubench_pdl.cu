// Graph node overhead with and without programmatic dependent launch (PDL) on sm_100a:
// a chain of NK dependent small kernels (each 148 x 256 threads, a short dependent read-modify-
// write) captured into a CUDA graph and replayed.  Reports microseconds per kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pdl tools/ubench_pdl.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_step(float* x, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.999f + 1.f;
}

int main() {
  const int n = 148 * 256, NK = 200, REP = 20;
  float* x;
  cudaMalloc(&x, n * sizeof(float));
  cudaMemset(x, 0, n * sizeof(float));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < NK; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_step, x, n, pdl);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int r = 0; r < REP; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("pdl=%d: %.3f us per kernel node (%s)\n", pdl, ms * 1e3 / (REP * NK), cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
