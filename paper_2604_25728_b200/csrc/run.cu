// The Algorithm-1 driver (Alg. 1, stopping criterion
// P:L485 / P:L533): up to T outer iterations of sqngd_step(A+B), each followed by the hard-waveform
// WPSL; per restart the best (lowest hard WPSL) state is kept as the output snapshot (Alg. 1
// "Output: (X_hard, H)"), and training stops when no restart's hard WPSL has improved for
// `patience` consecutive outer iterations (DESIGN.md §3 "Stopping rule").  The bookkeeping runs on
// the device (k_run_track / k_run_done) so the loop needs no per-iteration host round trip; the host
// polls the stop flag every `check_every` iterations.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "run.cuh"

namespace {

struct RunPtrs {
  const float* z; const float* rho; const float* w; const float* theta;  // current state
  float* bz; float* brho; float* bw; float* btheta;                     // best snapshot
  size_t nz, nrho, nw, ntheta;                                           // floats per restart
};

struct RunDev {  // device-side bookkeeping (one allocation)
  int done;                 // the rule fired (frozen afterwards)
  int stop_iter;            // outer iterations run when it fired
};

// One block per restart: compare the hard WPSL of outer iteration t (1-based) with the best so far.
// An improvement is a decrease by more than `tol` ("by >= 1e-6, linear, N-normalized";
// fp32 noise would otherwise keep resetting the stall counter); the hard loss L at the last
// improvement is kept so the stop test can require that L kept decreasing over the window.
__global__ void k_run_track(int t, const sqngd_metrics* hard, double tol, double* best_wpsl, int32_t* best_iter,
                            int* stall, double* loss_ref, double* loss_cur, double* hist, double* lhist, int R,
                            RunDev* rd, RunPtrs p) {
  const int r = blockIdx.x;
  __shared__ int improve;
  if (rd->done) return;  // uniform: the rule already fired, the snapshot is final
  if (threadIdx.x == 0) {
    const double v = hard[r].wpsl, L = hard[r].loss;
    if (hist) hist[(size_t)(t - 1) * R + r] = v;
    if (lhist) lhist[(size_t)(t - 1) * R + r] = L;
    loss_cur[r] = L;
    improve = v < best_wpsl[r] - tol || (t == 1 && v == v);  // (a NaN never improves)
    if (improve) {
      best_wpsl[r] = v;
      best_iter[r] = t;
      stall[r] = 0;
      loss_ref[r] = L;
    } else {
      stall[r] += 1;
    }
  }
  __syncthreads();
  if (!improve) return;
  auto copy = [&](const float* src, float* dst, size_t n) {
    if (!src || !dst) return;
    for (size_t k = threadIdx.x; k < n; k += blockDim.x) dst[(size_t)r * n + k] = src[(size_t)r * n + k];
  };
  copy(p.z, p.bz, p.nz);
  copy(p.rho, p.brho, p.nrho);
  copy(p.w, p.bw, p.nw);
  copy(p.theta, p.btheta, p.ntheta);
}

// The rule fires when every restart has gone `patience` iterations without an improvement and (if
// required) its hard loss L is below the value it had at the last improvement: "further reduction of
// L does not lead to improvement in the WPSL".
__global__ void k_run_done(int t, const int* stall, const double* loss_ref, const double* loss_cur, int R,
                           int patience, int need_dec, RunDev* rd) {
  if (rd->done || patience <= 0) return;
  int all = 1;
  for (int r = 0; r < R; ++r) all &= stall[r] >= patience && (!need_dec || loss_cur[r] < loss_ref[r]);
  if (all) {
    rd->done = 1;
    rd->stop_iter = t;
  }
}

}  // namespace

#define RK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      cleanup();                                                                         \
      return sq_ctx_fail(ctx, SQNGD_E_CUDA, #x, cudaGetErrorString(e_));                 \
    }                                                                                    \
  } while (0)

extern "C" sqngd_status sqngd_run(sqngd_ctx ctx, sqngd_state* state, const sqngd_run_opts* opts, sqngd_state* best,
                                  double* best_wpsl, int32_t* best_iter, double* wpsl_hist, double* loss_hist,
                                  sqngd_run_result* result, sqngd_stream stream) {
  auto cleanup = []() {};
  if (!ctx || !state || !opts || !best || !best_wpsl || !best_iter || !result || opts->T < 1 ||
      opts->check_every < 1 || !best->z || !best->rho || !best->w || !(opts->tol >= 0.0))
    return sq_ctx_fail(ctx, SQNGD_E_INVALID, "sqngd_run: bad argument", "");
  const sqngd_config& c = *sq_ctx_config(ctx);
  const bool net = c.net_width > 0;
  if (net && !best->theta) return sq_ctx_fail(ctx, SQNGD_E_INVALID, "sqngd_run: generator mode needs best->theta", "");
  RK(cudaSetDevice(sq_ctx_device(ctx)));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // bookkeeping buffers live in the context (one allocation, reused by every call): the hard-metrics
  // pointer handed to sqngd_step stays the same, so its step graph is captured once
  const size_t R = (size_t)c.R;
  const size_t nz = (size_t)c.M * c.N, nrho = (size_t)c.B * c.r_n, nw = 2 * (size_t)c.M * c.N;
  const size_t nth = net ? (size_t)sqngd_net_num_params(&c) : 0;
  const size_t off_stall = R * sizeof(sqngd_metrics), off_lref = off_stall + ((R * sizeof(int) + 7) & ~(size_t)7);
  const size_t off_lcur = off_lref + R * sizeof(double), off_rd = off_lcur + R * sizeof(double);
  const size_t off_cand = (off_rd + sizeof(RunDev) + 255) & ~(size_t)255;  // the iterate a step starts from
  const size_t cand_floats = R * (nz + nrho + nw + nth);
  void* host = nullptr;
  char* ws = static_cast<char*>(sq_ctx_run_ws(ctx, off_cand + cand_floats * sizeof(float), &host, sizeof(RunDev)));
  if (!ws || !host) return sq_ctx_fail(ctx, SQNGD_E_NOMEM, "sqngd_run: workspace", "");
  sqngd_metrics* hard = reinterpret_cast<sqngd_metrics*>(ws);
  int* stall = reinterpret_cast<int*>(ws + off_stall);
  double* loss_ref = reinterpret_cast<double*>(ws + off_lref);
  double* loss_cur = reinterpret_cast<double*>(ws + off_lcur);
  RunDev* rd = reinterpret_cast<RunDev*>(ws + off_rd);
  RunDev* rd_host = static_cast<RunDev*>(host);
  float* cz = reinterpret_cast<float*>(ws + off_cand);
  float* crho = cz + R * nz;
  float* cw = crho + R * nrho;
  float* cth = cw + R * nw;
  RK(cudaMemsetAsync(stall, 0, sizeof(int) * c.R, st));
  RK(cudaMemsetAsync(rd, 0, sizeof(RunDev), st));
  {  // best_wpsl = +inf, best_iter = 0
    static_assert(sizeof(double) == 8, "");
    const double inf = INFINITY;
    for (int r = 0; r < c.R; ++r) RK(cudaMemcpyAsync(best_wpsl + r, &inf, sizeof(double), cudaMemcpyHostToDevice, st));
    RK(cudaMemsetAsync(best_iter, 0, sizeof(int32_t) * c.R, st));
    RK(cudaStreamSynchronize(st));  // (the host `inf` is a stack value)
  }
  // Iterate t (the state after t outer iterations) is scored by the hard metrics of step t + 1, which
  // evaluates it in its first Step-A evaluation (sqngd_step hard_out); its snapshot source is the copy
  // taken before that step.  The last iterate is scored by one explicit forward after the loop.
  RunPtrs pc{};  // snapshot source: the candidate copy
  pc.z = cz; pc.rho = crho; pc.w = cw; pc.theta = net ? cth : nullptr;
  pc.bz = best->z; pc.brho = best->rho; pc.bw = best->w; pc.btheta = net ? best->theta : nullptr;
  pc.nz = nz; pc.nrho = nrho; pc.nw = nw; pc.ntheta = nth;
  RunPtrs ps = pc;  // snapshot source: the live state (last iterate)
  ps.z = state->z; ps.rho = state->rho; ps.w = state->w; ps.theta = net ? state->theta : nullptr;
  auto track = [&](int it, const RunPtrs& p) -> cudaError_t {
    k_run_track<<<c.R, 256, 0, st>>>(it, hard, opts->tol, best_wpsl, best_iter, stall, loss_ref, loss_cur, wpsl_hist,
                                     loss_hist, c.R, rd, p);
    k_run_done<<<1, 1, 0, st>>>(it, stall, loss_ref, loss_cur, c.R, opts->patience, opts->require_loss_decrease, rd);
    return cudaGetLastError();
  };
  int64_t t = 0;
  bool stopped = false;
  for (t = 1; t <= opts->T; ++t) {
    if (t >= 2) {
      RK(cudaMemcpyAsync(cz, state->z, sizeof(float) * R * nz, cudaMemcpyDeviceToDevice, st));
      RK(cudaMemcpyAsync(crho, state->rho, sizeof(float) * R * nrho, cudaMemcpyDeviceToDevice, st));
      RK(cudaMemcpyAsync(cw, state->w, sizeof(float) * R * nw, cudaMemcpyDeviceToDevice, st));
      if (net) RK(cudaMemcpyAsync(cth, state->theta, sizeof(float) * R * nth, cudaMemcpyDeviceToDevice, st));
    }
    sqngd_status s = sqngd_step(ctx, state, SQNGD_BLOCK_AB, nullptr, hard, stream);
    if (s != SQNGD_OK) return s;
    if (t >= 2) RK(track((int)t - 1, pc));
    if (t % opts->check_every == 0) {
      RK(cudaMemcpyAsync(rd_host, rd, sizeof(RunDev), cudaMemcpyDeviceToHost, st));
      RK(cudaStreamSynchronize(st));
      if (rd_host->done) {
        stopped = true;
        break;
      }
    }
  }
  if (!stopped) {  // the last iterate T
    t = opts->T;
    sqngd_status s = sq_ctx_hard_metrics(ctx, state, hard, stream);
    if (s != SQNGD_OK) return s;
    RK(track((int)opts->T, ps));
    RK(cudaMemcpyAsync(rd_host, rd, sizeof(RunDev), cudaMemcpyDeviceToHost, st));
    RK(cudaStreamSynchronize(st));
    stopped = rd_host->done != 0;
  }
  result->iterations = stopped ? rd_host->stop_iter : opts->T;
  result->steps_run = stopped ? t : opts->T;
  result->stopped = stopped ? 1 : 0;
  return sqngd_sync(ctx, stream);
}
