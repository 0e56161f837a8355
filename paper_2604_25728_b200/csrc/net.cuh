// Internal interface between the C-ABI host code (sqngd.cu) and the generator kernels (net.cu):
// the transmit-side ResNet z = f_theta(y0) of PAPER.md Eq. 20,
// SURVEY.md §8(f) NEXT-2.  Architecture and parameter layout: include/sqngd.h (sqngd_net_*),
// DESIGN.md §3 "Generator".
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "adam.cuh"

namespace sq {

constexpr int NET_CL = 8;        // CTAs per cluster of the layer-serial kernels (one cluster per restart)
constexpr int NET_IN_COLS = 256; // columns of W_in per k_net_in CTA (one row per warp)
constexpr int NET_FWD_ROWS = 64; // rows of W_out per k_net_out CTA (8 per warp)
constexpr int NET_OUT_ROWS = 16; // rows of W_out per k_net_out_bwd CTA (2 per warp, loads up front)

struct NetDims {
  int R = 0, Din = 0, W = 0, D = 0;
  size_t P = 0;                                   // parameters per restart
  size_t o_bin = 0, o_blk = 0, o_wout = 0, o_bout = 0;  // W_in at offset 0
  int n_in = 0;                                   // column chunks of W_in (partials of W_in y0)
  int n_out = 0;                                  // clusters of W_out row chunks (partials of W_out^T g)
  int n_hid = 0;                                  // k_net_hid CTAs per restart
  size_t smem_fwd = 0, smem_bwd = 0;              // dynamic shared memory of the cluster kernels
};

struct NetWs {
  float* tape = nullptr;  // [R][2D+1][W]: h_0..h_D, u_0..u_{D-1}
  float* pin = nullptr;   // [R][n_in][W]  partials of W_in y0
  float* pout = nullptr;  // [R][n_out][W] partials of W_out^T (dL/do)
  float* ga0 = nullptr;   // [R][W] dL/d(W_in y0 + b_in)
  float* gvec = nullptr;  // [R][D][2][W] hidden-gradient factors: dL/dh_{d+1}, dL/d(W1_d h_d + b1_d)
};

// Validates (W % 8 == 0, 8 <= W <= 128, D >= 0, shared memory of the cluster kernels <= 200 KB).
bool net_dims(int R, int Din, int W, int D, NetDims* out, const char** why);
size_t net_ws_floats(const NetDims& d);
NetWs net_ws_carve(const NetDims& d, float* base);
cudaError_t net_prepare(const NetDims& d);

// z = f_theta(y0) for all R restarts; writes the tape.  fresh_in: compute the W_in y0 partials
// first (else they were left by the previous net_backward in Adam mode).  launches += kernels.
cudaError_t net_forward(const NetDims& d, const NetWs& ws, const float* theta, const float* y0, float* z,
                        bool fresh_in, cudaStream_t st, int64_t* launches);

// Reverse mode from gz = dL/dz, z = the last forward's output (tape in ws).
// gtheta != nullptr: writes dL/dtheta (every entry once, layout of theta).
// gtheta == nullptr: Adam (m, v, ap; skipped when status has ST_NONFINITE) in place on theta, and
// the W_in y0 partials of the updated W_in for the next net_forward(fresh_in = false).
cudaError_t net_backward(const NetDims& d, const NetWs& ws, float* theta, const float* y0, const float* z,
                         const float* gz, float* gtheta, float* m, float* v, const AdamP& ap, const int* status,
                         cudaStream_t st, int64_t* launches);

}  // namespace sq
