// Generator kernels: z = f_theta(y0), its reverse mode, and Adam on theta.
//
//   h_0 = tanh(W_in y0 + b_in);  u_d = tanh(W1_d h_d + b1_d);  h_{d+1} = h_d + W2_d u_d + b2_d;
//   z = sigmoid(W_out h_D + b_out)            (Eq. 20)
//
// Batch size is one input vector per restart (y0 is fixed, Alg. 1), so every layer is a
// matrix-VECTOR product: the two Din x W affine maps are HBM/L2-bound streams (and their Adam
// updates, 24 B per parameter), the 2D hidden W x W layers are latency-bound.  Kernels:
//   k_net_in        W_in rows x 256-column chunks: partials of W_in y0 (forward), or the
//                   outer-product gradient dL/dW_in = ga0 y0^T fused with Adam AND the next
//                   forward's partials of the updated W_in (one pass over W_in, m, v)
//   k_net_mid_fwd   one 8-CTA cluster per restart: every CTA keeps its W/8 rows of all 2D hidden
//                   matrices in shared memory, computes its rows of each layer and pushes them into
//                   every CTA's shared memory over DSMEM; one cluster barrier per layer
//   k_net_out       W_out rows (warp per row): z = sigmoid(W_out h_D + b_out)
//   k_net_out_bwd   dL/do = dL/dz z (1-z); dL/dW_out = go h_D^T fused with Adam, and per-CTA
//                   partials of W_out^T go (old weights)
//   k_net_mid_bwd   the cluster again, layers in reverse: transposed products W^T g as per-CTA
//                   partials exchanged over DSMEM and summed in a fixed order; Adam on the CTA's rows
// Every reduction has a fixed order (no float atomics): results are deterministic.
#include <cooperative_groups.h>

#include "net.cuh"

namespace cg = cooperative_groups;

namespace sq {
namespace {

enum { NM_FWD = 0, NM_GRAD = 1, NM_ADAM = 2 };

struct NetArgs {
  int Din, W, D, n_in, n_out;
  size_t P, o_bin, o_blk, o_wout, o_bout;
  float* theta;
  const float* y0;
  float* z;
  const float* gz;
  float* gtheta;
  float *m, *v;
  float* tape;
  float* pin;
  float* pout;
  float* ga0;
  AdamP ap;
  const int* status;
};

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// One bias-corrected Adam update (the same arithmetic as k_adam, Q15).
struct AdamC {
  float lr, b1, b2, eps, c1, c2;
  __device__ __forceinline__ float upd(float x, float& m, float& v, float g) const {
    m = b1 * m + (1.f - b1) * g;
    v = b2 * v + (1.f - b2) * g * g;
    return x - lr * (m / c1) / (sqrtf(v / c2) + eps);
  }
};

__device__ __forceinline__ AdamC adam_c(const AdamP& ap) {
  AdamC a;
  a.lr = ap.lr; a.b1 = ap.b1; a.b2 = ap.b2; a.eps = ap.eps;
  ap.corr(a.c1, a.c2);
  return a;
}

// ----------------------------------------------------------------------------------- W_in
// grid (n_in, ceil(W/8), R), 256 threads: warp w owns row i = 8 blockIdx.y + w, lane owns 8 columns
// of the 256-column chunk (two float4 when Din % 4 == 0, else 8 strided scalars).
template <int MODE, bool VEC>
__global__ void __launch_bounds__(256) k_net_in(NetArgs a) {
  const int r = blockIdx.z, lane = threadIdx.x & 31;
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= a.W) return;
  const int j0 = blockIdx.x * NET_IN_COLS;
  const size_t base = (size_t)r * a.P + (size_t)i * a.Din;
  const float* y = a.y0 + (size_t)r * a.Din;
  float gi = 0.f;
  bool upd = true;
  AdamC ad{};
  if (MODE != NM_FWD) gi = a.ga0[(size_t)r * a.W + i];
  if (MODE == NM_ADAM) {
    upd = !(*a.status & ST_NONFINITE);  // keep the last finite iterate
    ad = adam_c(a.ap);
  }
  float p = 0.f;
  if (VEC) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + h * 128 + lane * 4;
      if (j >= a.Din) break;
      const float4 y4 = *reinterpret_cast<const float4*>(y + j);
      float4* wp = reinterpret_cast<float4*>(a.theta + base + j);
      float4 w4 = *wp;
      if (MODE == NM_GRAD) {
        *reinterpret_cast<float4*>(a.gtheta + base + j) = make_float4(gi * y4.x, gi * y4.y, gi * y4.z, gi * y4.w);
        continue;
      }
      if (MODE == NM_ADAM && upd) {
        float4* mp = reinterpret_cast<float4*>(a.m + base + j);
        float4* vp = reinterpret_cast<float4*>(a.v + base + j);
        float4 m4 = *mp, v4 = *vp;
        w4.x = ad.upd(w4.x, m4.x, v4.x, gi * y4.x);
        w4.y = ad.upd(w4.y, m4.y, v4.y, gi * y4.y);
        w4.z = ad.upd(w4.z, m4.z, v4.z, gi * y4.z);
        w4.w = ad.upd(w4.w, m4.w, v4.w, gi * y4.w);
        *wp = w4;
        *mp = m4;
        *vp = v4;
      }
      p = fmaf(w4.x, y4.x, p);
      p = fmaf(w4.y, y4.y, p);
      p = fmaf(w4.z, y4.z, p);
      p = fmaf(w4.w, y4.w, p);
    }
  } else {
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int j = j0 + h * 32 + lane;
      if (j >= a.Din) break;
      const float yj = y[j];
      float wj = a.theta[base + j];
      if (MODE == NM_GRAD) {
        a.gtheta[base + j] = gi * yj;
        continue;
      }
      if (MODE == NM_ADAM && upd) {
        float mj = a.m[base + j], vj = a.v[base + j];
        wj = ad.upd(wj, mj, vj, gi * yj);
        a.theta[base + j] = wj;
        a.m[base + j] = mj;
        a.v[base + j] = vj;
      }
      p = fmaf(wj, yj, p);
    }
  }
  if (MODE == NM_GRAD) return;
  p = warp_sum(p);
  if (lane == 0) a.pin[((size_t)r * a.n_in + blockIdx.x) * a.W + i] = p;
}

// ----------------------------------------------------------------------------------- W_out
// grid (n_out, R), 256 threads: warp w owns rows 8w..8w+7 of the CTA's 64; lanes < W/4 own 4 columns.
__global__ void __launch_bounds__(256) k_net_out(NetArgs a) {
  const int r = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W4 = a.W >> 2;
  const float* hD = a.tape + ((size_t)r * (2 * a.D + 1) + a.D) * a.W;
  const float4 h4 = lane < W4 ? reinterpret_cast<const float4*>(hD)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float* th = a.theta + (size_t)r * a.P;
  for (int k = 0; k < 8; ++k) {
    const int i = blockIdx.x * NET_OUT_ROWS + warp * 8 + k;
    if (i >= a.Din) break;
    float p = 0.f;
    if (lane < W4) {
      const float4 w4 = reinterpret_cast<const float4*>(th + a.o_wout + (size_t)i * a.W)[lane];
      p = w4.x * h4.x;
      p = fmaf(w4.y, h4.y, p);
      p = fmaf(w4.z, h4.z, p);
      p = fmaf(w4.w, h4.w, p);
    }
    p = warp_sum(p);
    if (lane == 0) a.z[(size_t)r * a.Din + i] = 1.f / (1.f + expf(-(p + th[a.o_bout + i])));
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_net_out_bwd(NetArgs a) {
  __shared__ float4 red[8][32];
  const int r = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W4 = a.W >> 2;
  const float* hD = a.tape + ((size_t)r * (2 * a.D + 1) + a.D) * a.W;
  const float4 h4 = lane < W4 ? reinterpret_cast<const float4*>(hD)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t tb = (size_t)r * a.P;
  bool upd = true;
  AdamC ad{};
  if (MODE == NM_ADAM) {
    upd = !(*a.status & ST_NONFINITE);
    ad = adam_c(a.ap);
  }
  if (MODE == NM_GRAD && blockIdx.x == 0 && threadIdx.x < a.P - (a.o_bout + a.Din))
    a.gtheta[tb + a.o_bout + a.Din + threadIdx.x] = 0.f;  // stride padding (< 4 floats)
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < 8; ++k) {
    const int i = blockIdx.x * NET_OUT_ROWS + warp * 8 + k;
    if (i >= a.Din) break;
    const float zi = a.z[(size_t)r * a.Din + i];
    const float go = a.gz[(size_t)r * a.Din + i] * zi * (1.f - zi);  // sigmoid'
    if (lane < W4) {
      const size_t o = tb + a.o_wout + (size_t)i * a.W + 4 * lane;
      float4* wp = reinterpret_cast<float4*>(a.theta + o);
      const float4 w4 = *wp;  // old weights for W_out^T go
      acc.x = fmaf(w4.x, go, acc.x);
      acc.y = fmaf(w4.y, go, acc.y);
      acc.z = fmaf(w4.z, go, acc.z);
      acc.w = fmaf(w4.w, go, acc.w);
      const float4 g4 = make_float4(go * h4.x, go * h4.y, go * h4.z, go * h4.w);
      if (MODE == NM_GRAD) {
        *reinterpret_cast<float4*>(a.gtheta + o) = g4;
      } else if (upd) {
        float4* mp = reinterpret_cast<float4*>(a.m + o);
        float4* vp = reinterpret_cast<float4*>(a.v + o);
        float4 m4 = *mp, v4 = *vp, n4;
        n4.x = ad.upd(w4.x, m4.x, v4.x, g4.x);
        n4.y = ad.upd(w4.y, m4.y, v4.y, g4.y);
        n4.z = ad.upd(w4.z, m4.z, v4.z, g4.z);
        n4.w = ad.upd(w4.w, m4.w, v4.w, g4.w);
        *wp = n4;
        *mp = m4;
        *vp = v4;
      }
    }
    if (lane == 0) {  // b_out
      const size_t o = tb + a.o_bout + i;
      if (MODE == NM_GRAD) {
        a.gtheta[o] = go;
      } else if (upd) {
        float mb = a.m[o], vb = a.v[o];
        a.theta[o] = ad.upd(a.theta[o], mb, vb, go);
        a.m[o] = mb;
        a.v[o] = vb;
      }
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && lane < W4) {  // fixed-order sum over the 8 warps
    float4 s = red[0][lane];
    for (int q = 1; q < 8; ++q) {
      const float4 t = red[q][lane];
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    reinterpret_cast<float4*>(a.pout + ((size_t)r * a.n_out + blockIdx.x) * a.W)[lane] = s;
  }
}

// ----------------------------------------------------------------------------------- hidden layers
// One cluster of NET_CL CTAs per restart (grid (NET_CL, R)), 128 threads.  CTA c owns rows
// [c RW, (c+1) RW) of every hidden matrix, RW = W / NET_CL; its rows of W1_d and W2_d are one
// contiguous block each in theta, staged in shared memory at entry.
__device__ __forceinline__ void load_slices(const NetArgs& a, const float* th, int c, int RW, float* wsl) {
  const int blk = RW * a.W;  // floats per matrix slice (multiple of 4)
  const size_t stride_d = 2 * (size_t)a.W * a.W + 2 * (size_t)a.W;
  for (int k = threadIdx.x; k < 2 * a.D * (blk >> 2); k += blockDim.x) {
    const int s = k / (blk >> 2), e = k - s * (blk >> 2);
    const int d = s >> 1, which = s & 1;  // 0: W1_d, 1: W2_d
    const size_t o = a.o_blk + d * stride_d + (which ? (size_t)a.W * a.W + a.W : 0) + (size_t)c * blk;
    reinterpret_cast<float4*>(wsl + (size_t)s * blk)[e] = reinterpret_cast<const float4*>(th + o)[e];
  }
}

// row il of the CTA's slice of matrix s, dotted with the shared vector x (length W); warp-wide
__device__ __forceinline__ float row_dot(const float* wsl, int s, int il, int RW, int W, const float* x, int lane) {
  const float4* w4 = reinterpret_cast<const float4*>(wsl + ((size_t)s * RW + il) * W);
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float p = 0.f;
  for (int k = lane; k < (W >> 2); k += 32) {
    const float4 w = w4[k], v = x4[k];
    p = fmaf(w.x, v.x, p);
    p = fmaf(w.y, v.y, p);
    p = fmaf(w.z, v.z, p);
    p = fmaf(w.w, v.w, p);
  }
  return warp_sum(p);
}

__global__ void __cluster_dims__(NET_CL, 1, 1) __launch_bounds__(128) k_net_mid_fwd(NetArgs a) {
  extern __shared__ __align__(16) float sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), r = blockIdx.y;
  const int W = a.W, RW = W / NET_CL, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wsl = sm;                              // [2D][RW][W]
  float* hb = wsl + (size_t)2 * a.D * RW * W;   // [2][W]
  float* ub = hb + 2 * W;                       // [W]
  const float* th = a.theta + (size_t)r * a.P;
  float* tape = a.tape + (size_t)r * (2 * a.D + 1) * W;
  load_slices(a, th, c, RW, wsl);
  for (int j = threadIdx.x; j < W; j += blockDim.x) {  // h_0, redundantly in every CTA (fixed order)
    float s = th[a.o_bin + j];
    const float* pp = a.pin + (size_t)r * a.n_in * W + j;
    for (int q = 0; q < a.n_in; ++q) s += pp[(size_t)q * W];
    const float h = tanhf(s);
    hb[j] = h;
    if (c == 0) tape[j] = h;
  }
  cl.sync();  // slices staged, h_0 ready, every CTA of the cluster running (DSMEM targets live)
  const size_t stride_d = 2 * (size_t)W * W + 2 * (size_t)W;
  int cur = 0;
  for (int d = 0; d < a.D; ++d) {
    const float* b1 = th + a.o_blk + d * stride_d + (size_t)W * W;
    const float* b2 = b1 + W + (size_t)W * W;
    for (int il = warp; il < RW; il += 4) {
      const int i = c * RW + il;
      const float u = tanhf(row_dot(wsl, 2 * d, il, RW, W, hb + cur * W, lane) + b1[i]);
      if (lane < NET_CL) *cl.map_shared_rank(ub + i, lane) = u;
      if (lane == 0) tape[(size_t)(a.D + 1 + d) * W + i] = u;
    }
    cl.sync();
    for (int il = warp; il < RW; il += 4) {
      const int i = c * RW + il;
      const float h = hb[cur * W + i] + row_dot(wsl, 2 * d + 1, il, RW, W, ub, lane) + b2[i];
      if (lane < NET_CL) *cl.map_shared_rank(hb + (cur ^ 1) * W + i, lane) = h;
      if (lane == 0) tape[(size_t)(d + 1) * W + i] = h;
    }
    cl.sync();
    cur ^= 1;
  }
}

template <int MODE>
__global__ void __cluster_dims__(NET_CL, 1, 1) __launch_bounds__(128) k_net_mid_bwd(NetArgs a) {
  extern __shared__ __align__(16) float sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), r = blockIdx.y;
  const int W = a.W, RW = W / NET_CL, D = a.D, t = threadIdx.x;
  float* wsl = sm;                                // [2D][RW][W] old weights
  float* tv = wsl + (size_t)2 * D * RW * W;       // [2D+1][W] tape: h_0..h_D, u_0..u_{D-1}
  float* gh = tv + (size_t)(2 * D + 1) * W;       // [W]
  float* ga = gh + W;                             // [W]
  float* xb = ga + W;                             // [2][NET_CL][W] transposed partials per source CTA
  float* sred = xb + 2 * NET_CL * W;              // [128] partial sums of the W_out^T go reduction
  float* th = a.theta + (size_t)r * a.P;
  const float* tape = a.tape + (size_t)r * (2 * D + 1) * W;
  load_slices(a, th, c, RW, wsl);
  for (int k = t; k < (2 * D + 1) * W; k += blockDim.x) tv[k] = tape[k];
  bool upd = true;
  AdamC ad{};
  if (MODE == NM_ADAM) {
    upd = !(*a.status & ST_NONFINITE);
    ad = adam_c(a.ap);
  }
  const size_t tb = (size_t)r * a.P;
  auto step = [&](size_t o, float g) {  // one parameter: gradient write or Adam
    if (MODE == NM_GRAD) {
      a.gtheta[tb + o] = g;
    } else if (upd) {
      float mm = a.m[tb + o], vv = a.v[tb + o];
      th[o] = ad.upd(th[o], mm, vv, g);
      a.m[tb + o] = mm;
      a.v[tb + o] = vv;
    }
  };
  {  // gh = W_out^T go: CTA c reduces its RW columns over the n_out partials, pushes them to all CTAs
    const int S = blockDim.x / RW, jl = t % RW, q0 = t / RW;
    float s = 0.f;
    const float* pp = a.pout + (size_t)r * a.n_out * W + c * RW + jl;
    for (int q = q0; q < a.n_out; q += S) s += pp[(size_t)q * W];
    sred[t] = s;
    cl.sync();  // also: every CTA of the cluster is running before the first DSMEM store
    if (t < RW) {
      float g = 0.f;
      for (int q = 0; q < S; ++q) g += sred[q * RW + t];
      for (int q = 0; q < NET_CL; ++q) *cl.map_shared_rank(gh + c * RW + t, q) = g;
    }
  }
  cl.sync();
  const size_t stride_d = 2 * (size_t)W * W + 2 * (size_t)W;
  for (int d = D - 1; d >= 0; --d) {
    const size_t oW1 = a.o_blk + d * stride_d, ob1 = oW1 + (size_t)W * W;
    const size_t oW2 = ob1 + W, ob2 = oW2 + (size_t)W * W;
    const float* u = tv + (size_t)(D + 1 + d) * W;
    const float* h = tv + (size_t)d * W;
    // W2_d: partial of W2^T gh over the CTA's rows (old weights), then the update of those rows
    for (int j = t; j < W; j += blockDim.x) {
      float p = 0.f;
      for (int il = 0; il < RW; ++il) p = fmaf(wsl[((size_t)(2 * d + 1) * RW + il) * W + j], gh[c * RW + il], p);
      for (int q = 0; q < NET_CL; ++q) *cl.map_shared_rank(xb + (size_t)c * W + j, q) = p;
      for (int il = 0; il < RW; ++il) step(oW2 + (size_t)(c * RW + il) * W + j, gh[c * RW + il] * u[j]);
    }
    if (t < RW) step(ob2 + c * RW + t, gh[c * RW + t]);
    cl.sync();
    for (int j = t; j < W; j += blockDim.x) {  // ga = (W2^T gh) tanh'(.)
      float s = 0.f;
      for (int q = 0; q < NET_CL; ++q) s += xb[(size_t)q * W + j];
      ga[j] = s * (1.f - u[j] * u[j]);
    }
    __syncthreads();
    float* xb1 = xb + (size_t)NET_CL * W;
    for (int j = t; j < W; j += blockDim.x) {  // W1_d
      float p = 0.f;
      for (int il = 0; il < RW; ++il) p = fmaf(wsl[((size_t)(2 * d) * RW + il) * W + j], ga[c * RW + il], p);
      for (int q = 0; q < NET_CL; ++q) *cl.map_shared_rank(xb1 + (size_t)c * W + j, q) = p;
      for (int il = 0; il < RW; ++il) step(oW1 + (size_t)(c * RW + il) * W + j, ga[c * RW + il] * h[j]);
    }
    if (t < RW) step(ob1 + c * RW + t, ga[c * RW + t]);
    cl.sync();
    for (int j = t; j < W; j += blockDim.x) {  // skip path + inner path
      float s = 0.f;
      for (int q = 0; q < NET_CL; ++q) s += xb1[(size_t)q * W + j];
      gh[j] += s;
    }
    __syncthreads();
  }
  // ga0 = gh tanh'(a_0); b_in (the CTA's rows); W_in is done by k_net_in
  for (int j = t; j < W; j += blockDim.x) {
    const float g0 = gh[j] * (1.f - tv[j] * tv[j]);
    if (c == 0) a.ga0[(size_t)r * W + j] = g0;
    if (j / RW == c) step(a.o_bin + j, g0);
  }
  // (the last DSMEM stores precede the last cl.sync(): no CTA can still write into this one)
}

NetArgs make_args(const NetDims& d, const NetWs& ws) {
  NetArgs a{};
  a.Din = d.Din; a.W = d.W; a.D = d.D; a.n_in = d.n_in; a.n_out = d.n_out;
  a.P = d.P; a.o_bin = d.o_bin; a.o_blk = d.o_blk; a.o_wout = d.o_wout; a.o_bout = d.o_bout;
  a.tape = ws.tape; a.pin = ws.pin; a.pout = ws.pout; a.ga0 = ws.ga0;
  return a;
}

template <int MODE>
void launch_in(const NetDims& d, const NetArgs& a, cudaStream_t st) {
  const dim3 g(d.n_in, (d.W + 7) / 8, d.R);
  if (d.Din % 4 == 0) k_net_in<MODE, true><<<g, 256, 0, st>>>(a);
  else k_net_in<MODE, false><<<g, 256, 0, st>>>(a);
}

}  // namespace

bool net_dims(int R, int Din, int W, int D, NetDims* out, const char** why) {
  NetDims d;
  if (R < 1 || Din < 1) { *why = "generator: R and M N must be positive"; return false; }
  if (W < 8 || W > 128 || W % 8) { *why = "generator: net_width must be a multiple of 8 in [8, 128]"; return false; }
  if (D < 0) { *why = "generator: net_depth must be >= 0"; return false; }
  d.R = R; d.Din = Din; d.W = W; d.D = D;
  const size_t w = W, din = Din;
  d.o_bin = w * din;
  d.o_blk = d.o_bin + w;
  d.o_wout = d.o_blk + (size_t)D * (2 * w * w + 2 * w);
  d.o_bout = d.o_wout + din * w;
  d.P = (d.o_bout + din + 3) & ~(size_t)3;  // per-restart stride: float4-aligned restarts
  d.n_in = (Din + NET_IN_COLS - 1) / NET_IN_COLS;
  d.n_out = (Din + NET_OUT_ROWS - 1) / NET_OUT_ROWS;
  const size_t RW = W / NET_CL;
  d.smem_fwd = (2 * (size_t)D * RW * w + 3 * w) * sizeof(float);
  d.smem_bwd = (2 * (size_t)D * RW * w + (2 * (size_t)D + 1) * w + 2 * w + 2 * NET_CL * w + 128) * sizeof(float);
  if (d.smem_bwd > 200 * 1024) { *why = "generator: hidden layers exceed the cluster's shared memory (depth too large)"; return false; }
  *out = d;
  return true;
}

size_t net_ws_floats(const NetDims& d) {
  const size_t w = d.W;
  return (size_t)d.R * ((2 * (size_t)d.D + 1) * w + (size_t)d.n_in * w + (size_t)d.n_out * w + w) + 16;
}

NetWs net_ws_carve(const NetDims& d, float* base) {
  NetWs ws;
  const size_t w = d.W;
  ws.tape = base;
  ws.pin = ws.tape + (size_t)d.R * (2 * d.D + 1) * w;
  ws.pout = ws.pin + (size_t)d.R * d.n_in * w;
  ws.ga0 = ws.pout + (size_t)d.R * d.n_out * w;
  return ws;
}

cudaError_t net_prepare(const NetDims& d) {
  cudaError_t e = cudaFuncSetAttribute(k_net_mid_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem_fwd);
  if (e) return e;
  e = cudaFuncSetAttribute(k_net_mid_bwd<NM_GRAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem_bwd);
  if (e) return e;
  return cudaFuncSetAttribute(k_net_mid_bwd<NM_ADAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem_bwd);
}

cudaError_t net_forward(const NetDims& d, const NetWs& ws, const float* theta, const float* y0, float* z,
                        bool fresh_in, cudaStream_t st, int64_t* launches) {
  NetArgs a = make_args(d, ws);
  a.theta = const_cast<float*>(theta);  // read-only in the forward kernels
  a.y0 = y0;
  a.z = z;
  if (fresh_in) {
    launch_in<NM_FWD>(d, a, st);
    *launches += 1;
  }
  k_net_mid_fwd<<<dim3(NET_CL, d.R), 128, d.smem_fwd, st>>>(a);
  k_net_out<<<dim3(d.n_out, d.R), 256, 0, st>>>(a);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t net_backward(const NetDims& d, const NetWs& ws, float* theta, const float* y0, const float* z,
                         const float* gz, float* gtheta, float* m, float* v, const AdamP& ap, const int* status,
                         cudaStream_t st, int64_t* launches) {
  NetArgs a = make_args(d, ws);
  a.theta = theta; a.y0 = y0; a.z = const_cast<float*>(z); a.gz = gz; a.gtheta = gtheta;
  a.m = m; a.v = v; a.ap = ap; a.status = status;
  const dim3 go(d.n_out, d.R), gm(NET_CL, d.R);
  if (gtheta) {
    k_net_out_bwd<NM_GRAD><<<go, 256, 0, st>>>(a);
    k_net_mid_bwd<NM_GRAD><<<gm, 128, d.smem_bwd, st>>>(a);
    launch_in<NM_GRAD>(d, a, st);
  } else {
    k_net_out_bwd<NM_ADAM><<<go, 256, 0, st>>>(a);
    k_net_mid_bwd<NM_ADAM><<<gm, 128, d.smem_bwd, st>>>(a);
    launch_in<NM_ADAM>(d, a, st);
  }
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace sq
