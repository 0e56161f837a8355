// Generator kernels: z = f_theta(y0), its reverse mode, and Adam on theta.
//
//   h_0 = tanh(W_in y0 + b_in);  u_d = tanh(W1_d h_d + b1_d);  h_{d+1} = h_d + W2_d u_d + b2_d;
//   z = sigmoid(W_out h_D + b_out)            (Eq. 20)
//
// Batch size is one input vector per restart (y0 is fixed, Alg. 1), so every layer is a
// matrix-VECTOR product: the two Din x W affine maps are HBM/L2-bound streams (and their Adam
// updates, 24 B per parameter), the 2D hidden W x W layers are latency-bound.  Kernels:
//   k_net_upd       W_in rows x 256-column chunks: partials of W_in y0 (forward), or the
//                   outer-product gradient dL/dW_in = ga0 y0^T fused with Adam AND the next
//                   forward's partials of the updated W_in (one pass over W_in, m, v)
//   k_net_mid_fwd   one 8-CTA cluster per restart: every CTA keeps its W/8 rows of all 2D hidden
//                   matrices in shared memory, computes its rows of each layer and pushes them into
//                   every CTA's shared memory over DSMEM; one cluster barrier per layer
//   k_net_out       W_out rows (warp per row): z = sigmoid(W_out h_D + b_out)
//   k_net_out_bwd   dL/do = dL/dz z (1-z); dL/dW_out = go h_D^T fused with Adam, and per-CTA
//                   partials of W_out^T go (old weights)
//   k_net_mid_bwd   the cluster again, layers in reverse: transposed products W^T g as per-CTA
//                   partials exchanged over DSMEM and summed in a fixed order; stores the factor
//                   vectors of the hidden parameters' outer-product gradients
//                   + (same launch) all hidden parameters: gradient = outer product, fused Adam
// Every reduction has a fixed order (no float atomics): results are deterministic.
#include <cooperative_groups.h>

#include <cstdlib>

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
  float* gvec;
  AdamP ap;
  const int* status;
};

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ---- bulk async copies (TMA engine, non-tensor) completing on a CTA mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: multiple of 16; src, dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- DSMEM all-gathers without cluster barriers: each value is pushed with st.async into the peer's
// shared memory and completes bytes on the PEER's mbarrier; a receiver waits on its own barrier for
// the phase's expected bytes (one barrier per exchange phase, each used once per launch).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_async(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
// push v to address `dst` (a local shared pointer) in every CTA of the cluster, phase barrier `bar`
__device__ __forceinline__ void push_all(const float* dst, float v, uint64_t* bar) {
  const uint32_t a = smem_u32(dst), b = smem_u32(bar);
#pragma unroll
  for (int q = 0; q < NET_CL; ++q) st_async(mapa_u32(a, q), v, mapa_u32(b, q));
}
constexpr int NET_MAXD = 15;  // exchange barriers per launch: 2 D + 1 <= 31

// One bias-corrected Adam update (Q15): x - lr m^ / (sqrt(v^) + eps), m^ = m / c1, v^ = v / c2, with the
// step constants lr / c1 and 1 / c2 folded once and a fast divide (relative error ~1e-7 of the step).
struct AdamC {
  float b1, b2, eps, lr_c1, inv_c2;
  __device__ __forceinline__ float upd(float x, float& m, float& v, float g) const {
    m = b1 * m + (1.f - b1) * g;
    v = b2 * v + (1.f - b2) * g * g;
    return x - __fdividef(lr_c1 * m, sqrtf(v * inv_c2) + eps);
  }
};

// The bias corrections need the device-side step count (fp64 pow): one thread per CTA computes
// them and shares them through shared memory (call from every thread, CTA-uniform control flow).
__device__ __forceinline__ AdamC adam_c(const AdamP& ap) {
  __shared__ float cc[2];
  if (threadIdx.x == 0) {
    float c1, c2;
    ap.corr(c1, c2);
    cc[0] = ap.lr / c1;
    cc[1] = 1.f / c2;
  }
  __syncthreads();
  AdamC a;
  a.b1 = ap.b1; a.b2 = ap.b2; a.eps = ap.eps; a.lr_c1 = cc[0]; a.inv_c2 = cc[1];
  return a;
}

// ----------------------------------------------------------------------------------- W_in
// One k_net_upd block (bx, by): warp w owns row i = 8 by + w, lane owns 8 columns
// of the 256-column chunk (two float4 when Din % 4 == 0, else 8 strided scalars).
template <int MODE, bool VEC>
__device__ __forceinline__ void net_in_block(const NetArgs& a, int bx, int by, int r, const AdamC& ad, bool upd) {
  const int lane = threadIdx.x & 31;
  const int i = by * 8 + (threadIdx.x >> 5);
  if (i >= a.W) return;
  const int j0 = bx * NET_IN_COLS;
  const size_t base = (size_t)r * a.P + (size_t)i * a.Din;
  const float* y = a.y0 + (size_t)r * a.Din;
  float gi = 0.f;
  if (MODE != NM_FWD) gi = a.ga0[(size_t)r * a.W + i];
  float p = 0.f;
  if (VEC) {
    // both float4 column groups' operands are loaded before any store (a store between them would
    // serialize a second memory round trip)
    float4 y4[2], w4[2], m4[2], v4[2];
    bool in[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + h * 128 + lane * 4;
      in[h] = j < a.Din;
      const int jj = in[h] ? j : 0;
      y4[h] = *reinterpret_cast<const float4*>(y + jj);
      if (MODE != NM_GRAD) w4[h] = *reinterpret_cast<const float4*>(a.theta + base + jj);
      if (MODE == NM_ADAM) {
        m4[h] = *reinterpret_cast<const float4*>(a.m + base + jj);
        v4[h] = *reinterpret_cast<const float4*>(a.v + base + jj);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!in[h]) break;
      const int j = j0 + h * 128 + lane * 4;
      const float4 yv = y4[h];
      if (MODE == NM_GRAD) {
        *reinterpret_cast<float4*>(a.gtheta + base + j) = make_float4(gi * yv.x, gi * yv.y, gi * yv.z, gi * yv.w);
        continue;
      }
      float4 wv = w4[h];
      if (MODE == NM_ADAM && upd) {
        float4 mv = m4[h], vv = v4[h];
        wv.x = ad.upd(wv.x, mv.x, vv.x, gi * yv.x);
        wv.y = ad.upd(wv.y, mv.y, vv.y, gi * yv.y);
        wv.z = ad.upd(wv.z, mv.z, vv.z, gi * yv.z);
        wv.w = ad.upd(wv.w, mv.w, vv.w, gi * yv.w);
        *reinterpret_cast<float4*>(a.theta + base + j) = wv;
        *reinterpret_cast<float4*>(a.m + base + j) = mv;
        *reinterpret_cast<float4*>(a.v + base + j) = vv;
      }
      p = fmaf(wv.x, yv.x, p);
      p = fmaf(wv.y, yv.y, p);
      p = fmaf(wv.z, yv.z, p);
      p = fmaf(wv.w, yv.w, p);
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
  if (bx == 0 && lane == 31) {  // b_in[i]: dL/db_in = ga0
    const size_t ob = (size_t)r * a.P + a.o_bin + i;
    if (MODE == NM_GRAD) {
      a.gtheta[ob] = gi;
    } else if (MODE == NM_ADAM && upd) {
      float mb = a.m[ob], vb = a.v[ob];
      a.theta[ob] = ad.upd(a.theta[ob], mb, vb, gi);
      a.m[ob] = mb;
      a.v[ob] = vb;
    }
  }
  if (MODE == NM_GRAD) return;
  p = warp_sum(p);
  if (lane == 0) a.pin[((size_t)r * a.n_in + bx) * a.W + i] = p;
}

// ----------------------------------------------------------------------------------- W_out
// Forward: grid (ceil(Din / 64), R), 256 threads; warp w owns rows 8w..8w+7 of the CTA's 64 (all eight
// rows' loads issued before the reductions); lanes < W/4 own 4 columns.
__global__ void __launch_bounds__(256) k_net_out(NetArgs a) {
  SQ_PDL_WAIT();
  const int r = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W4 = a.W >> 2;
  const float* __restrict__ hD = a.tape + ((size_t)r * (2 * a.D + 1) + a.D) * a.W;
  const float4 h4 = lane < W4 ? reinterpret_cast<const float4*>(hD)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float* __restrict__ th = a.theta + (size_t)r * a.P;
  const int i0 = blockIdx.x * NET_FWD_ROWS + warp * 8;
  float4 w4[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = min(i0 + k, a.Din - 1);
    w4[k] = lane < W4 ? __ldg(reinterpret_cast<const float4*>(th + a.o_wout + (size_t)i * a.W) + lane)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float bo = lane < 8 ? __ldg(th + a.o_bout + min(i0 + lane, a.Din - 1)) : 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float p = w4[k].x * h4.x;
    p = fmaf(w4[k].y, h4.y, p);
    p = fmaf(w4[k].z, h4.z, p);
    p = fmaf(w4[k].w, h4.w, p);
    p = warp_sum(p) + __shfl_sync(0xffffffffu, bo, k);
    if (lane == k && i0 + k < a.Din) a.z[(size_t)r * a.Din + i0 + k] = 1.f / (1.f + expf(-p));
  }
}

// Backward: grid (8 n_out, R) in clusters of NET_CL along x, 256 threads; warp w owns rows 2w, 2w+1 of
// the CTA's 16 (loads first).  The CTA partials of W_out^T go are summed across the cluster over DSMEM
// (fixed order), one partial per cluster.
template <int MODE>
__global__ void __cluster_dims__(NET_CL, 1, 1) __launch_bounds__(256) k_net_out_bwd(NetArgs a) {
  SQ_PDL_WAIT();
  __shared__ float4 red[8][32];
  __shared__ float4 cpart[32];
  const int r = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W4 = a.W >> 2;
  const float* __restrict__ hD = a.tape + ((size_t)r * (2 * a.D + 1) + a.D) * a.W;
  const float4 h4 = lane < W4 ? reinterpret_cast<const float4*>(hD)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t tb = (size_t)r * a.P;
  float* __restrict__ th = a.theta;
  float* __restrict__ mm = a.m;
  float* __restrict__ vv = a.v;
  bool upd = true;
  AdamC ad{};
  if (MODE == NM_ADAM) {
    upd = !(*a.status & ST_NONFINITE);
    ad = adam_c(a.ap);
  }
  if (MODE == NM_GRAD && blockIdx.x == 0 && threadIdx.x < a.P - (a.o_bout + a.Din))
    a.gtheta[tb + a.o_bout + a.Din + threadIdx.x] = 0.f;  // stride padding (< 4 floats)
  const int i0 = blockIdx.x * NET_OUT_ROWS + warp * 2;
  float go[2];
  float4 w4[2], m4[2], v4[2];
  bool ok[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    ok[k] = i0 + k < a.Din;
    const int i = min(i0 + k, a.Din - 1);
    const float zi = a.z[(size_t)r * a.Din + i];
    go[k] = ok[k] ? a.gz[(size_t)r * a.Din + i] * zi * (1.f - zi) : 0.f;  // sigmoid'
    const size_t o = tb + a.o_wout + (size_t)i * a.W + 4 * lane;
    if (lane < W4) {
      w4[k] = *reinterpret_cast<const float4*>(th + o);
      if (MODE == NM_ADAM) {
        m4[k] = *reinterpret_cast<const float4*>(mm + o);
        v4[k] = *reinterpret_cast<const float4*>(vv + o);
      }
    } else {
      w4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);  // W_out^T go over the warp's rows (old weights)
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    acc.x = fmaf(w4[k].x, go[k], acc.x);
    acc.y = fmaf(w4[k].y, go[k], acc.y);
    acc.z = fmaf(w4[k].z, go[k], acc.z);
    acc.w = fmaf(w4[k].w, go[k], acc.w);
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && lane < W4) {  // fixed-order sum over the 8 warps
    float4 s = red[0][lane];
    for (int q = 1; q < 8; ++q) {
      const float4 t = red[q][lane];
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    cpart[lane] = s;
  }
  // Cluster exchange first, while no global store is outstanding (a release barrier would wait for
  // them); the CTA's parameter stores follow and overlap the other CTAs' DSMEM reads.
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const int c = (int)cl.block_rank(), RW = a.W / NET_CL;
  if ((int)threadIdx.x < RW) {  // CTA c sums its column slice over the cluster's CTAs
    const int j = c * RW + threadIdx.x;
    float* cp = reinterpret_cast<float*>(cpart);
    float g = 0.f;
    for (int q = 0; q < NET_CL; ++q) g += *cl.map_shared_rank(cp + j, q);
    a.pout[((size_t)r * a.n_out + blockIdx.x / NET_CL) * a.W + j] = g;
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // done reading remote cpart
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (!ok[k]) continue;
    const size_t o = tb + a.o_wout + (size_t)(i0 + k) * a.W + 4 * lane;
    if (lane < W4) {
      const float4 w = w4[k];
      const float4 g4 = make_float4(go[k] * h4.x, go[k] * h4.y, go[k] * h4.z, go[k] * h4.w);
      if (MODE == NM_GRAD) {
        *reinterpret_cast<float4*>(a.gtheta + o) = g4;
      } else if (upd) {
        float4 n4, mk = m4[k], vk = v4[k];
        n4.x = ad.upd(w.x, mk.x, vk.x, g4.x);
        n4.y = ad.upd(w.y, mk.y, vk.y, g4.y);
        n4.z = ad.upd(w.z, mk.z, vk.z, g4.z);
        n4.w = ad.upd(w.w, mk.w, vk.w, g4.w);
        *reinterpret_cast<float4*>(th + o) = n4;
        *reinterpret_cast<float4*>(mm + o) = mk;
        *reinterpret_cast<float4*>(vv + o) = vk;
      }
    }
    if (lane == 31) {  // b_out
      const size_t ob = tb + a.o_bout + i0 + k;
      if (MODE == NM_GRAD) {
        a.gtheta[ob] = go[k];
      } else if (upd) {
        float mb = mm[ob], vb = vv[ob];
        th[ob] = ad.upd(th[ob], mb, vb, go[k]);
        mm[ob] = mb;
        vv[ob] = vb;
      }
    }
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // keep cpart alive for the others
}

// Hidden-layer parameters (gradients are outer products of the factor vectors k_net_mid_bwd stored):
// W1_d: ga_d h_d^T, b1_d: ga_d, W2_d: gh_{d+1} u_d^T, b2_d: gh_{d+1}.  grid (ceil(D (2W^2+2W) / 1024), R),
// 256 threads, one float4 per thread (segment lengths are multiples of 4).
template <int MODE>
__device__ __forceinline__ void net_hid_block(const NetArgs& a, int bx, int r, const AdamC& ad, bool upd) {
  const int W = a.W;
  const size_t stride_d = 2 * (size_t)W * W + 2 * (size_t)W;
  const size_t e = 4 * ((size_t)bx * blockDim.x + threadIdx.x);
  if (e >= (size_t)a.D * stride_d) return;
  const int d = (int)(e / stride_d);
  size_t q = e - d * stride_d;
  const float* fac = a.gvec + ((size_t)r * a.D + d) * 2 * W;          // [gh_{d+1} | ga_d]
  const float* tape = a.tape + (size_t)r * (2 * a.D + 1) * W;
  const float* rowf;   // factor over rows i
  const float* colv;   // vector over columns j (nullptr: bias)
  if (q < (size_t)W * W) {                       rowf = fac + W; colv = tape + (size_t)d * W; }                      // W1
  else if ((q -= (size_t)W * W) < (size_t)W) {   rowf = fac + W; colv = nullptr; }                                 // b1
  else if ((q -= W) < (size_t)W * W) {           rowf = fac;     colv = tape + (size_t)(a.D + 1 + d) * W; }        // W2
  else {                                         q -= (size_t)W * W; rowf = fac; colv = nullptr; }                 // b2
  float g[4];
  if (colv) {
    const int i = (int)(q / W), j = (int)(q - (size_t)i * W);
    const float fi = rowf[i];
    const float4 c4 = *reinterpret_cast<const float4*>(colv + j);
    g[0] = fi * c4.x; g[1] = fi * c4.y; g[2] = fi * c4.z; g[3] = fi * c4.w;
  } else {
    const float4 f4 = *reinterpret_cast<const float4*>(rowf + q);
    g[0] = f4.x; g[1] = f4.y; g[2] = f4.z; g[3] = f4.w;
  }
  const size_t o = (size_t)r * a.P + a.o_blk + e;
  if (MODE == NM_GRAD) {
    *reinterpret_cast<float4*>(a.gtheta + o) = make_float4(g[0], g[1], g[2], g[3]);
    return;
  }
  if (!upd) return;
  float4 w4 = *reinterpret_cast<float4*>(a.theta + o), m4 = *reinterpret_cast<float4*>(a.m + o),
         v4 = *reinterpret_cast<float4*>(a.v + o);
  w4.x = ad.upd(w4.x, m4.x, v4.x, g[0]);
  w4.y = ad.upd(w4.y, m4.y, v4.y, g[1]);
  w4.z = ad.upd(w4.z, m4.z, v4.z, g[2]);
  w4.w = ad.upd(w4.w, m4.w, v4.w, g[3]);
  *reinterpret_cast<float4*>(a.theta + o) = w4;
  *reinterpret_cast<float4*>(a.m + o) = m4;
  *reinterpret_cast<float4*>(a.v + o) = v4;
}

// The parameter-update pass: W_in (and b_in) blocks [0, n_in ceil(W/8)), then the hidden-parameter
// blocks; grid (n_in ceil(W/8) + n_hid, R), 256 threads.  NM_FWD: the W_in y0 partials only.
template <int MODE, bool VEC>
__global__ void __launch_bounds__(256) k_net_upd(NetArgs a) {
  SQ_PDL_WAIT();
  const int r = blockIdx.y;
  bool upd = true;
  AdamC ad{};
  if (MODE == NM_ADAM) {
    upd = !(*a.status & ST_NONFINITE);  // keep the last finite iterate
    ad = adam_c(a.ap);
  }
  const int wy = (a.W + 7) / 8, nin = a.n_in * wy;
  if ((int)blockIdx.x < nin) net_in_block<MODE, VEC>(a, blockIdx.x % a.n_in, blockIdx.x / a.n_in, r, ad, upd);
  else if (MODE != NM_FWD) net_hid_block<MODE>(a, blockIdx.x - nin, r, ad, upd);
}

// ----------------------------------------------------------------------------------- hidden layers
// One cluster of NET_CL CTAs per restart (grid (NET_CL, R)), 128 threads.  CTA c owns rows
// [c RW, (c+1) RW) of every hidden matrix, RW = W / NET_CL; its rows of W1_d and W2_d are one
// contiguous block each in theta, staged in shared memory at entry.
// One elected thread stages the CTA's slices of all 2D hidden matrices (and optionally the tape) with
// bulk async copies; every thread later waits on `bar` (phase 0).  Returns immediately when D = 0.
__device__ __forceinline__ void stage_slices(const NetArgs& a, const float* th, int c, int RW, float* wsl,
                                             const float* tape_src, float* tape_dst, uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar);
    const uint32_t blk = RW * a.W;  // floats per matrix slice (a multiple of 4)
    const uint32_t bytes = 2u * a.D * blk * 4u + (tape_dst ? (2u * a.D + 1u) * a.W * 4u : 0u);
    if (bytes) {
      mbar_expect_tx(bar, bytes);
      const size_t stride_d = 2 * (size_t)a.W * a.W + 2 * (size_t)a.W;
      for (int s = 0; s < 2 * a.D; ++s) {
        const int d = s >> 1, which = s & 1;  // 0: W1_d, 1: W2_d
        const size_t o = a.o_blk + d * stride_d + (which ? (size_t)a.W * a.W + a.W : 0) + (size_t)c * blk;
        bulk_g2s(wsl + (size_t)s * blk, th + o, blk * 4u, bar);
      }
      if (tape_dst) bulk_g2s(tape_dst, tape_src, (2u * a.D + 1u) * a.W * 4u, bar);
    }
  }
}

// Column-slice reduction: CTA c sums partials[q][c RW + jl] over q < n (fixed order per thread,
// S = blockDim / RW threads per column, 4 independent chains); result in sred[t].
__device__ __forceinline__ void slice_partial(const float* pp, int n, int W, int RW, float* sred) {
  const int t = threadIdx.x, S = blockDim.x / RW, q0 = t / RW;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int q = q0;
  for (; q + 3 * S < n; q += 4 * S) {
    s0 += pp[(size_t)q * W];
    s1 += pp[(size_t)(q + S) * W];
    s2 += pp[(size_t)(q + 2 * S) * W];
    s3 += pp[(size_t)(q + 3 * S) * W];
  }
  for (; q < n; q += S) s0 += pp[(size_t)q * W];
  sred[t] = (s0 + s1) + (s2 + s3);
}

// Up to 4 rows per warp (RW <= 16): partial dots of the CTA's rows il = warp + 4k of matrix s with the
// shared vector x, reduced across the warp together (4 independent shuffle chains).
__device__ __forceinline__ void rows_dot4(const float* wsl, int s, int RW, int W, const float* x, int warp, int lane,
                                          float p[4]) {
  const float4 xv = lane < (W >> 2) ? reinterpret_cast<const float4*>(x)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int il = warp + 4 * k;
    p[k] = 0.f;
    if (il < RW && lane < (W >> 2)) {
      const float4 w = reinterpret_cast<const float4*>(wsl + ((size_t)s * RW + il) * W)[lane];
      p[k] = w.x * xv.x;
      p[k] = fmaf(w.y, xv.y, p[k]);
      p[k] = fmaf(w.z, xv.z, p[k]);
      p[k] = fmaf(w.w, xv.w, p[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] += __shfl_xor_sync(0xffffffffu, p[k], o);
}

// The tape rows double as the DSMEM exchange buffers (each written once): every CTA holds the full
// tape tv = [h_0..h_D | u_0..u_{D-1}] in shared memory and writes its column slice to global at the
// end.  Exchange phase k (0: h_0, 1 + 2d: u_d, 2 + 2d: h_{d+1}) completes on xbar[k].
__global__ void __cluster_dims__(NET_CL, 1, 1) __launch_bounds__(128) k_net_mid_fwd(NetArgs a) {
  SQ_PDL_WAIT();
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) uint64_t bar, xbar[2 * NET_MAXD + 1];
  __shared__ float sred[128];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), r = blockIdx.y, t = threadIdx.x;
  const int W = a.W, RW = W / NET_CL, lane = t & 31, warp = t >> 5, D = a.D;
  float* wsl = sm;                              // [2D][RW][W]
  float* tv = wsl + (size_t)2 * D * RW * W;     // [2D+1][W] tape
  float* bsl = tv + (size_t)(2 * D + 1) * W;    // [2D][RW] the CTA's rows of b1_d, b2_d
  const float* th = a.theta + (size_t)r * a.P;
  stage_slices(a, th, c, RW, wsl, nullptr, nullptr, &bar);  // overlaps the h_0 reduction below
  if (t == 0)
    for (int k = 0; k <= 2 * D; ++k) {
      mbar_init(&xbar[k]);
      mbar_expect_tx(&xbar[k], W * 4u);  // one full row per phase (RW floats from each CTA)
    }
  const size_t stride_d = 2 * (size_t)W * W + 2 * (size_t)W;
  for (int k = t; k < 2 * D * RW; k += blockDim.x) {
    const int s2 = k / RW, il = k - s2 * RW;
    bsl[k] = th[a.o_blk + (s2 >> 1) * stride_d + (size_t)W * W + (s2 & 1) * ((size_t)W * W + W) + c * RW + il];
  }
  // h_0: CTA c reduces its RW columns of the W_in y0 partials and pushes tanh(.) to every CTA
  slice_partial(a.pin + (size_t)r * a.n_in * W + c * RW + t % RW, a.n_in, W, RW, sred);
  cl.sync();  // barriers initialized in every CTA before the first st.async
  if (t < RW) {
    const int j = c * RW + t;
    float g = th[a.o_bin + j];
    for (int k = 0; k < (int)blockDim.x / RW; ++k) g += sred[k * RW + t];
    push_all(tv + j, tanhf(g), &xbar[0]);
  }
  if (D) mbar_wait(&bar, 0);
  mbar_wait(&xbar[0], 0);
  float p[4];
  for (int d = 0; d < D; ++d) {
    const float* h = tv + (size_t)d * W;
    float* u = tv + (size_t)(D + 1 + d) * W;
    rows_dot4(wsl, 2 * d, RW, W, h, warp, lane, p);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int il = warp + 4 * k;
      if (il < RW && lane < NET_CL)
        st_async(mapa_u32(smem_u32(u + c * RW + il), lane), tanhf(p[k] + bsl[2 * d * RW + il]),
                 mapa_u32(smem_u32(&xbar[1 + 2 * d]), lane));
    }
    mbar_wait(&xbar[1 + 2 * d], 0);
    rows_dot4(wsl, 2 * d + 1, RW, W, u, warp, lane, p);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int il = warp + 4 * k;
      const int i = c * RW + il;
      if (il < RW && lane < NET_CL)
        st_async(mapa_u32(smem_u32(tv + (size_t)(d + 1) * W + i), lane), h[i] + p[k] + bsl[(2 * d + 1) * RW + il],
                 mapa_u32(smem_u32(&xbar[2 + 2 * d]), lane));
    }
    mbar_wait(&xbar[2 + 2 * d], 0);
  }
  float* tape = a.tape + (size_t)r * (2 * D + 1) * W;
  for (int k = t; k < (2 * D + 1) * RW; k += blockDim.x) {  // the CTA's column slice of the tape
    const int row = k / RW, j = c * RW + (k - row * RW);
    tape[(size_t)row * W + j] = tv[(size_t)row * W + j];
  }
  // every CTA received all of its expected bytes, so no st.async can still target this CTA
}

// Reverse mode through the hidden layers (old weights from shared memory).  Writes the factor vectors
// of every hidden parameter's outer-product gradient, gvec[r][d] = [gh_{d+1} | ga_d], and
// ga0 = dL/d(W_in y0 + b_in); the parameter updates are done by the wide kernels k_net_hid / k_net_in.
// Exchange phases: 0 the gh slices (W floats), then per layer (from d = D-1 down) the CTA partials of
// W2_d^T gh and of W1_d^T ga (NET_CL x W floats each) into xb[0] / xb[1]; a buffer is refilled only
// after every CTA has consumed it (the refill needs data each CTA sends after its reads).
__global__ void __cluster_dims__(NET_CL, 1, 1) __launch_bounds__(128) k_net_mid_bwd(NetArgs a) {
  SQ_PDL_WAIT();
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) uint64_t bar, xbar[2 * NET_MAXD + 1];
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), r = blockIdx.y;
  const int W = a.W, RW = W / NET_CL, D = a.D, t = threadIdx.x;
  float* wsl = sm;                                // [2D][RW][W] old weights
  float* tv = wsl + (size_t)2 * D * RW * W;       // [2D+1][W] tape: h_0..h_D, u_0..u_{D-1}
  float* gh = tv + (size_t)(2 * D + 1) * W;       // [W]
  float* ga = gh + W;                             // [W]
  float* xb = ga + W;                             // [2][NET_CL][W] transposed partials per source CTA
  float* sred = xb + 2 * NET_CL * W;              // [128] partial sums of the W_out^T go reduction
  float* gv = sred + 128;                         // [D][2][W] factor vectors (written to global at the end)
  const float* th = a.theta + (size_t)r * a.P;
  const float* tape = a.tape + (size_t)r * (2 * D + 1) * W;
  float* gvec = a.gvec + (size_t)r * D * 2 * W;
  stage_slices(a, th, c, RW, wsl, tape, tv, &bar);  // weights + tape, overlapping the reduction below
  if (t == 0) {
    mbar_init(&xbar[0]);
    mbar_expect_tx(&xbar[0], W * 4u);
    for (int k = 1; k <= 2 * D; ++k) {
      mbar_init(&xbar[k]);
      mbar_expect_tx(&xbar[k], NET_CL * W * 4u);
    }
  }
  // gh = W_out^T go: CTA c reduces its RW columns over the n_out partials, pushes them to all CTAs
  slice_partial(a.pout + (size_t)r * a.n_out * W + c * RW + t % RW, a.n_out, W, RW, sred);
  cl.sync();  // barriers initialized in every CTA before the first st.async
  if (t < RW) {
    float g = 0.f;
    for (int k = 0; k < (int)blockDim.x / RW; ++k) g += sred[k * RW + t];
    push_all(gh + c * RW + t, g, &xbar[0]);
  }
  mbar_wait(&bar, 0);  // (the tape is always staged, so the barrier always completes)
  mbar_wait(&xbar[0], 0);
  int ph = 1;
  for (int d = D - 1; d >= 0; --d, ph += 2) {
    const float* u = tv + (size_t)(D + 1 + d) * W;
    for (int j = t; j < W; j += blockDim.x) {  // partial of W2^T gh over the CTA's rows
      float p = 0.f;
      for (int il = 0; il < RW; ++il) p = fmaf(wsl[((size_t)(2 * d + 1) * RW + il) * W + j], gh[c * RW + il], p);
      push_all(xb + (size_t)c * W + j, p, &xbar[ph]);
      gv[(size_t)d * 2 * W + j] = gh[j];  // dL/dh_{d+1}: W2_d, b2_d
    }
    mbar_wait(&xbar[ph], 0);
    for (int j = t; j < W; j += blockDim.x) {  // ga = (W2^T gh) tanh'(.)
      float s = 0.f;
      for (int q = 0; q < NET_CL; ++q) s += xb[(size_t)q * W + j];
      ga[j] = s * (1.f - u[j] * u[j]);
      gv[(size_t)d * 2 * W + W + j] = ga[j];  // W1_d, b1_d
    }
    __syncthreads();
    float* xb1 = xb + (size_t)NET_CL * W;
    for (int j = t; j < W; j += blockDim.x) {  // partial of W1^T ga
      float p = 0.f;
      for (int il = 0; il < RW; ++il) p = fmaf(wsl[((size_t)(2 * d) * RW + il) * W + j], ga[c * RW + il], p);
      push_all(xb1 + (size_t)c * W + j, p, &xbar[ph + 1]);
    }
    mbar_wait(&xbar[ph + 1], 0);
    for (int j = t; j < W; j += blockDim.x) {  // skip path + inner path
      float s = 0.f;
      for (int q = 0; q < NET_CL; ++q) s += xb1[(size_t)q * W + j];
      gh[j] += s;
    }
    __syncthreads();
  }
  if (c == 0) {  // ga0 = gh tanh'(a_0) and the factor vectors
    for (int j = t; j < W; j += blockDim.x) a.ga0[(size_t)r * W + j] = gh[j] * (1.f - tv[j] * tv[j]);
    for (int k = t; k < 2 * D * W; k += blockDim.x) gvec[k] = gv[k];
  }
  // every CTA received all of its expected bytes, so no st.async can still target this CTA
}

NetArgs make_args(const NetDims& d, const NetWs& ws) {
  NetArgs a{};
  a.Din = d.Din; a.W = d.W; a.D = d.D; a.n_in = d.n_in; a.n_out = d.n_out;
  a.P = d.P; a.o_bin = d.o_bin; a.o_blk = d.o_blk; a.o_wout = d.o_wout; a.o_bout = d.o_bout;
  a.tape = ws.tape; a.pin = ws.pin; a.pout = ws.pout; a.ga0 = ws.ga0; a.gvec = ws.gvec;
  return a;
}

template <int MODE>
void launch_upd(const NetDims& d, const NetArgs& a, cudaStream_t st) {
  const dim3 g(d.n_in * ((d.W + 7) / 8) + (MODE == NM_FWD ? 0 : d.n_hid), d.R);
  if (d.Din % 4 == 0) k_net_upd<MODE, true><<<g, 256, 0, st>>>(a);
  else k_net_upd<MODE, false><<<g, 256, 0, st>>>(a);
}

}  // namespace

bool net_dims(int R, int Din, int W, int D, NetDims* out, const char** why) {
  NetDims d;
  if (R < 1 || Din < 1) { *why = "generator: R and M N must be positive"; return false; }
  if (W < 8 || W > 128 || W % 8) { *why = "generator: net_width must be a multiple of 8 in [8, 128]"; return false; }
  if (D < 0 || D > NET_MAXD) { *why = "generator: net_depth must be in [0, 15]"; return false; }
  d.R = R; d.Din = Din; d.W = W; d.D = D;
  const size_t w = W, din = Din;
  d.o_bin = w * din;
  d.o_blk = d.o_bin + w;
  d.o_wout = d.o_blk + (size_t)D * (2 * w * w + 2 * w);
  d.o_bout = d.o_wout + din * w;
  d.P = (d.o_bout + din + 3) & ~(size_t)3;  // per-restart stride: float4-aligned restarts
  d.n_in = (Din + NET_IN_COLS - 1) / NET_IN_COLS;
  d.n_out = ((Din + NET_OUT_ROWS - 1) / NET_OUT_ROWS + NET_CL - 1) / NET_CL;  // clusters of k_net_out_bwd
  d.n_hid = (int)(((size_t)D * (2 * w * w + 2 * w) / 4 + 255) / 256);
  const size_t RW = W / NET_CL;
  d.smem_fwd = (2 * (size_t)D * RW * w + (2 * (size_t)D + 1) * w + 2 * (size_t)D * RW) * sizeof(float);
  d.smem_bwd = (2 * (size_t)D * RW * w + (2 * (size_t)D + 1) * w + 2 * w + 2 * NET_CL * w + 128 + 2 * (size_t)D * w) *
               sizeof(float);
  if (d.smem_bwd > 200 * 1024) { *why = "generator: hidden layers exceed the cluster's shared memory (depth too large)"; return false; }
  // (a single-CTA variant streaming the hidden matrices through a TMA ring measured slower than the
  // 8-CTA cluster at C3 -- forward 18.4 vs 10.8 us, backward 16.6 vs 11.9 us: one SM pulls the 640 KB
  // of hidden weights at ~50 GB/s -- and was removed in round 2)
  *out = d;
  return true;
}

size_t net_ws_floats(const NetDims& d) {
  const size_t w = d.W;
  return (size_t)d.R * ((2 * (size_t)d.D + 1) * w + (size_t)d.n_in * w + (size_t)d.n_out * w + w +
                        2 * (size_t)d.D * w) + 16;
}

NetWs net_ws_carve(const NetDims& d, float* base) {
  NetWs ws;
  const size_t w = d.W;
  ws.tape = base;
  ws.pin = ws.tape + (size_t)d.R * (2 * d.D + 1) * w;
  ws.pout = ws.pin + (size_t)d.R * d.n_in * w;
  ws.ga0 = ws.pout + (size_t)d.R * d.n_out * w;
  ws.gvec = ws.ga0 + (size_t)d.R * w;
  return ws;
}

cudaError_t net_prepare(const NetDims& d) {
  cudaError_t e;
  e = cudaFuncSetAttribute(k_net_mid_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem_fwd);
  if (e) return e;
  return cudaFuncSetAttribute(k_net_mid_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem_bwd);
}

cudaError_t net_forward(const NetDims& d, const NetWs& ws, const float* theta, const float* y0, float* z,
                        bool fresh_in, cudaStream_t st, int64_t* launches) {
  NetArgs a = make_args(d, ws);
  a.theta = const_cast<float*>(theta);  // read-only in the forward kernels
  a.y0 = y0;
  a.z = z;
  if (fresh_in) {
    launch_upd<NM_FWD>(d, a, st);
    *launches += 1;
  }
  k_net_mid_fwd<<<dim3(NET_CL, d.R), 128, d.smem_fwd, st>>>(a);
  k_net_out<<<dim3((d.Din + NET_FWD_ROWS - 1) / NET_FWD_ROWS, d.R), 256, 0, st>>>(a);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t net_backward(const NetDims& d, const NetWs& ws, float* theta, const float* y0, const float* z,
                         const float* gz, float* gtheta, float* m, float* v, const AdamP& ap, const int* status,
                         cudaStream_t st, int64_t* launches) {
  NetArgs a = make_args(d, ws);
  a.theta = theta; a.y0 = y0; a.z = const_cast<float*>(z); a.gz = gz; a.gtheta = gtheta;
  a.m = m; a.v = v; a.ap = ap; a.status = status;
  const dim3 go(d.n_out * NET_CL, d.R), gm(NET_CL, d.R);
  if (gtheta) {
    k_net_out_bwd<NM_GRAD><<<go, 256, 0, st>>>(a);
    k_net_mid_bwd<<<gm, 128, d.smem_bwd, st>>>(a);
    launch_upd<NM_GRAD>(d, a, st);
  } else {
    k_net_out_bwd<NM_ADAM><<<go, 256, 0, st>>>(a);
    k_net_mid_bwd<<<gm, 128, d.smem_bwd, st>>>(a);
    launch_upd<NM_ADAM>(d, a, st);
  }
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace sq
