// Low-rank Doppler engine: Chebyshev-node interpolation of the
// AF in Doppler, for narrow uniform grids.
//
// Eq. 6 with the Doppler phase centred on n_c = (N+1)/2:
//   A(tau, f) = e^{j 2 pi n_c f / N} At(tau, f),
//   At(tau, f) = sum_n s(n) e^{j 2 pi (n - n_c) f / N} conj(w(n + tau)).
// |A| = |At|, and the loss (Eqs. 7-9, 37-42) sees the AF only through |A|, so the
// engine works with At throughout; its cotangent is G~ = dL/dAt^* (same form as
// a7: phi w At / |At|).  As a function of f, At(tau, .) is a band-limited
// trigonometric polynomial whose frequencies (n - n_c)/N lie in [-1/2, 1/2]; on a
// grid of width <= 1 (the paper's [-0.5, 0.5]) it is interpolated to
// ~5e-8 relative accuracy by Q = 10 Chebyshev nodes f*_q (first kind):
//   At(tau, f_k) = sum_q l_q(f_k) At(tau, f*_q)      (l_q: Lagrange basis, real).
// The node AFs R_q(tau) = At(tau, f*_q) are exact correlations, computed by the FFT
// path of Eq. 36 with the node modulation V_q(n) = e^{j 2 pi (n - n_c) f*_q / N}
// (k_xhat + k_node); the dense (K x Q) Doppler contraction and its adjoint run
// fused with the cell epilogue in k_lr; the adjoint correlations go back through
// the FFT path at the Q nodes only (k_adj_g, k_adj_gc).  Transforms per
// evaluation drop from O(M^2 K) to O(M^2 Q).
//
// Symmetry: the uniform grid and the Chebyshev nodes are both symmetric about the
// grid centre, so l_q(f_{K-1-k}) = l_{Q-1-q}(f_k).  With E_q = R_q + R_{Q-1-q},
// O_q = R_q - R_{Q-1-q}, alpha_q = (l_q + l_{Q-1-q})/2, beta_q = (l_q - l_{Q-1-q})/2
// (q < Q/2):  At(f_k) = Pe + Po,  At(f_{K-1-k}) = Pe - Po,  Pe = sum alpha E,
// Po = sum beta O -- one bin pair costs Q complex-by-real FMAs each way instead of 2Q.
#pragma once
#include <stdint.h>

#include <cuda_fp16.h>

#include "af_kernels.cuh"
#include "common.cuh"

#ifndef SQNGD_NODE_PK  // k_node's transforms: scalar complex arithmetic (packed: 110 vs 85 registers, slower)
#define SQNGD_NODE_PK 0
#endif
#ifndef SQNGD_LRT_PREFETCH
#define SQNGD_LRT_PREFETCH 0
#endif

namespace sq {

// Per-restart record of the Chebyshev engine, filled by k_lr with order-independent
// atomics (max of the unit shifts as positive-float bits, max of the packed keys), so
// the result is deterministic; reset by k_node of the same evaluation.
struct LrRed {
  unsigned int mbits;  // max unit shift (float bits; 0 = none)
  unsigned int tie_a;  // 1 + float bits of the largest value at which a unit saw two of its cells tie (auto)
  unsigned long long key_a, key_c;
  unsigned int tie_c;  // (cross maps)
  unsigned int pad;
};

// Warp max of packed keys that also notes a tie: at the butterfly stage where the two halves holding
// two distinct cells of the maximal value meet, both halves carry that value with different indices.
__device__ __forceinline__ unsigned long long warp_key_max_tie(unsigned long long key, uint32_t& tv) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
    if (y && key && (y >> 32) == (key >> 32) && y != key) tv = max(tv, (uint32_t)(key >> 32) + 1u);
    key = y > key ? y : key;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tv = max(tv, __shfl_xor_sync(0xffffffffu, tv, o));
  return key;
}

// Node AFs for every unit (r, m, l, q): R_{ml,q}(tau) = IFFT_P(X~_{m,q} conj(H_l))[(-tau) mod P]
// (Eq. 36, Q1), stored at Rn[((r M + m) M + l) Q + q][tau + N - 1].
template <class PL, int G, int MINB>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_node(int u0, int units, int M, int Q, int N, int LS, const float2* __restrict__ Xc, const float2* __restrict__ H,
           const float2* __restrict__ ftw, float2* __restrict__ Rn, int R, LrRed* lred) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  if (blockIdx.x == 0)  // this evaluation's k_lr maxima
    for (int i = threadIdx.x; i < R; i += blockDim.x) lred[i] = LrRed{};
  const int uu = u0 + (u < units ? u : units - 1);  // units [u0, u0 + units): this rank's rows
  const int q = uu % Q, pr = uu / Q;  // pr = (r M + m) M + l
  const int l = pr % M, rm = pr / M, r = rm / M;
  const float2* X = Xc + ((size_t)rm * Q + q) * P;
  const float2* Hl = H + ((size_t)r * M + l) * P;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = cmulc(__ldg(Hl + t + i * T), __ldg(X + t + i * T));  // conj(X conj(H))
  int par = 0;
  fft<PL, -1, false, SQNGD_NODE_PK>(v, ftw, xbuf, t, par, sync);  // v = conj(r)
  if (u >= units) return;
  float2* out = Rn + (size_t)uu * LS + (N - 1);
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = t + i * T;
    if (j < N || j > P - N) out[lag_of(j, N, P)] = make_float2(v[i].x, -v[i].y);
  }
}

struct LrArgs {
  int R, M, N, L, K, nch, kw, LS, QS;  // kw: warps (bin-pair ranges) per unit; QS: coefficient row stride
  int tau_lo, tau_hi, excl0;
  float bp, invN;
  const float* weights;  // [K][L] or nullptr
  const float* wmax;     // [L] max_k weights (HW only)
  const float* coef;     // [(K/2) + 1][QS]: alpha_0..alpha_{Q/2-1}, beta_0..beta_{Q/2-1}; last row: middle bin
  const float2* Rn;      // [R M M][Q][LS] node AFs
  float2* Gn;            // [R M M][Q][LS] node cotangents (scaled to the unit shift)
  float* af_mag;         // [R][M][M][K][L] or nullptr (forward only)
  Part part;             // unit slots, u = pair nch + chunk
  LrRed* lred;           // [R]
};

// One Doppler cell of the fused epilogue (a5 / a7): key tracking, surrogate term, cotangent.
// LM: 0 MAX (keys only), 1 LSE, 2 PNORM.  Returns G~ (unnormalised: gphi w At / |At|).
template <int LM, bool HW, bool GRAD, bool GE_RULE, bool GF_ONLY = false>
__device__ __forceinline__ float2 lr_cell(float2 A, int k, const LrArgs& a, int idx, bool valid, float lbN, float nlbs,
                                          float qN, float& best, int& bk, float& S, float* mcell, bool mst,
                                          float msc = 1.f) {
  // |A|^2 + 1e-30: the floor keeps rsqrt finite at A = 0 and is far below one ulp of any
  // non-negligible cell, so the key and the magnitude are unchanged
  const float a2 = fmaf(A.x, A.x, fmaf(A.y, A.y, 1e-30f));
  float wt = 1.f, kv = a2;
  if (HW) {
    wt = valid ? __ldg(a.weights + (size_t)k * a.L + idx) : 0.f;
    kv = wt > 0.f ? a2 * wt * wt : -1.f;
  }
  const bool upd = GE_RULE ? (kv >= best) : (kv > best);
  best = upd ? kv : best;
  bk = upd ? k : bk;
  if (LM == 0) {
    if (mst) *mcell = sqrtf(a2) * msc;  // (mcell: this cell's |A| map address)
    return make_float2(0.f, 0.f);
  }
  const float rsq = rsqa(a2);
  const float mag = a2 * rsq;
  if (mst) *mcell = mag * msc;
  float phi, gphi;
  if (LM == 1) {
    phi = ex2a(fmaf(lbN, HW ? wt * mag : mag, nlbs));
    if (HW) phi = wt > 0.f ? phi : 0.f;
    gphi = phi;
  } else {
    const float q = (HW ? wt * mag : mag) * qN;
    gphi = ex2a((a.bp - 1.f) * lg2a(q));
    phi = gphi * q;
  }
  S += phi;
  if (!GRAD) return make_float2(0.f, 0.f);
  const float gf = gphi * (HW ? wt * rsq : rsq);
  if (GF_ONLY) return make_float2(gf, 0.f);  // the caller forms gf A itself (fused into its sums)
  return make_float2(A.x * gf, A.y * gf);
}

// Rescale factor of a sum accumulated with shift `from` to the shift `to` (LSE: e^{beta(from-to)};
// PNORM: (from/to)^(p-1) for the cotangents, times from/to for the sum).
template <int LM>
__device__ __forceinline__ void lr_rescale(float from, float to, float lb, float bp, float& fS, float& fG) {
  if (LM == 1) {
    fS = fG = ex2a(lb * (from - to));
  } else {
    const float rt = to > 0.f ? from / to : 0.f;
    fG = rt > 0.f ? ex2a((bp - 1.f) * lg2a(rt)) : 0.f;
    fS = fG * rt;
  }
}

// ---------------------------------------------------------------------------------------
// Tensor-core variant of k_lr: the Doppler contraction and its adjoint as warp-level
// mma.sync m16n8k8 TF32 products in 3xTF32 form (a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi,
// fp32 accumulation: ~2^-21 relative, near the fp32 path's accuracy).  A warp owns 16 lags x a
// range of 8-pair tiles; with g = lane / 4, c = lane % 4 a thread holds lags g and g + 8.
//   forward  Pe = E . alpha, Po = O . beta : A[16 lags x 8 (j < Q/2, zero-padded)] x B[8 x 8 pairs]
//   adjoint  GE += SG . alpha^T, GO += DG . beta^T : A[16 lags x 8 pairs] x B[8 pairs x 8 j]
// The forward D fragment (rows g, g+8; pairs 2c, 2c+1) is exactly the adjoint A fragment
// once the tile's pairs are ordered (2c -> k-column c, 2c+1 -> c+4), so G never leaves the
// registers.  B fragments come pre-split (hi, lo) and pre-permuted from the host tables.
// The middle bin of an odd K (f = grid centre, beta = 0) is one extra cell per lag, done on
// the CUDA cores by the last warp of the unit.
struct LrtArgs {
  int R, M, N, L, K, nch, kw, LS, NT, NTF;  // nch: 16-lag chunks; NT: 8-pair tiles of the K/2 bin pairs; NTF: full ones
  int row0;                                 // first (restart, transmit channel) row of this rank's shard
  int tau_lo, tau_hi, excl0;
  float bp, invN;
  const float* weights;  // [K][L] or nullptr
  const float* wmax;     // [L]
  const float4* tabF;    // [NT][32][2]: forward B fragments {a_b0h, a_b1h, a_b0l, a_b1l}, {beta ...}
  const float4* tabA;    // [NT][32][2]: adjoint B fragments
  const float* coefm;    // [Q/2] middle-bin coefficients l_j(f_centre) (odd K)
  const uint4* tabF16;   // [NT][32]: forward B fragments, m16n8k16 f16 {alpha b0, b1, beta b0, b1}
  const uint2* tabM16;   // [32]: middle-bin B fragment (column 0)
  const float2* Rn;      // [R M M][Q][LS]
  float2* Gn;            // [R M M][Q][LS]
  float* af_mag;         // forward only
  int mld;               // |A| map row pitch (floats)
  Part part;             // unit slots, u = pair nch + chunk
  LrRed* lred;
};

// x = hi + lo with hi = x truncated to TF32 (the tensor core reads the top 19 bits of an
// operand register, so hi may be passed as the bits of x itself) and lo = x - hi exact.
// (cvt.rna.tf32 is emulated on sm_100a: 4 integer ops; truncation is 2: LOP3 + FADD.)
__device__ __forceinline__ void tf32_split(float x, uint32_t& h, uint32_t& l) {
  h = __float_as_uint(x);
  l = __float_as_uint(x - __uint_as_float(h & 0xFFFFE000u));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += (ah + al)(bh + bl), the al bl term dropped; small terms first.
__device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], float4 b) {
  mma_tf32(d, al, __float_as_uint(b.x), __float_as_uint(b.y));
  mma_tf32(d, ah, __float_as_uint(b.z), __float_as_uint(b.w));
  mma_tf32(d, ah, __float_as_uint(b.x), __float_as_uint(b.y));
}
__device__ __forceinline__ void split4(const float (&x)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) tf32_split(x[i], h[i], l[i]);
}

// split4 with the A-fragment reorder of k_lrt's adjoint (x in D order: (g,2c) (g,2c+1) (g+8,2c) (g+8,2c+1);
// h, l in A order (g,c) (g+8,c) (g,c+4) (g+8,c+4)), the two subtractions per pair packed.
__device__ __forceinline__ void split4_pk(const float (&x)[4], uint32_t (&h)[4], uint32_t (&l)[4]);

// Forward contraction in FP16 with the 3-term split packed along K (m16n8k16, one MMA per
// product): the 15 used K columns hold hi(x_j), lo(x_j), hi(x_j) against hi(c_j), hi(c_j),
// lo(c_j) (j < 5; layout in k_lrt), so A.B = x_hi c_hi + x_lo c_hi + x_hi c_lo.
// Range: |x| <= 2N <= 8192 and |c| < 3 fit FP16; lo parts below the FP16 normal range lose at
// most 6e-8 absolute each, i.e. < 2e-7 N per cell (the parity floor is 2e-6 N).
#ifndef SQNGD_LRT_F16
#define SQNGD_LRT_F16 1
#endif
__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// K-column k of the packed split of x[0..4] (k < 15), as an FP16 value
__device__ __forceinline__ unsigned short f16_col(int k, const float (&x)[5]) {
  const int part = k / 5, j = k - 5 * part;
  float v = x[0];
  v = j == 1 ? x[1] : v;
  v = j == 2 ? x[2] : v;
  v = j == 3 ? x[3] : v;
  v = j == 4 ? x[4] : v;
  const __half hi = __float2half_rn(v);
  const __half lo = __float2half_rn(v - __half2float(hi));
  const __half r = part == 1 ? lo : (part < 3 ? hi : __float2half_rn(0.f));
  return __half_as_ushort(r);
}
__device__ __forceinline__ uint32_t f16_pair(int k, const float (&x)[5]) {
  return (uint32_t)f16_col(k, x) | ((uint32_t)f16_col(k + 1, x) << 16);
}

#ifndef SQNGD_LRT_PACKED
#define SQNGD_LRT_PACKED 1
#endif

__device__ __forceinline__ void split4_pk(const float (&x)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
  // x in D order; the fragment quads h, l pair (x0, x2) and (x1, x3), so the subtractions pack over those
  const f32x2 v02 = pk2(x[0], x[2]), v13 = pk2(x[1], x[3]);
  const f32x2 t02 = pk2(__uint_as_float(__float_as_uint(x[0]) & 0xFFFFE000u), __uint_as_float(__float_as_uint(x[2]) & 0xFFFFE000u));
  const f32x2 t13 = pk2(__uint_as_float(__float_as_uint(x[1]) & 0xFFFFE000u), __uint_as_float(__float_as_uint(x[3]) & 0xFFFFE000u));
  const f32x2 d02 = sub2(v02, t02), d13 = sub2(v13, t13);
  h[0] = __float_as_uint(x[0]); h[1] = __float_as_uint(x[2]); h[2] = __float_as_uint(x[1]); h[3] = __float_as_uint(x[3]);
  l[0] = __float_as_uint(lo2(d02)); l[1] = __float_as_uint(hi2(d02));
  l[2] = __float_as_uint(lo2(d13)); l[3] = __float_as_uint(hi2(d13));
}

#ifndef SQNGD_LRT_UNROLL
#define SQNGD_LRT_UNROLL 1
#endif
constexpr int kLrtUnroll = SQNGD_LRT_UNROLL;  // tile-loop unroll of k_lrt (tuning)

// one warp per CTA (kw = 1); 16 resident CTAs/SM caps the registers at 128 (no spills).  Re-measured
// after the FP16 forward / lane-owned K layout: 128 registers beat the former cap of 96 (20 CTAs/SM,
// 12 B of spills) by 2% at C3 (1.804 vs 1.840 ms per step) and 2.5% at C5; 154 registers (12 CTAs)
// and a tile-loop unroll of 2 were slower (tools: SQNGD_LRT_MINB / SQNGD_LRT_UNROLL).
#ifndef SQNGD_LRT_MAXT
#define SQNGD_LRT_MAXT 32
#define SQNGD_LRT_MINB 16
#endif
// KM: kernel mode -- 0 forward (sums, keys), 1 forward + adjoint (cotangents), 2 forward writing the
// |A| map; the map stores are compiled only into mode 2.
template <int Q, int LM, bool HW, int KM>
__global__ void __launch_bounds__(SQNGD_LRT_MAXT, SQNGD_LRT_MINB) k_lrt(const LrtArgs a) {
  SQ_PDL_WAIT();
  constexpr bool GRAD = KM == 1, MAP = KM == 2;
  constexpr bool PK = SQNGD_LRT_PACKED && !HW && !MAP;  // packed-FP32 epilogue for the full tiles
  constexpr int QH = Q / 2;
  constexpr int NR = 6 + (GRAD ? 16 : 0);  // per-lane record: key(2), shift(2), S(2), GE/GO(16)
  extern __shared__ float4 lr_smem[];
  float* rs = reinterpret_cast<float*>(lr_smem);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int g = lane >> 2, cq = lane & 3;
  // grid (chunk, m M + l, restart): no integer divisions by runtime sizes
  // grid (chunk, l, row - row0): row = r M + m is this rank's (restart, transmit channel) row
  const int ch = blockIdx.x;
  const int rm = a.row0 + (int)blockIdx.z;
  const int pr = rm * a.M + blockIdx.y;
  const int u = pr * a.nch + ch;
  const int M = a.M;
  const int rr_ = rm / M;
  const int m = rm - rr_ * M, l = blockIdx.y;
  const bool is_auto = m == l;
  int idx[2];
  bool inL[2], valid[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    idx[h] = ch * 16 + g + 8 * h;
    const int tau = idx[h] - (a.N - 1);
    inL[h] = idx[h] < a.L;
    valid[h] = inL[h] && tau >= a.tau_lo && tau <= a.tau_hi && !(is_auto && a.excl0 && tau == 0);
  }
  // node values -> A fragments (element e: row h = e & 1, column j = c + 4 (e >> 1))
  constexpr bool F16 = SQNGD_LRT_F16 && Q <= 10;  // the packed split needs 3 Q/2 <= 15 K columns
  uint32_t aEr[4], aEi[4], aOr[4], aOi[4];  // F16: m16n8k16 A fragments (rows g, g+8; K columns 2c.., 2c+8..)
  uint32_t aErh[4], aErl[4], aEih[4], aEil[4], aOrh[4], aOrl[4], aOih[4], aOil[4];  // TF32 3x
  float nm2[2] = {0.f, 0.f};
  float sc[2] = {1.f, 1.f}, isc[2] = {1.f, 1.f};  // per-lag prescale of the FP16 path (1 for TF32)
  if constexpr (F16) {
    // K layout (16 columns): lane c holds k = 2c, 2c+1 (registers 0/1) and 2c+8, 2c+9 (2/3) and
    // owns node pair j = c: (hi_c, lo_c | hi_c, e_c) with e = hi_4, lo_4, hi_4, 0 for c = 0..3;
    // the host B table holds the matching (hi(a_c), hi(a_c) | lo(a_c), ...) rows, so the sum over K
    // is x_hi a_hi + x_lo a_hi + x_hi a_lo for every j < 5.  Each lane loads two node pairs.
    const float2* Rp = a.Rn + (size_t)pr * Q * a.LS;
    const bool own = cq < QH, ext = QH > 4 && cq < 3;
    float2 xv[2], yv[2], x4v[2], y4v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float2 x = make_float2(0.f, 0.f), y = x, x4 = x, y4 = x;
      if (inL[h]) {
        if (own) {
          x = __ldg(Rp + (size_t)cq * a.LS + idx[h]);
          y = __ldg(Rp + (size_t)(Q - 1 - cq) * a.LS + idx[h]);
        }
        if (ext) {
          x4 = __ldg(Rp + (size_t)4 * a.LS + idx[h]);
          y4 = __ldg(Rp + (size_t)(Q - 5) * a.LS + idx[h]);
        }
      }
      nm2[h] = fmaxf(fmaxf(fmaf(x.x, x.x, x.y * x.y), fmaf(y.x, y.x, y.y * y.y)),
                     fmaxf(fmaf(x4.x, x4.x, x4.y * x4.y), fmaf(y4.x, y4.x, y4.y * y4.y)));
      nm2[h] = fmaxf(nm2[h], __shfl_xor_sync(0xffffffffu, nm2[h], 1));
      nm2[h] = fmaxf(nm2[h], __shfl_xor_sync(0xffffffffu, nm2[h], 2));
      xv[h] = x; yv[h] = y; x4v[h] = x4; y4v[h] = y4;
      // Per-lag power-of-two prescale sigma (exact): the node sums |E|, |O| <= 2 max_q |R_q| are
      // brought to <= 8192, inside FP16's range and far above its subnormals whatever ||s|| ||w|| is
      // (unscaled values overflow FP16 once ||s|| ||w|| > ~32K and lose their lo parts
      // for small norms).  The cell epilogue works on sigma A: the cotangent gphi A / |A| is
      // invariant, and the magnitude-based terms take the 1/sigma into their per-lag constants.
      int ex = 0;
      if (nm2[h] > 0.f) {
        const float t = 8192.f / (2.f * sqrtf(nm2[h]));
        ex = (int)((__float_as_uint(t) >> 23) & 0xFFu) - 127;
        ex = ex < -100 ? -100 : (ex > 100 ? 100 : ex);
      }
      sc[h] = __uint_as_float((uint32_t)(127 + ex) << 23);
      isc[h] = __uint_as_float((uint32_t)(127 - ex) << 23);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 x = make_float2(xv[h].x * sc[h], xv[h].y * sc[h]), y = make_float2(yv[h].x * sc[h], yv[h].y * sc[h]);
      const float2 x4 = make_float2(x4v[h].x * sc[h], x4v[h].y * sc[h]);
      const float2 y4 = make_float2(y4v[h].x * sc[h], y4v[h].y * sc[h]);
      const float vc[4] = {x.x + y.x, x.y + y.y, x.x - y.x, x.y - y.y};
      const float v4[4] = {x4.x + y4.x, x4.y + y4.y, x4.x - y4.x, x4.y - y4.y};
      uint32_t* frag[4] = {aEr, aEi, aOr, aOi};
#pragma unroll
      for (int pidx = 0; pidx < 4; ++pidx) {
        const __half hc = __float2half_rn(vc[pidx]);
        const __half lc = __float2half_rn(vc[pidx] - __half2float(hc));
        const __half h4 = __float2half_rn(v4[pidx]);
        const __half l4 = __float2half_rn(v4[pidx] - __half2float(h4));
        const __half e = cq == 1 ? l4 : h4;  // lane 3: x4 = y4 = 0
        frag[pidx][h] = (uint32_t)__half_as_ushort(hc) | ((uint32_t)__half_as_ushort(lc) << 16);
        frag[pidx][2 + h] = (uint32_t)__half_as_ushort(hc) | ((uint32_t)__half_as_ushort(e) << 16);
      }
    }
  } else {
    float Er[4], Ei[4], Or[4], Oi[4];
    const float2* Rp = a.Rn + (size_t)pr * Q * a.LS;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = e & 1, j = cq + 4 * (e >> 1);
      float2 x = make_float2(0.f, 0.f), y = x;
      if (j < QH && inL[h]) {
        x = __ldg(Rp + (size_t)j * a.LS + idx[h]);
        y = __ldg(Rp + (size_t)(Q - 1 - j) * a.LS + idx[h]);
      }
      Er[e] = x.x + y.x; Ei[e] = x.y + y.y; Or[e] = x.x - y.x; Oi[e] = x.y - y.y;
      nm2[h] = fmaxf(nm2[h], fmaxf(fmaf(x.x, x.x, x.y * x.y), fmaf(y.x, y.x, y.y * y.y)));
    }
    split4(Er, aErh, aErl); split4(Ei, aEih, aEil); split4(Or, aOrh, aOrl); split4(Oi, aOih, aOil);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // the quad holds all j of its two lags
    nm2[h] = fmaxf(nm2[h], __shfl_xor_sync(0xffffffffu, nm2[h], 1));
    nm2[h] = fmaxf(nm2[h], __shfl_xor_sync(0xffffffffu, nm2[h], 2));
  }
  const float bp = a.bp;
  const float lb = bp * 1.4426950408889634f;
  float shift[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float wm = HW ? (inL[h] ? __ldg(a.wmax + idx[h]) : 0.f) : 1.f;
    if (LM == 1) shift[h] = sqrtf(nm2[h]) * a.invN * wm + 40.f / bp;
    if (LM == 2) shift[h] = fmaxf(sqrtf(nm2[h]) * a.invN * wm, 1e-30f);
  }
  const int t0 = (int)((long long)a.NT * wp / a.kw), t1 = (int)((long long)a.NT * (wp + 1) / a.kw);
  float* mrow[2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
    mrow[h] = (MAP && a.af_mag && inL[h]) ? a.af_mag + (size_t)pr * a.K * a.mld + idx[h] : nullptr;
  // MAP: per-lag bases of the two bin streams of this lane (bins 2c and K-1-2c), advanced per tile
  bool mok[2];
  float* mb0[2];
  float* mb1[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mok[h] = mrow[h] != nullptr;
    if (!mok[h]) mrow[h] = a.af_mag;  // (a valid base; nothing is stored through it)
    mb0[h] = mrow[h] + (ptrdiff_t)(2 * cq) * a.mld;
    mb1[h] = mrow[h] + (ptrdiff_t)(a.K - 1 - 2 * cq) * a.mld;
  }

  float bl[2], bh[2], S[2];
  int kl[2], kh[2];
  float GEr[4], GEi[4], GOr[4], GOi[4];
  LrArgs la;  // lr_cell reads weights, L, bp only
  la.weights = a.weights; la.L = a.L; la.bp = a.bp;
  const int Kp = a.K / 2;
  const bool odd = (a.K & 1) != 0;
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bl[h] = bh[h] = -1.f;
      kl[h] = kh[h] = 0;
      S[h] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) GEr[i] = GEi[i] = GOr[i] = GOi[i] = 0.f;
    f32x2 S2[2] = {0ull, 0ull};  // packed-path sums (two cells per lane of the pair), folded into S below
    float lbN[2], nlbs[2], qN[2];  // per lag: the prescale's 1/sigma folded into the magnitude terms
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lbN[h] = lb * a.invN * isc[h];
      nlbs[h] = valid[h] ? -lb * shift[h] : -INFINITY;
      qN[h] = valid[h] ? a.invN / shift[h] * isc[h] : 0.f;
    }
    // one 8-pair tile: forward MMAs, 8 cells per thread, adjoint MMAs.  MASKED: the remainder
    // tile of a K/2 that is not a multiple of 8 (pairs >= K/2 are zero padding).
    auto ldB = [&](int t, float4& x0, float4& x1, float4& y0, float4& y1) {
      if constexpr (F16) {
        const uint4 f16 = __ldg(a.tabF16 + (size_t)t * 32 + lane);
        x0 = make_float4(__uint_as_float(f16.x), __uint_as_float(f16.y), __uint_as_float(f16.z),
                         __uint_as_float(f16.w));
        x1 = x0;
      } else {
        const float4* tf = a.tabF + ((size_t)t * 32 + lane) * 2;
        x0 = __ldg(tf); x1 = __ldg(tf + 1);
      }
      const float4* ta = a.tabA + ((size_t)t * 32 + lane) * 2;
      if (GRAD) { y0 = __ldg(ta); y1 = __ldg(ta + 1); }
    };
    auto tile = [&](int t, auto masked_c, float4 fa, float4 fb, float4 ga, float4 gb) {
      constexpr bool MASKED = decltype(masked_c)::value;
      float Per[4] = {0.f, 0.f, 0.f, 0.f}, Pei[4] = {0.f, 0.f, 0.f, 0.f};
      float Por[4] = {0.f, 0.f, 0.f, 0.f}, Poi[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (F16) {
        mma_f16(Per, aEr, __float_as_uint(fa.x), __float_as_uint(fa.y));
        mma_f16(Pei, aEi, __float_as_uint(fa.x), __float_as_uint(fa.y));
        mma_f16(Por, aOr, __float_as_uint(fa.z), __float_as_uint(fa.w));
        mma_f16(Poi, aOi, __float_as_uint(fa.z), __float_as_uint(fa.w));
        (void)fb;
      } else {
        mma3(Per, aErh, aErl, fa);
        mma3(Pei, aEih, aEil, fa);
        mma3(Por, aOrh, aOrl, fb);
        mma3(Poi, aOih, aOil, fb);
      }
      float SGr[4], SGi[4], DGr[4], DGi[4];
      if constexpr (PK && !MASKED) {
        // The same cells as the scalar loop below, two at a time: the D elements (2h, 2h + 1) of lag row h
        // (bins p, p + 1 and K-1-p, K-2-p) form packed pairs; MUFU and the argmax keys stay per cell.
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e0 = 2 * h;
          const int p = 8 * t + 2 * cq;
          const f32x2 per = pk2(Per[e0], Per[e0 + 1]), por = pk2(Por[e0], Por[e0 + 1]);
          const f32x2 pei = pk2(Pei[e0], Pei[e0 + 1]), poi = pk2(Poi[e0], Poi[e0 + 1]);
          const f32x2 x0 = add2(per, por), y0 = add2(pei, poi);  // A0: bins p, p + 1
          const f32x2 x1 = sub2(per, por), y1 = sub2(pei, poi);  // A1: bins K-1-p, K-2-p
          const f32x2 eps = pk2(1e-30f, 1e-30f);
          const f32x2 q0 = fma2(x0, x0, fma2(y0, y0, eps)), q1 = fma2(x1, x1, fma2(y1, y1, eps));
          // keys in the scalar loop's cell order (ties: the lowest bin, as lr_cell's > / >= rules)
          {
            const float c0 = lo2(q0), c1 = lo2(q1), c2 = hi2(q0), c3 = hi2(q1);
            bool u = c0 > bl[h]; bl[h] = u ? c0 : bl[h]; kl[h] = u ? p : kl[h];
            u = c1 >= bh[h]; bh[h] = u ? c1 : bh[h]; kh[h] = u ? a.K - 1 - p : kh[h];
            u = c2 > bl[h]; bl[h] = u ? c2 : bl[h]; kl[h] = u ? p + 1 : kl[h];
            u = c3 >= bh[h]; bh[h] = u ? c3 : bh[h]; kh[h] = u ? a.K - 2 - p : kh[h];
          }
          if constexpr (LM != 0) {
            const f32x2 r0 = pk2(rsqa(lo2(q0)), rsqa(hi2(q0))), r1 = pk2(rsqa(lo2(q1)), rsqa(hi2(q1)));
            const f32x2 m0 = mul2(q0, r0), m1 = mul2(q1, r1);  // |A|
            f32x2 g0, g1, ph0, ph1;                             // gphi, phi
            if constexpr (LM == 1) {
              const f32x2 lbv = pk2(lbN[h], lbN[h]), nlv = pk2(nlbs[h], nlbs[h]);
              const f32x2 z0 = fma2(lbv, m0, nlv), z1 = fma2(lbv, m1, nlv);
              g0 = pk2(ex2a(lo2(z0)), ex2a(hi2(z0)));
              g1 = pk2(ex2a(lo2(z1)), ex2a(hi2(z1)));
              ph0 = g0; ph1 = g1;
            } else {
              const f32x2 qv = pk2(qN[h], qN[h]), bm = pk2(a.bp - 1.f, a.bp - 1.f);
              const f32x2 w0 = mul2(m0, qv), w1 = mul2(m1, qv);
              const f32x2 l0 = mul2(bm, pk2(lg2a(lo2(w0)), lg2a(hi2(w0))));
              const f32x2 l1 = mul2(bm, pk2(lg2a(lo2(w1)), lg2a(hi2(w1))));
              g0 = pk2(ex2a(lo2(l0)), ex2a(hi2(l0)));
              g1 = pk2(ex2a(lo2(l1)), ex2a(hi2(l1)));
              ph0 = mul2(g0, w0); ph1 = mul2(g1, w1);
            }
            S2[h] = add2(S2[h], add2(ph0, ph1));
            if constexpr (GRAD) {
              // SG = gf0 A0 + gf1 A1, DG = gf0 A0 - gf1 A1 (gf = gphi / |A|) per element, on the scalar
              // pipe: the adjoint's A fragments pair the elements (2h, 2h + 2), not this (2h, 2h + 1), and
              // scalar results are placed in fragment order for free, packed ones would need moves
              const f32x2 f0 = mul2(g0, r0), f1 = mul2(g1, r1);
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const float gf0 = i ? hi2(f0) : lo2(f0), gf1 = i ? hi2(f1) : lo2(f1);
                const float a0x = i ? hi2(x0) : lo2(x0), a0y = i ? hi2(y0) : lo2(y0);
                const float a1x = i ? hi2(x1) : lo2(x1), a1y = i ? hi2(y1) : lo2(y1);
                const float tr = gf0 * a0x, ti = gf0 * a0y;
                SGr[e0 + i] = fmaf(gf1, a1x, tr); SGi[e0 + i] = fmaf(gf1, a1y, ti);
                DGr[e0 + i] = fmaf(-gf1, a1x, tr); DGi[e0 + i] = fmaf(-gf1, a1y, ti);
              }
            }
          }
        }
      } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // D element e: row h = e >> 1, pair p = 8t + 2c + (e & 1)
        const int h = e >> 1;
        const int p = 8 * t + 2 * cq + (e & 1);
        const float2 A0 = make_float2(Per[e] + Por[e], Pei[e] + Poi[e]);
        const float2 A1 = make_float2(Per[e] - Por[e], Pei[e] - Poi[e]);
        // map addresses (MAP only): bin p = 8t + 2c + (e & 1) and bin K-1-p of this lag row
        const ptrdiff_t mo = (ptrdiff_t)8 * t * a.mld + ((e & 1) ? a.mld : 0);
        float* mc0 = mb0[h] + mo;
        float* mc1 = mb1[h] - mo;
        float gf0, gf1;  // cotangent factors: G = gf A
        if (!MASKED) {
          gf0 = lr_cell<LM, HW, GRAD, false, true>(A0, p, la, idx[h], valid[h], lbN[h], nlbs[h], qN[h], bl[h], kl[h],
                                                   S[h], mc0, MAP && mok[h], isc[h]).x;
          gf1 = lr_cell<LM, HW, GRAD, true, true>(A1, a.K - 1 - p, la, idx[h], valid[h], lbN[h], nlbs[h], qN[h],
                                                  bh[h], kh[h], S[h], mc1, MAP && mok[h], isc[h]).x;
        } else {
          const bool pv = p < Kp;
          const bool v0 = valid[h] && pv;
          float b0 = bl[h], b1 = bh[h];
          int k0 = kl[h], k1 = kh[h];
          gf0 = lr_cell<LM, HW, GRAD, false, true>(A0, pv ? p : 0, la, idx[h], v0, lbN[h], v0 ? nlbs[h] : -INFINITY,
                                                   v0 ? qN[h] : 0.f, b0, k0, S[h], mc0, MAP && mok[h] && pv, isc[h]).x;
          gf1 = lr_cell<LM, HW, GRAD, true, true>(A1, pv ? a.K - 1 - p : 0, la, idx[h], v0, lbN[h],
                                                  v0 ? nlbs[h] : -INFINITY, v0 ? qN[h] : 0.f, b1, k1, S[h],
                                                  mc1, MAP && mok[h] && pv, isc[h]).x;
          if (pv) { bl[h] = b0; kl[h] = k0; bh[h] = b1; kh[h] = k1; }
          if (!v0) gf0 = gf1 = 0.f;
        }
        if (GRAD) {  // SG = gf0 A0 + gf1 A1, DG = gf0 A0 - gf1 A1
          const float tr = gf0 * A0.x, ti = gf0 * A0.y;
          SGr[e] = fmaf(gf1, A1.x, tr); SGi[e] = fmaf(gf1, A1.y, ti);
          DGr[e] = fmaf(-gf1, A1.x, tr); DGi[e] = fmaf(-gf1, A1.y, ti);
        } else {
          SGr[e] = SGi[e] = DGr[e] = DGi[e] = 0.f;
        }
      }
      }
      if (GRAD && PK && !MASKED) {  // the same split, its subtractions packed
        uint32_t hh[4], ll[4];
        split4_pk(SGr, hh, ll); mma3(GEr, hh, ll, ga);
        split4_pk(SGi, hh, ll); mma3(GEi, hh, ll, ga);
        split4_pk(DGr, hh, ll); mma3(GOr, hh, ll, gb);
        split4_pk(DGi, hh, ll); mma3(GOi, hh, ll, gb);
      } else if (GRAD) {
        // D order (g,2c) (g,2c+1) (g+8,2c) (g+8,2c+1) -> A order (g,c) (g+8,c) (g,c+4) (g+8,c+4)
        const float sr[4] = {SGr[0], SGr[2], SGr[1], SGr[3]}, si[4] = {SGi[0], SGi[2], SGi[1], SGi[3]};
        const float dr[4] = {DGr[0], DGr[2], DGr[1], DGr[3]}, di[4] = {DGi[0], DGi[2], DGi[1], DGi[3]};
        uint32_t hh[4], ll[4];
        split4(sr, hh, ll); mma3(GEr, hh, ll, ga);
        split4(si, hh, ll); mma3(GEi, hh, ll, ga);
        split4(dr, hh, ll); mma3(GOr, hh, ll, gb);
        split4(di, hh, ll); mma3(GOi, hh, ll, gb);
      }
    };
    const int tf_end = t1 < a.NTF ? t1 : a.NTF;
    float4 nfa = make_float4(0.f, 0.f, 0.f, 0.f), nfb = nfa, nga = nfa, ngb = nfa;
    if (t0 < tf_end) ldB(t0, nfa, nfb, nga, ngb);
#pragma unroll kLrtUnroll
    for (int t = t0; t < tf_end; ++t) {  // B fragments of the next tile are loaded one tile ahead
      const float4 fa = nfa, fb = nfb, ga = nga, gb = ngb;
      // forward-only: issued before the tile (its latency hides behind the tile; A/B-measured 46.4 ->
      // 43.3 us at C3); with the adjoint the registers are short and after the tile measured faster
      if (!GRAD || SQNGD_LRT_PREFETCH) {
        if (t + 1 < tf_end) ldB(t + 1, nfa, nfb, nga, ngb);
        tile(t, std::integral_constant<bool, false>{}, fa, fb, ga, gb);
      } else {
        tile(t, std::integral_constant<bool, false>{}, fa, fb, ga, gb);
        if (t + 1 < tf_end) ldB(t + 1, nfa, nfb, nga, ngb);
      }
    }
    if constexpr (PK && LM != 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) S[h] += lo2(S2[h]) + hi2(S2[h]);
    }
    if (t1 > a.NTF && t0 <= a.NTF) {
      float4 fa, fb, ga = make_float4(0.f, 0.f, 0.f, 0.f), gb = ga;
      ldB(a.NTF, fa, fb, ga, gb);
      tile(a.NTF, std::integral_constant<bool, true>{}, fa, fb, ga, gb);
    }
    if (odd && wp == a.kw - 1) {
      // middle bin f = grid centre (beta = 0) on the CUDA cores: At = sum_j alpha_j E_j, summed over the
      // quad's j columns; every lane of the quad evaluates the cell (G is needed in all of them), the
      // sum and the key are counted by lane c = 0 only.
      float2 Am[2];
      if constexpr (F16) {  // one extra MMA pair: the middle-bin coefficients in B column 0 (held by the c = 0 lanes)
        const uint2 bm = __ldg(a.tabM16 + lane);
        float Mr[4] = {0.f, 0.f, 0.f, 0.f}, Mi[4] = {0.f, 0.f, 0.f, 0.f};
        mma_f16(Mr, aEr, bm.x, bm.y);
        mma_f16(Mi, aEi, bm.x, bm.y);
        const int src = lane & ~3;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          Am[h] = make_float2(__shfl_sync(0xffffffffu, Mr[2 * h], src), __shfl_sync(0xffffffffu, Mi[2 * h], src));
      } else {
      const float am0 = cq < QH ? __ldg(a.coefm + cq) : 0.f, am1 = cq + 4 < QH ? __ldg(a.coefm + cq + 4) : 0.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float e0r = __uint_as_float(aErh[h]), e0i = __uint_as_float(aEih[h]);  // hi holds x itself
        const float e1r = __uint_as_float(aErh[2 + h]), e1i = __uint_as_float(aEih[2 + h]);
        float xr = fmaf(am0, e0r, am1 * e1r), xi = fmaf(am0, e0i, am1 * e1i);
        xr += __shfl_xor_sync(0xffffffffu, xr, 1);
        xi += __shfl_xor_sync(0xffffffffu, xi, 1);
        xr += __shfl_xor_sync(0xffffffffu, xr, 2);
        xi += __shfl_xor_sync(0xffffffffu, xi, 2);
        Am[h] = make_float2(xr, xi);
      }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float Sm = 0.f, bm = bl[h];
        int km = kl[h];
        const float2 Gm = lr_cell<LM, HW, GRAD, false>(Am[h], Kp, la, idx[h], valid[h], lbN[h], nlbs[h], qN[h], bm, km, Sm,
                                                       mrow[h] + (ptrdiff_t)Kp * a.mld, MAP && mok[h] && cq == 0, isc[h]);
        if (cq == 0) { S[h] += Sm; bl[h] = bm; kl[h] = km; }
        if (GRAD) {
#pragma unroll
          for (int i = 2 * h; i < 2 * h + 2; ++i) {  // D elements of row h: j = 2c + (i & 1)
            const int j = 2 * cq + (i & 1);
            const float aj = j < QH ? __ldg(a.coefm + j) : 0.f;
            GEr[i] = fmaf(aj, Gm.x, GEr[i]);
            GEi[i] = fmaf(aj, Gm.y, GEi[i]);
          }
        }
      }
    }
    if (LM == 0) break;
    bool bad = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float vb = sqrtf(fmaxf(fmaxf(bl[h], bh[h]), 0.f)) * isc[h] * a.invN;
      const bool bd = valid[h] && (LM == 1 ? lb * (vb - shift[h]) > 96.f
                                           : (vb > shift[h] && (bp * log2f(vb / shift[h])) > 96.f));
      bad |= bd;
      if (bd) shift[h] = vb;
    }
    if (!__any_sync(0xffffffffu, bad) || pass == 1) break;
    // lanes of a quad share rows: keep their shifts identical
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      shift[h] = fmaxf(shift[h], __shfl_xor_sync(0xffffffffu, shift[h], 1));
      shift[h] = fmaxf(shift[h], __shfl_xor_sync(0xffffffffu, shift[h], 2));
    }
    mok[0] = mok[1] = false;  // (the map holds the first pass)
  }

  // ---- lane record: key over both rows, per-row shift / sum, cotangent fragments
  unsigned long long key = 0ull;
  // SQNGD_FLAG_TIE inside the unit (forward modes only: the loss+gradient kernel keeps its code; its
  // evaluations flag ties between units, k_lr_finish): 1 + the largest value at which two cells tie
  constexpr bool TT = !GRAD;
  uint32_t tv = 0u;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float best = bl[h];
    int bk = kl[h];
    const bool eq = bh[h] == best;  // the lag's two bin streams (below / above the grid centre) tie
    if (bh[h] > best) { best = bh[h]; bk = kh[h]; }
    best *= isc[h] * isc[h];  // exact: sigma is a power of two
    const uint32_t cell = ((uint32_t)((m * M + l) * a.L + idx[h])) * (uint32_t)a.K + (uint32_t)bk;
    const unsigned long long kk = (valid[h] && best >= 0.f) ? pack_key(best, cell) : 0ull;
    if (TT && kk && (eq || (key && (kk >> 32) == (key >> 32)))) tv = max(tv, (uint32_t)(kk >> 32) + 1u);
    key = kk > key ? kk : key;
  }
  if (a.kw > 1) {
    float* rec = rs + (size_t)wp * NR * 32 + lane;
    rec[0] = __uint_as_float((uint32_t)(key >> 32));
    rec[32] = __uint_as_float((uint32_t)key);
    rec[64] = shift[0]; rec[96] = shift[1];
    rec[128] = S[0]; rec[160] = S[1];
    if (GRAD) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        rec[(6 + i) * 32] = GEr[i];
        rec[(10 + i) * 32] = GEi[i];
        rec[(14 + i) * 32] = GOr[i];
        rec[(18 + i) * 32] = GOi[i];
      }
    }
    __syncthreads();
    if (wp != 0) return;
    for (int w = 1; w < a.kw; ++w) {
      const float* o = rs + (size_t)w * NR * 32 + lane;
      const unsigned long long ko =
          ((unsigned long long)__float_as_uint(o[0]) << 32) | (unsigned long long)__float_as_uint(o[32]);
      key = ko > key ? ko : key;
      if (LM != 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float so = o[64 + 32 * h];
          const float mx = fmaxf(shift[h], so);
          float fS0 = 1.f, fG0 = 1.f, fS1 = 1.f, fG1 = 1.f;
          if (valid[h] && so != shift[h]) {  // only after a redo
            lr_rescale<LM>(shift[h], mx, lb, bp, fS0, fG0);
            lr_rescale<LM>(so, mx, lb, bp, fS1, fG1);
          }
          S[h] = S[h] * fS0 + o[128 + 32 * h] * fS1;
          if (GRAD) {
#pragma unroll
            for (int i = 2 * h; i < 2 * h + 2; ++i) {  // D elements of row h
              GEr[i] = GEr[i] * fG0 + o[(6 + i) * 32] * fG1;
              GEi[i] = GEi[i] * fG0 + o[(10 + i) * 32] * fG1;
              GOr[i] = GOr[i] * fG0 + o[(14 + i) * 32] * fG1;
              GOi[i] = GOi[i] * fG0 + o[(18 + i) * 32] * fG1;
            }
          }
          shift[h] = mx;
        }
      }
    }
  }

  // ---- unit reduction (warp 0)
  if constexpr (TT) {
    key = warp_key_max_tie(key, tv);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
      key = y > key ? y : key;
    }
  }
  float mw = 0.f, fS[2] = {0.f, 0.f}, fG[2] = {0.f, 0.f};
  if (LM != 0) {
    mw = fmaxf(valid[0] ? shift[0] : 0.f, valid[1] ? shift[1] : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (valid[h]) lr_rescale<LM>(shift[h], mw, lb, bp, fS[h], fG[h]);
  }
  // every lane of a quad holds the same row sums only for its own pairs: sum all lanes
  float Su = S[0] * fS[0] + S[1] * fS[1];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Su += __shfl_xor_sync(0xffffffffu, Su, o);
  if (GRAD) {
    float2* gp = a.Gn + (size_t)pr * Q * a.LS;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // D element i: row h = i >> 1, j = 2c + (i & 1)
      const int h = i >> 1, j = 2 * cq + (i & 1);
      if (j < QH && inL[h]) {
        const float f = fG[h];
        gp[(size_t)j * a.LS + idx[h]] = make_float2((GEr[i] + GOr[i]) * f, (GEi[i] + GOi[i]) * f);
        gp[(size_t)(Q - 1 - j) * a.LS + idx[h]] = make_float2((GEr[i] - GOr[i]) * f, (GEi[i] - GOi[i]) * f);
      }
    }
  }
  if (lane == 0) {
    a.part.key[2 * (size_t)u] = is_auto ? key : 0ull;
    a.part.key[2 * (size_t)u + 1] = is_auto ? 0ull : key;
    a.part.m[u] = mw;
    a.part.S[u] = Su;
    const int r = rr_;
    if (key) atomicMax(is_auto ? &a.lred[r].key_a : &a.lred[r].key_c, key);
    if (TT && tv) atomicMax(is_auto ? &a.lred[r].tie_a : &a.lred[r].tie_c, tv);
    if (LM != 0 && mw > 0.f) atomicMax(&a.lred[r].mbits, __float_as_uint(mw));
  }
}

// Per restart: the global shift m (LrRed), S = sum_u S_u (m_u -> m), the reduction record
// and the metrics (a6).  One block per restart, fixed order (deterministic).
__global__ void __launch_bounds__(1024) k_lr_finish(int GPR, int g_lo, int g_hi, int mode, double bp, Part part,
                                                    const LrRed* __restrict__ lred, Red* red, MetricsArgs ma,
                                                    int* status) {
  SQ_PDL_WAIT();
  __shared__ double shd[32];
  const int r = blockIdx.x;
  const float mf = __uint_as_float(lred[r].mbits);
  const float lb = (float)(bp * 1.4426950408889634);
  double S = 0.0;
  if (mode != 0 && mf > 0.f) {
    const float* Sp = part.S + (size_t)r * GPR;
    const float* mp = part.m + (size_t)r * GPR;
    const int glo = max(0, g_lo - r * GPR), ghi = min(GPR, g_hi - r * GPR);  // this rank's units
#pragma unroll 4
    for (int g = glo + threadIdx.x; g < ghi; g += blockDim.x) {
      const float Sg = __ldcg(Sp + g), mg = __ldcg(mp + g);
      float fS = 0.f, fG;
      if (mode == 1) lr_rescale<1>(mg, mf, lb, (float)bp, fS, fG);
      else lr_rescale<2>(mg, mf, lb, (float)bp, fS, fG);
      S += (Sg > 0.f && mg > 0.f) ? (double)Sg * fS : 0.0;
    }
  }
  auto dsum = [](double x, double y) { return x + y; };
  S = block_reduce(S, dsum, shd);
  const bool want_met = ma.out || ma.loss_hist || ma.p_out;
  const bool scan = want_met && ma.tie_scan;
  // SQNGD_FLAG_TIE between units: the highest-index unit keys (only when a metrics record is written)
  unsigned long long ah = 0ull, ch = 0ull;
  if (scan) {
    __shared__ unsigned long long shk[32];
    const unsigned long long* kp = part.key + 2 * (size_t)r * GPR;
    const int glo = max(0, g_lo - r * GPR), ghi = min(GPR, g_hi - r * GPR);
    for (int g = glo + threadIdx.x; g < ghi; g += blockDim.x) {
      ah = max(ah, key_hi_index(__ldcg(kp + 2 * g)));
      ch = max(ch, key_hi_index(__ldcg(kp + 2 * g + 1)));
    }
    auto umax = [](unsigned long long x, unsigned long long y) { return x > y ? x : y; };
    ah = block_reduce(ah, umax, shk);
    ch = block_reduce(ch, umax, shk);
  }
  if (threadIdx.x == 0) {
    const LrRed lr = lred[r];
    red[r].m = mf > 0.f ? (double)mf : -INFINITY;
    red[r].S = S;
    red[r].key_a = lr.key_a;
    red[r].key_c = lr.key_c;
    red[r].tie = (scan && (key_tied(lr.key_a, ah, lr.tie_a) || key_tied(lr.key_c, ch, lr.tie_c) ||
                               (lr.key_a && (lr.key_a >> 32) == (lr.key_c >> 32)))) ? 1u : 0u;
  }
  __syncthreads();
  if (threadIdx.x < 32 && want_met) metrics_warp(ma, r, status);
}

struct AdjGArgs {
  int M, N, Q, LS, nch, csh, units, mode;  // csh: log2 of the k_lr unit's lag chunk (5 or 4)
  int row_lo, row_hi;    // this rank's (restart, transmit channel) rows; other rows contribute zeros
  int u0;                // k_adj_gc: first CTA unit of the shard
  int lsplit;            // k_adj_gc: CTAs per node, each summing M / lsplit of the l (its own partial slot)
  float bp;
  const float2* Gn;      // node cotangents (unit-scaled)
  const float* um;       // per k_lr unit: its shift (part.m)
  const LrRed* lred;     // per restart: the global shift
  const float2* Xc;      // [R][M][Q][P] node spectra X~ (Step A)
  const float2* H;       // [R][M][P] filter spectra / P (Step B)
  float2* out;           // Step A: [units][P] spectral partials
  const float2* Vt;      // [Q][N] node modulation (Step B)
  float2* tslot;         // [R M Q][NS] time-domain node partials
  int NS;
};

// Step-A node adjoint correlations, one transform per unit ((r M + l) M + m) Q + q:
//   out = X~_{m,q} . conj(FFT_P(G^_{ml,q} placed at (-tau) mod P))   (rescaled to the restart's shift);
// the combine sums the M Q slots of filter row (r, l).  Units of rows (r, m) outside this rank's shard
// write zero slots (multi-GPU, the all-reduce adds the other ranks' rows).
template <class PL, int G, int MINB>
__global__ void __launch_bounds__(PL::T* G, MINB) k_adj_g(const AdjGArgs a, const float2* __restrict__ ftw) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int uu = u < a.units ? u : a.units - 1;
  const int M = a.M, Q = a.Q, N = a.N;
  const int q = uu % Q;
  const int rest = uu / Q;
  const int m = rest % M;
  const int rl = rest / M;
  const int l = rl % M;
  const int r = rl / M;
  const int row = r * M + m;
  if (row < a.row_lo || row >= a.row_hi) {  // (uniform over the group)
    if (u < a.units) {
      float2* out = a.out + (size_t)uu * P;
#pragma unroll
      for (int i = 0; i < E; ++i) out[t + i * T] = make_float2(0.f, 0.f);
    }
    return;
  }
  const int pr = row * M + l;
  const float2* Gp = a.Gn + ((size_t)pr * Q + q) * a.LS;
  const float* ump = a.um + (size_t)pr * a.nch;
  const float mf = __uint_as_float(a.lred[r].mbits);
  const float lb = a.bp * 1.4426950408889634f;
  float2 v[E];
  float mu[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {  // all loads first (the rescale below would otherwise wait on each)
    const int j = t + i * T;
    const bool in = j < N || j > P - N;
    const int idx = in ? lag_of(j, N, P) + N - 1 : 0;
    mu[i] = __ldg(ump + (idx >> a.csh));
    v[i] = __ldg(Gp + idx);
  }
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = t + i * T;
    const bool in = j < N || j > P - N;
    float fS, fG;
    if (a.mode == 1) lr_rescale<1>(mu[i], mf, lb, a.bp, fS, fG);
    else lr_rescale<2>(mu[i], mf, lb, a.bp, fS, fG);
    fG = (in && mu[i] > 0.f && mf > 0.f) ? fG : 0.f;
    v[i] = make_float2(v[i].x * fG, v[i].y * fG);
  }
  float2 hx[E];  // the spectrum the transform is multiplied with, fetched while the FFT runs (the
                 // output stores below would otherwise serialize one load round trip per element)
  {
    const float2* HX = a.Xc + ((size_t)row * Q + q) * P;
#pragma unroll
    for (int i = 0; i < E; ++i) hx[i] = __ldg(HX + t + i * T);
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);
  if (u >= a.units) return;
  float2* out = a.out + (size_t)uu * P;
#pragma unroll
  for (int i = 0; i < E; ++i) out[t + i * T] = cmulc(hx[i], v[i]);
}

// Step-B node adjoints with the sum over l inside the CTA: NG groups of one CTA split l and their
// accumulators are summed in shared memory in group order (deterministic).  CTA u = node * lsplit + h,
// node = (r M + m) Q + q (u0 + blockIdx.x: this rank's rows); CTA h of a node takes the l in
// [h M / lsplit, (h + 1) M / lsplit) (the IFFT is linear, so the combine adds the lsplit partials):
//   e_h = IFFT_P(sum_l FFT(G^_{ml,q}) H_l),   tslot[u][n] = e_h(n) conj(V_q(n)).
template <class PL, int NG>
__global__ void __launch_bounds__(PL::T* NG) k_adj_gc(const AdjGArgs a, const float2* __restrict__ ftw) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int M = a.M, Q = a.Q, N = a.N;
  const int u = a.u0 + blockIdx.x;
  const int node = u / a.lsplit, h = u - node * a.lsplit;
  const int q = node % Q, rm = node / Q;
  const int r = rm / M;
  const int l_lo = (int)((long long)M * h / a.lsplit), l_hi = (int)((long long)M * (h + 1) / a.lsplit);
  const float mf = __uint_as_float(a.lred[r].mbits);
  const float lb = a.bp * 1.4426950408889634f;
  float2 acc[E];
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
  int par = 0;
  for (int l = l_lo + grp; l < l_hi; l += NG) {
    const int pr = rm * M + l;
    const float2* Gp = a.Gn + ((size_t)pr * Q + q) * a.LS;
    const float* ump = a.um + (size_t)pr * a.nch;
    float2 v[E];
    float mu[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {  // all loads first (the rescale below would otherwise wait on each)
      const int j = t + i * T;
      const bool in = j < N || j > P - N;
      const int idx = in ? lag_of(j, N, P) + N - 1 : 0;
      mu[i] = __ldg(ump + (idx >> a.csh));
      v[i] = __ldg(Gp + idx);
    }
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int j = t + i * T;
      const bool in = j < N || j > P - N;
      float fS, fG;
      if (a.mode == 1) lr_rescale<1>(mu[i], mf, lb, a.bp, fS, fG);
      else lr_rescale<2>(mu[i], mf, lb, a.bp, fS, fG);
      fG = (in && mu[i] > 0.f && mf > 0.f) ? fG : 0.f;
      v[i] = make_float2(v[i].x * fG, v[i].y * fG);
    }
    float2 hx[E];  // the spectrum the transform is multiplied with, fetched while the FFT runs
    const float2* HX = a.H + ((size_t)r * M + l) * P;
#pragma unroll
    for (int i = 0; i < E; ++i) hx[i] = __ldg(HX + t + i * T);
    fft<PL, -1>(v, ftw, xbuf, t, par, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmul(v[i], hx[i]));
  }
  // fixed-order sum of the groups' accumulators (the exchange buffers are free now)
  __syncthreads();
  if (grp != 0) {
#pragma unroll
    for (int i = 0; i < E; ++i) xbuf[t + i * T] = acc[i];
  }
  __syncthreads();
  if (grp != 0) return;
  for (int g = 1; g < NG; ++g) {
    const float2* ob = reinterpret_cast<float2*>(smem_raw) + g * (FftSmem<PL>::TOTAL);
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], ob[t + i * T]);
  }
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i].y = -acc[i].y;
  fft<PL, -1>(acc, ftw, xbuf, t, par, sync);  // acc = conj(e)
  const float2* vr = a.Vt + (size_t)q * N;
  float2* o = a.tslot + (size_t)u * a.NS;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    if (n < N) {
      const float2 z = cmul(acc[i], __ldg(vr + n));
      o[n] = make_float2(z.x, -z.y);  // e conj(V_q)
    }
  }
}

}  // namespace sq
