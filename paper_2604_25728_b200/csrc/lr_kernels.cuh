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
// the FFT path at the Q nodes only (k_adj_g, k_lrB_tail).  Transforms per
// evaluation drop from O(M^2 K) to O(M^2 Q).
//
// Symmetry: the uniform grid and the Chebyshev nodes are both symmetric about the
// grid centre, so l_q(f_{K-1-k}) = l_{Q-1-q}(f_k).  With E_q = R_q + R_{Q-1-q},
// O_q = R_q - R_{Q-1-q}, alpha_q = (l_q + l_{Q-1-q})/2, beta_q = (l_q - l_{Q-1-q})/2
// (q < Q/2):  At(f_k) = Pe + Po,  At(f_{K-1-k}) = Pe - Po,  Pe = sum alpha E,
// Po = sum beta O -- one bin pair costs Q complex-by-real FMAs each way instead of 2Q.
#pragma once
#include <stdint.h>

#include "af_kernels.cuh"

namespace sq {

// Node AFs for every unit (r, m, l, q): R_{ml,q}(tau) = IFFT_P(X~_{m,q} conj(H_l))[(-tau) mod P]
// (Eq. 36, Q1), stored at Rn[((r M + m) M + l) Q + q][tau + N - 1].
template <class PL, int G, int MINB>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_node(int units, int M, int Q, int N, int LS, const float2* __restrict__ Xc, const float2* __restrict__ H,
           const float2* __restrict__ ftw, float2* __restrict__ Rn) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int uu = u < units ? u : units - 1;
  const int q = uu % Q, pr = uu / Q;  // pr = (r M + m) M + l
  const int l = pr % M, rm = pr / M, r = rm / M;
  const float2* X = Xc + ((size_t)rm * Q + q) * P;
  const float2* Hl = H + ((size_t)r * M + l) * P;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = cmulc(__ldg(Hl + t + i * T), __ldg(X + t + i * T));  // conj(X conj(H))
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);  // v = conj(r)
  if (u >= units) return;
  float2* out = Rn + (size_t)uu * LS + (N - 1);
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = t + i * T;
    if (j < N || j > P - N) out[lag_of(j, N, P)] = make_float2(v[i].x, -v[i].y);
  }
}

struct LrArgs {
  int R, M, N, L, K, nch, kparts, LS, QS;  // QS: coefficient row stride (Q rounded up to 4)
  int tau_lo, tau_hi, excl0;
  float bp, invN;
  const float* weights;  // [K][L] or nullptr
  const float* wmax;     // [L] max_k weights (HW only)
  const float* coef;     // [(K/2) + 1][QS]: alpha_0..alpha_{Q/2-1}, beta_0..beta_{Q/2-1}; last row: middle bin
  const float2* Rn;      // [R M M][Q][LS] node AFs
  float2* Gn;            // [kparts][R M M][Q][LS] node cotangents (unit-scaled)
  float* af_mag;         // [R][M][M][K][L] or nullptr (forward only)
  Part part;             // unit slots, u = ((pair nch) + chunk) kparts + kpart
};

// One Doppler cell of the fused epilogue (a5 / a7): key tracking, surrogate term, cotangent.
// LM: 0 MAX (keys only), 1 LSE, 2 PNORM.  Returns G~ (unnormalised: gphi w At / |At|).
template <int LM, bool HW, bool GRAD, bool GE_RULE>
__device__ __forceinline__ float2 lr_cell(float2 A, int k, const LrArgs& a, int idx, bool valid, float lbN, float nlbs,
                                          float qN, float& best, int& bk, float& S, float* mrow) {
  const float a2 = fmaf(A.x, A.x, A.y * A.y);
  float wt = 1.f, kv = a2;
  if (HW) {
    wt = valid ? __ldg(a.weights + (size_t)k * a.L + idx) : 0.f;
    kv = wt > 0.f ? a2 * wt * wt : -1.f;
  }
  const bool upd = GE_RULE ? (kv >= best) : (kv > best);
  best = upd ? kv : best;
  bk = upd ? k : bk;
  if (LM == 0) {
    if (mrow) mrow[(size_t)k * a.L] = sqrtf(a2);
    return make_float2(0.f, 0.f);
  }
  const float rsq = rsqa(fmaxf(a2, 1e-30f));
  const float mag = a2 * rsq;
  if (mrow) mrow[(size_t)k * a.L] = mag;
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
  return make_float2(A.x * gf, A.y * gf);
}

// Fused Doppler contraction + cell epilogue + adjoint contraction.  One warp per unit
// (pair (r, m, l), 32 consecutive lags, one range of bin pairs); a thread owns one lag.
// Each thread accumulates its surrogate sum and cotangents with its own shift (node
// maximum + 40/beta for LSE, so no term overflows); the warp rescales to the unit's
// shift at the end and writes (key, shift, sum) into the unit's slot and the node
// cotangents G^_q(tau) = sum_k l_q(f_k) G~(tau, f_k) into Gn.  A thread whose cells
// exceed its shift by more than 96/(beta log2 e) redoes the unit with the exact maximum.
template <int Q, int LM, bool HW, bool GRAD>
__global__ void __launch_bounds__(128) k_lr(const LrArgs a, int units) {
  constexpr int QH = Q / 2;
  extern __shared__ float4 lr_smem[];
  float* cf = reinterpret_cast<float*>(lr_smem);
  const int Kp = a.K / 2;
  const bool odd = (a.K & 1) != 0;
  const int ncf = (Kp + 1) * a.QS;
  for (int i = threadIdx.x; i < ncf; i += blockDim.x) cf[i] = __ldg(a.coef + i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (u >= units) return;  // warp-uniform
  const int kp = u % a.kparts;
  const int c = (u / a.kparts) % a.nch;
  const int pr = u / (a.kparts * a.nch);
  const int M = a.M;
  const int l = pr % M, m = (pr / M) % M;
  const int idx = c * 32 + lane;
  const int tau = idx - (a.N - 1);
  const bool inL = idx < a.L;
  const bool is_auto = m == l;
  const bool valid = inL && tau >= a.tau_lo && tau <= a.tau_hi && !(is_auto && a.excl0 && tau == 0);

  float2 Ev[QH], Ov[QH];
  float nm2 = 0.f;
  {
    const float2* Rp = a.Rn + (size_t)pr * Q * a.LS + (inL ? idx : 0);
#pragma unroll
    for (int j = 0; j < QH; ++j) {
      const float2 x = inL ? __ldg(Rp + (size_t)j * a.LS) : make_float2(0.f, 0.f);
      const float2 y = inL ? __ldg(Rp + (size_t)(Q - 1 - j) * a.LS) : make_float2(0.f, 0.f);
      Ev[j] = cadd(x, y);
      Ov[j] = csub(x, y);
      nm2 = fmaxf(nm2, fmaxf(fmaf(x.x, x.x, x.y * x.y), fmaf(y.x, y.x, y.y * y.y)));
    }
  }
  const int p0 = (int)((long long)Kp * kp / a.kparts), p1 = (int)((long long)Kp * (kp + 1) / a.kparts);
  const bool do_mid = odd && kp == a.kparts - 1;
  const float bp = a.bp;
  const float lb = bp * 1.4426950408889634f;
  const float wm = HW ? (inL ? __ldg(a.wmax + idx) : 0.f) : 1.f;
  float shift = 0.f;
  if (LM == 1) shift = sqrtf(nm2) * a.invN * wm + 40.f / bp;
  if (LM == 2) shift = fmaxf(sqrtf(nm2) * a.invN * wm, 1e-30f);
  float* mrow = (!GRAD && a.af_mag && inL) ? a.af_mag + (size_t)pr * a.K * a.L + idx : nullptr;

  float bl, bh, bmid, S;
  int kl, kh, kmid;
  float2 GE[QH], GO[QH];
  for (int pass = 0; pass < 2; ++pass) {
    bl = bh = bmid = -1.f;
    kl = kh = kmid = 0;
    S = 0.f;
#pragma unroll
    for (int j = 0; j < QH; ++j) GE[j] = GO[j] = make_float2(0.f, 0.f);
    const float lbN = lb * a.invN;
    const float nlbs = valid ? -lb * shift : -INFINITY;
    const float qN = valid ? a.invN / shift : 0.f;
#pragma unroll 1
    for (int p = p0; p < p1; ++p) {
      const float4* cp = reinterpret_cast<const float4*>(cf + p * a.QS);
      float co[(Q + 3) & ~3];
#pragma unroll
      for (int i = 0; i < (Q + 3) / 4; ++i) {
        const float4 t4 = cp[i];
        co[4 * i] = t4.x; co[4 * i + 1] = t4.y; co[4 * i + 2] = t4.z; co[4 * i + 3] = t4.w;
      }
      float2 Pe = make_float2(0.f, 0.f), Po = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < QH; ++j) {
        Pe.x = fmaf(co[j], Ev[j].x, Pe.x);
        Pe.y = fmaf(co[j], Ev[j].y, Pe.y);
        Po.x = fmaf(co[QH + j], Ov[j].x, Po.x);
        Po.y = fmaf(co[QH + j], Ov[j].y, Po.y);
      }
      const float2 G0 = lr_cell<LM, HW, GRAD, false>(cadd(Pe, Po), p, a, idx, valid, lbN, nlbs, qN, bl, kl, S, mrow);
      const float2 G1 =
          lr_cell<LM, HW, GRAD, true>(csub(Pe, Po), a.K - 1 - p, a, idx, valid, lbN, nlbs, qN, bh, kh, S, mrow);
      if (GRAD) {
        const float2 sg = cadd(G0, G1), dg = csub(G0, G1);
#pragma unroll
        for (int j = 0; j < QH; ++j) {
          GE[j].x = fmaf(co[j], sg.x, GE[j].x);
          GE[j].y = fmaf(co[j], sg.y, GE[j].y);
          GO[j].x = fmaf(co[QH + j], dg.x, GO[j].x);
          GO[j].y = fmaf(co[QH + j], dg.y, GO[j].y);
        }
      }
    }
    if (do_mid) {  // f = grid centre: beta = 0
      const float* cm = cf + Kp * a.QS;
      float2 Pe = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < QH; ++j) {
        Pe.x = fmaf(cm[j], Ev[j].x, Pe.x);
        Pe.y = fmaf(cm[j], Ev[j].y, Pe.y);
      }
      const float2 G0 = lr_cell<LM, HW, GRAD, false>(Pe, Kp, a, idx, valid, lbN, nlbs, qN, bmid, kmid, S, mrow);
      if (GRAD) {
#pragma unroll
        for (int j = 0; j < QH; ++j) {
          GE[j].x = fmaf(cm[j], G0.x, GE[j].x);
          GE[j].y = fmaf(cm[j], G0.y, GE[j].y);
        }
      }
    }
    if (LM == 0) break;
    const float b2 = fmaxf(fmaxf(bl, bh), bmid);
    const float vb = sqrtf(fmaxf(b2, 0.f)) * a.invN;
    const bool bad = valid && (LM == 1 ? lb * (vb - shift) > 96.f : (vb > shift && (bp * log2f(vb / shift)) > 96.f));
    if (!__any_sync(0xffffffffu, bad) || pass == 1) break;
    if (bad) shift = vb;
    mrow = nullptr;  // the map was written in the first pass
  }

  // ---- unit reduction: key, shift, sum; node cotangents
  float best = bl;
  int bk = kl;
  if (bmid > best) { best = bmid; bk = kmid; }
  if (bh > best) { best = bh; bk = kh; }
  const uint32_t cell = ((uint32_t)((m * M + l) * a.L + idx)) * (uint32_t)a.K + (uint32_t)bk;
  unsigned long long key = (valid && best >= 0.f) ? pack_key(best, cell) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
    key = y > key ? y : key;
  }
  float mw = 0.f, fS = 0.f, fG = 0.f;
  if (LM == 1) {
    mw = valid ? shift : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    fS = fG = valid ? ex2a(lb * (shift - mw)) : 0.f;
  } else if (LM == 2) {
    mw = valid ? shift : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    const float rt = valid && mw > 0.f ? shift / mw : 0.f;
    fG = rt > 0.f ? ex2a((bp - 1.f) * lg2a(rt)) : 0.f;
    fS = fG * rt;
  }
  float Su = S * fS;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Su += __shfl_xor_sync(0xffffffffu, Su, o);
  if (GRAD && inL) {
    float2* gp = a.Gn + (size_t)kp * ((size_t)a.R * M * M * Q * a.LS) + (size_t)pr * Q * a.LS + idx;
#pragma unroll
    for (int j = 0; j < QH; ++j) {
      gp[(size_t)j * a.LS] = make_float2((GE[j].x + GO[j].x) * fG, (GE[j].y + GO[j].y) * fG);
      gp[(size_t)(Q - 1 - j) * a.LS] = make_float2((GE[j].x - GO[j].x) * fG, (GE[j].y - GO[j].y) * fG);
    }
  }
  if (lane == 0) {
    a.part.key[2 * (size_t)u] = is_auto ? key : 0ull;
    a.part.key[2 * (size_t)u + 1] = is_auto ? 0ull : key;
    a.part.m[u] = mw;
    a.part.S[u] = Su;
  }
}

struct AdjGArgs {
  int M, N, Q, LS, nch, kparts, units;
  size_t gstride;        // Gn stride between k-parts
  const float2* Gn;      // node cotangents
  const float* scale;    // per k_lr unit: rescale to the restart's shift (k_reduce_groups)
  const float2* Xc;      // [R][M][Q][P] node spectra X~ (Step A)
  const float2* H;       // [R][M][P] filter spectra / P (Step B)
  float2* out;           // [units][P] spectral partials
};

// Node adjoint correlations, one transform per unit:
//   G^_{ml,q} = FFT_P(G^ placed at (-tau) mod P) (scaled to the restart's shift), then
//   Step B (WRT 2), unit ((r M + m) Q + q) M + l:  out = G^ . H_l            (sum over l: k_lrB_tail)
//   Step A (WRT 1), unit ((r M + l) M + m) Q + q:  out = X~_{m,q} . conj(G^)  (sum over m, q: combine)
template <class PL, int G, int MINB, int WRT>
__global__ void __launch_bounds__(PL::T* G, MINB) k_adj_g(const AdjGArgs a, const float2* __restrict__ ftw) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int uu = u < a.units ? u : a.units - 1;
  const int M = a.M, Q = a.Q, N = a.N;
  int r, m, l, q;
  if (WRT == 2) {
    l = uu % M;
    const int rest = uu / M;
    q = rest % Q;
    const int rm = rest / Q;
    m = rm % M;
    r = rm / M;
  } else {
    q = uu % Q;
    const int rest = uu / Q;
    m = rest % M;
    const int rl = rest / M;
    l = rl % M;
    r = rl / M;
  }
  const int pr = (r * M + m) * M + l;
  const float2* Gp = a.Gn + ((size_t)pr * Q + q) * a.LS;
  const float* scp = a.scale + (size_t)pr * a.nch * a.kparts;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = t + i * T;
    float2 g = make_float2(0.f, 0.f);
    if (j < N || j > P - N) {
      const int idx = lag_of(j, N, P) + N - 1;
      const float* sc = scp + (idx >> 5) * a.kparts;
      for (int kp = 0; kp < a.kparts; ++kp) {
        const float s = __ldg(sc + kp);
        const float2 x = __ldg(Gp + kp * a.gstride + idx);
        g.x = fmaf(s, x.x, g.x);
        g.y = fmaf(s, x.y, g.y);
      }
    }
    v[i] = g;
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);
  if (u >= a.units) return;
  float2* out = a.out + (size_t)uu * P;
  if (WRT == 2) {
    const float2* Hl = a.H + ((size_t)r * M + l) * P;
#pragma unroll
    for (int i = 0; i < E; ++i) out[t + i * T] = cmul(v[i], __ldg(Hl + t + i * T));
  } else {
    const float2* X = a.Xc + (((size_t)r * M + m) * Q + q) * P;
#pragma unroll
    for (int i = 0; i < E; ++i) out[t + i * T] = cmulc(__ldg(X + t + i * T), v[i]);
  }
}

// Step B node tail, unit (r M + m) Q + q:  e = IFFT_P(sum_l G^_{ml,q} H_l) (fixed order),
// out[u][n] = e(n) conj(V_q(n)) for n < N (row stride NS, even: the combine reads float4 pairs):
// the node's share of dL/ds_m^* before the sum over q.
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_lrB_tail(int units, int M, int Q, int N, int NS, const float2* __restrict__ slots, const float2* __restrict__ Vt,
               const float2* __restrict__ ftw, float2* __restrict__ out) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int uu = u < units ? u : units - 1;
  const int q = uu % Q;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = make_float2(0.f, 0.f);
  for (int l = 0; l < M; ++l) {
    const float2* sp = slots + ((size_t)uu * M + l) * P;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = cadd(v[i], __ldg(sp + t + i * T));
  }
#pragma unroll
  for (int i = 0; i < E; ++i) v[i].y = -v[i].y;
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);  // v = conj(e)
  if (u >= units) return;
  const float2* vr = Vt + (size_t)q * N;
  float2* o = out + (size_t)uu * NS;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    if (n < N) {
      const float2 z = cmul(v[i], __ldg(vr + n));
      o[n] = make_float2(z.x, -z.y);
    }
  }
}

}  // namespace sq
