// Fused AF/CAF forward + adjoint kernels.
//
// A *group* of T = P/E threads owns one evaluation unit at a time and keeps its
// spectra in registers (strided ownership, fft.cuh).
//
//   k_xhat, unit (r, m, k):                        a3
//     x_hat = s_m . e^{j 2 pi n f_k / N}            Eq. 33 (twiddle table built in fp64)
//     X_{m,k} = FFT_P(x_hat_pad)  -> X cache [R][M][K][P] (L2-resident for C1-C4)
//   forward (MODE_FWD), group (r, m, chunk of k):   a4-a5
//     for l: r = IFFT_P(X . conj(H_l)/P)            Eq. 36; A(tau) = r[(-tau) mod P] (Q1)
//            fused epilogue: |A|, ROI mask, packed (value, ~index) max keys for
//            WAPSL / WCPSL (Eqs. 7-9), LSE / p-norm partial sums, optional |A| map.
//   Step B adjoint (MODE_ADJ_B), group (r, m, chunk of k):  a4-a7, a8B
//     per l: r, then G = dL/dA^* (unnormalized: phi * w * A / |A|) in place,
//     G_hat = FFT_P(G), acc += G_hat . H_l/P;  after the l loop e = IFFT_P(acc) and
//     the group adds conj(e^{j 2 pi n f/N}) e[n] into its per-(r, m) partial.
//   Step A adjoint (MODE_ADJ_A), group (r, l, chunk of k), loop (k, m):  a4-a7, a8A
//     r, G, G_hat as above and acc += X . conj(G_hat); at the end of the chunk
//     d = IFFT_P(acc) is the group's dL/dw_l^* partial.
//
// The cotangent needs the LSE / p-norm normalizer of the *whole* loss, so the
// adjoint kernels accumulate with a group-uniform running shift m (online
// rescaling): phi = e^{beta (v - m)} (LSE) or (v / m)^{p-1} (PNORM); the combine
// kernel rescales every group to the global shift, so one pass is exact.
//
// Reductions are deterministic: fixed per-group partial slots, fixed-order
// combine, no floating-point atomics.
#pragma once
#include <stdint.h>

#include "fft.cuh"

namespace sq {

enum { MODE_FWD = 0, MODE_ADJ_A = 1, MODE_ADJ_B = 2 };

struct KP {
  int R, M, N, K, L, P;
  int tau_lo, tau_hi, excl0;
  int loss_mode;  // 0 MAX, 1 LSE, 2 PNORM
  float beta_or_p;
  float invN;
  const float* weights;  // [K][L] or nullptr
  int C, chunk;          // Doppler chunks per (r, a) and bins per chunk
  int g_lo, g_hi;        // groups evaluated by this rank (multi-GPU slice)
  int want_S;            // forward: accumulate surrogate sums
};

struct Part {
  unsigned long long* key;  // [Gtot][2]  (auto, cross)
  float* m;                 // [Gtot] shift of the group's sums
  float* S;                 // [Gtot] sum of phi (LSE: e^{b(v-m)}, PNORM: (v/m)^p)
  float* scale;             // [Gtot] rescale to the restart's global shift (combine)
  float2* g;                // [Gtot][N] adjoint partial (time domain)
};

__device__ __forceinline__ unsigned long long pack_key(float val, uint32_t idx) {
  return ((unsigned long long)__float_as_uint(val) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}

__device__ __forceinline__ unsigned group_mask(int T) {
  return T >= 32 ? 0xffffffffu : (((1u << T) - 1u) << ((threadIdx.x & 31) & ~(T - 1)));
}

// Group-level helpers: T <= 32 -> shuffles inside the group's lanes; T > 32 -> shuffles
// + one smem slot per warp + a group barrier (double-buffered slots).
template <int T>
struct Group {
  GroupSync sync;
  unsigned mask;
  float* red;
  unsigned long long* redk;
  int par;
  int t;

  __device__ __forceinline__ float max_f(float x) {
    constexpr int W = T < 32 ? T : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(mask, x, o));
    if constexpr (T > 32) {
      float* b = red + (par ? 32 : 0);
      par ^= 1;
      if ((t & 31) == 0) b[t >> 5] = x;
      sync();
      x = b[0];
#pragma unroll
      for (int w = 1; w < T / 32; ++w) x = fmaxf(x, b[w]);
    }
    return x;
  }
  __device__ __forceinline__ float sum_f(float x) {  // fixed order: bitwise reproducible
    constexpr int W = T < 32 ? T : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o);
    if constexpr (T > 32) {
      float* b = red + (par ? 32 : 0);
      par ^= 1;
      if ((t & 31) == 0) b[t >> 5] = x;
      sync();
      x = b[0];
#pragma unroll
      for (int w = 1; w < T / 32; ++w) x += b[w];
    }
    return x;
  }
  __device__ __forceinline__ unsigned long long max_u64(unsigned long long x) {
    constexpr int W = T < 32 ? T : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(mask, x, o);
      x = y > x ? y : x;
    }
    if constexpr (T > 32) {
      unsigned long long* b = redk + (par ? 32 : 0);
      par ^= 1;
      if ((t & 31) == 0) b[t >> 5] = x;
      sync();
      x = b[0];
#pragma unroll
      for (int w = 1; w < T / 32; ++w) x = b[w] > x ? b[w] : x;
    }
    return x;
  }
};

// Per-group shared memory (float2 units).
template <class PL, int MODE>
struct GroupSmem {
  static constexpr int XBUF = PL::NP > 1 ? 2 * PL::PADDED : 0;
  static constexpr int GACC = MODE == MODE_ADJ_B ? PL::P / 2 : 0;  // N <= P/2
  static constexpr int RED = 32;                                    // 64 floats (2 x 32)
  static constexpr int REDK = 64;                                   // 64 u64 (2 x 32)
  static constexpr int TOTAL = XBUF + GACC + RED + REDK;
};

// Per-thread ROI bitmasks over its E elements (bit i <-> j = t + i T), weights aside:
// auto maps drop tau = 0 when excl0 (Eq. 8), cross maps keep it (Eq. 9).
template <class PL>
__device__ __forceinline__ void roi_masks(const KP& kp, int t, uint32_t& roi_auto, uint32_t& roi_cross) {
  roi_auto = roi_cross = 0u;
#pragma unroll
  for (int i = 0; i < PL::E; ++i) {
    const int j = t + i * PL::T;
    const int tau = (j < kp.N) ? -j : (j > PL::P - kp.N ? PL::P - j : (1 << 24));
    const bool in = tau >= kp.tau_lo && tau <= kp.tau_hi;
    if (in) roi_cross |= 1u << i;
    if (in && !(kp.excl0 && tau == 0)) roi_auto |= 1u << i;
  }
}

__device__ __forceinline__ int lag_of(int j, int N, int P) { return (j < N) ? -j : P - j; }

// Running max with the oracle's tie rule (lowest lexicographic (m, l, tau, k) index wins).
__device__ __forceinline__ void best_update(float kv, uint32_t idx, float& best, uint32_t& bidx) {
  if (kv > best || (kv == best && idx < bidx)) {
    best = kv;
    bidx = idx;
  }
}

// a3: X_{m,k} = FFT_P(s_m e^{j 2 pi n f_k / N}) for every unit (r, m, k) -> X cache.
template <class PL, int G, int MINB>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_xhat(int units, int M, int N, int K, const float2* __restrict__ s, const float2* __restrict__ dtw,
           const float2* __restrict__ ftw, float2* __restrict__ Xc) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (PL::NP > 1 ? 2 * PL::PADDED : 0);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int uu = u < units ? u : units - 1;
  const int k = uu % K, rm = uu / K;
  const float2* sr = s + (size_t)rm * N;
  const float2* twr = dtw + (size_t)k * N;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    v[i] = n < N ? cmul(__ldg(sr + n), __ldg(twr + n)) : make_float2(0.f, 0.f);
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);
  if (u >= units) return;
  float2* out = Xc + (size_t)u * P;
#pragma unroll
  for (int i = 0; i < E; ++i) out[t + i * T] = v[i];
}

template <class PL, int G, int MINB, int MODE>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_af(const KP kp, const float2* __restrict__ Xc, const float2* __restrict__ Hh,
         const float2* __restrict__ dtw, const float2* __restrict__ ftw, float* __restrict__ af_mag, Part part) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  using GS = GroupSmem<PL, MODE>;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int gg = kp.g_lo + blockIdx.x * G + grp;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * GS::TOTAL;
  float2* xbuf = gsm;
  float2* gacc = gsm + GS::XBUF;

  Group<T> grpops;
  grpops.sync = GroupSync{1 + grp, T, group_mask(T)};
  grpops.mask = grpops.sync.mask;
  grpops.red = reinterpret_cast<float*>(gsm + GS::XBUF + GS::GACC);
  grpops.redk = reinterpret_cast<unsigned long long*>(gsm + GS::XBUF + GS::GACC + GS::RED);
  grpops.par = 0;
  grpops.t = t;

  const bool active = gg < kp.g_hi;
  const int M = kp.M, N = kp.N, K = kp.K;
  const int ra = active ? gg / kp.C : 0, c = active ? gg % kp.C : 0;
  const int r = ra / M, a = ra % M;
  const int k0 = c * kp.chunk;
  const int k1 = active ? min(K, k0 + kp.chunk) : k0;

  int par = 0;
  float best_a = -1.f, best_c = -1.f;  // running max of w^2 |A|^2 (auto, cross) and its cell index
  uint32_t bidx_a = 0xFFFFFFFFu, bidx_c = 0xFFFFFFFFu;
  uint32_t roi_auto, roi_cross;
  roi_masks<PL>(kp, t, roi_auto, roi_cross);
  const bool has_w = kp.weights != nullptr;
  const int mode = kp.loss_mode;
  const float bp = kp.beta_or_p;
  float shift = (mode == 2) ? 0.f : -INFINITY;  // forward: per-thread; adjoint: group-uniform
  float Ssum = 0.f;

  float2 v[E];
  float2 acc[MODE == MODE_FWD ? 1 : E];
  if constexpr (MODE != MODE_FWD) {
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
  }
  if constexpr (MODE == MODE_ADJ_B) {
    for (int n = t; n < N; n += T) gacc[n] = make_float2(0.f, 0.f);
  }

  const int inner = (MODE == MODE_ADJ_A) ? M : 1;
  for (int k = k0; k < k1; ++k) {
    for (int mi = 0; mi < inner; ++mi) {
      const int m = (MODE == MODE_ADJ_A) ? mi : a;
      const float2* Xr = Xc + (((size_t)r * M + m) * K + k) * P;
      if constexpr (MODE == MODE_ADJ_B) {
#pragma unroll
        for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
      }
      const int l_lo = (MODE == MODE_ADJ_A) ? a : 0, l_hi = (MODE == MODE_ADJ_A) ? a + 1 : M;
      for (int l = l_lo; l < l_hi; ++l) {
        const float2* Hl = Hh + ((size_t)r * M + l) * P;
        const bool is_auto = (m == l);
        const uint32_t roi = is_auto ? roi_auto : roi_cross;
        const uint32_t base_idx = (uint32_t)((m * M + l) * kp.L + N - 1);
        const float* wrow = has_w ? kp.weights + (size_t)k * kp.L + N - 1 : nullptr;
        // ---- a4: cross-spectrum + IFFT (Eq. 36); H is stored pre-scaled by 1/P
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = cmulc(__ldg(Xr + t + i * T), __ldg(Hl + t + i * T));
        fft<PL, +1>(v, ftw, xbuf, t, par, grpops.sync);
        // ---- a5: fused cell epilogue (max keys; forward sums / map)
        float lmax2 = -1.f, lbest = -1.f;
        uint32_t lidx = 0xFFFFFFFFu;
        if constexpr (MODE == MODE_FWD) {
          if (af_mag) {
            float* mrow = af_mag + ((((size_t)r * M + m) * M + l) * K + k) * (size_t)kp.L + N - 1;
#pragma unroll
            for (int i = 0; i < E; ++i) {
              const int j = t + i * T;
              if (j < N || j > P - N) mrow[lag_of(j, N, P)] = sqrtf(fmaf(v[i].x, v[i].x, v[i].y * v[i].y));
            }
          }
        }
#pragma unroll
        for (int i = 0; i < E; ++i) {
          if (!((roi >> i) & 1u)) continue;
          float kv = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
          if (has_w) {
            const float wt = __ldg(wrow + lag_of(t + i * T, N, P));
            if (!(wt > 0.f)) continue;
            kv *= wt * wt;
          }
          lmax2 = fmaxf(lmax2, kv);
          if (kv >= lbest) {  // rare after the first few cells: index only on a new max
            const uint32_t idx = (base_idx + (uint32_t)lag_of(t + i * T, N, P)) * (uint32_t)K + (uint32_t)k;
            best_update(kv, idx, lbest, lidx);
          }
          if constexpr (MODE == MODE_FWD) {
            if (kp.want_S) {
              const float vv = sqrtf(kv) * kp.invN;
              if (vv > shift) {  // per-thread online rescale
                if (Ssum > 0.f) Ssum *= (mode == 1) ? __expf(bp * (shift - vv)) : __powf(shift / vv, bp);
                shift = vv;
              }
              Ssum += (mode == 1) ? __expf(bp * (vv - shift)) : (shift > 0.f ? __powf(vv / shift, bp) : 0.f);
            }
          }
        }
        if (lbest >= 0.f) {
          if (is_auto) best_update(lbest, lidx, best_a, bidx_a);
          else best_update(lbest, lidx, best_c, bidx_c);
        }
        if constexpr (MODE != MODE_FWD) {
          // ---- a7: cotangent with a group-uniform running shift
          const float gmax2 = grpops.max_f(lmax2);
          const float gmax = gmax2 >= 0.f ? sqrtf(gmax2) * kp.invN : -1.f;
          if (gmax >= 0.f && gmax > shift) {
            float sc_S = 0.f, sc_G = 0.f;  // PNORM with shift 0: nothing accumulated (0^p = 0)
            if (mode == 1) {
              if (shift > -INFINITY) sc_S = sc_G = __expf(bp * (shift - gmax));
            } else if (shift > 0.f) {
              sc_G = __powf(shift / gmax, bp - 1.f);
              sc_S = sc_G * (shift / gmax);
            }
            Ssum *= sc_S;
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = make_float2(acc[i].x * sc_G, acc[i].y * sc_G);
            if constexpr (MODE == MODE_ADJ_B) {
              for (int n = t; n < N; n += T) gacc[n] = make_float2(gacc[n].x * sc_G, gacc[n].y * sc_G);
            }
            shift = gmax;
          }
          const float lb = bp * 1.4426950408889634f;  // exp(b x) = exp2(lb x)
#pragma unroll
          for (int i = 0; i < E; ++i) {
            float gfac = 0.f;
            if ((roi >> i) & 1u) {
              float wt = 1.f;
              if (has_w) wt = __ldg(wrow + lag_of(t + i * T, N, P));
              if (wt > 0.f) {
                const float a2 = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
                const float rsq = a2 > 0.f ? rsqrtf(a2) : 0.f;
                const float vv = wt * a2 * rsq * kp.invN;
                float phi, gphi;
                if (mode == 1) {
                  phi = exp2f(lb * (vv - shift));
                  gphi = phi;
                } else if (shift > 0.f) {
                  const float q = vv / shift;
                  gphi = __powf(q, bp - 1.f);
                  phi = gphi * q;
                } else {
                  phi = gphi = 0.f;
                }
                Ssum += phi;
                gfac = gphi * wt * rsq;  // unnormalized G = gphi * w * A / |A|  (0 at A = 0)
              }
            }
            v[i] = make_float2(v[i].x * gfac, v[i].y * gfac);
          }
          // ---- a7: G_hat = FFT(G placed at (-tau) mod P) -- the same positions as r
          fft<PL, -1>(v, ftw, xbuf, t, par, grpops.sync);
          if constexpr (MODE == MODE_ADJ_B) {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmul(v[i], __ldg(Hl + t + i * T)));
          } else {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmulc(__ldg(Xr + t + i * T), v[i]));  // X conj(G_hat)
          }
        }
      }  // l
      if constexpr (MODE == MODE_ADJ_B) {
        // ---- a8B: e = IFFT(sum_l G_hat H_l / P), demodulate, accumulate over the chunk's bins
        fft<PL, +1>(acc, ftw, xbuf, t, par, grpops.sync);
        const float2* twr = dtw + (size_t)k * N;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int n = t + i * T;
          if (n < N) gacc[n] = cadd(gacc[n], cmulc(acc[i], __ldg(twr + n)));
        }
      }
    }  // m (Step A)
  }    // k

  // ---- group partials
  const unsigned long long key_a =
      grpops.max_u64(best_a >= 0.f ? pack_key(best_a, bidx_a) : 0ull);
  const unsigned long long key_c =
      grpops.max_u64(best_c >= 0.f ? pack_key(best_c, bidx_c) : 0ull);
  float gshift = shift, gS;
  if constexpr (MODE == MODE_FWD) {
    gshift = grpops.max_f(shift);  // combine per-thread shifts inside the group
    float term = 0.f;
    if (Ssum > 0.f) term = (mode == 1) ? Ssum * __expf(bp * (shift - gshift)) : Ssum * __powf(shift / gshift, bp);
    gS = grpops.sum_f(term);
  } else {
    gS = grpops.sum_f(Ssum);
  }
  if (!active) return;
  if (t == 0) {
    part.key[2 * gg] = key_a;
    part.key[2 * gg + 1] = key_c;
    part.m[gg] = gshift;
    part.S[gg] = gS;
  }
  if constexpr (MODE == MODE_ADJ_A) {
    // ---- a8A: d = IFFT(sum X conj(G_hat)) -> the group's dL/dw_l^* partial (x 1/P in the combine)
    fft<PL, +1>(acc, ftw, xbuf, t, par, grpops.sync);
    float2* gout = part.g + (size_t)gg * N;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int n = t + i * T;
      if (n < N) gout[n] = acc[i];
    }
  } else if constexpr (MODE == MODE_ADJ_B) {
    float2* gout = part.g + (size_t)gg * N;
    for (int n = t; n < N; n += T) gout[n] = gacc[n];
  }
}

// a2: H_l = FFT_P([w_l; 0]) / P for every (r, l); one group per filter.
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_filter_fft(int RM, int N, const float2* __restrict__ w, const float2* __restrict__ ftw, float2* __restrict__ Hh) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int id = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (PL::NP > 1 ? 2 * PL::PADDED : 0);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int rl = id < RM ? id : RM - 1;
  float2 v[E];
  const float2* wr = w + (size_t)rl * N;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    v[i] = n < N ? __ldg(wr + n) : make_float2(0.f, 0.f);
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);
  if (id >= RM) return;
  const float sc = 1.0f / (float)P;
#pragma unroll
  for (int i = 0; i < E; ++i) Hh[(size_t)rl * P + t + i * T] = make_float2(v[i].x * sc, v[i].y * sc);
}

}  // namespace sq
