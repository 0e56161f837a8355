// Fused AF/CAF forward + adjoint kernels.
//
// A *group* of T = P/E threads owns one Doppler evaluation unit at a time and
// keeps every spectrum in registers (strided ownership, fft.cuh):
//
//   forward (MODE_FWD), unit (r, m, k):
//     x_hat = s_m . e^{j 2 pi n f_k / N}      Eq. 33 (twiddle table built in fp64)
//     X = FFT_P(x_hat_pad)                      Eq. 35-36
//     for l:  r = IFFT_P(X . conj(H_l)/P)       Eq. 36, A(tau) = r[(-tau) mod P] (Q1)
//             fused epilogue: |A|, ROI mask, packed (value, ~index) max keys for
//             WAPSL / WCPSL (Eqs. 7-9), LSE / p-norm partial sums, optional |A| map.
//   Step B adjoint (MODE_ADJ_B), unit (r, m, k): as forward, then per l
//     G = dL/dA^* (unnormalized: phi * w * A / |A|) in place, G_hat = FFT_P(G),
//     acc += G_hat . H_l/P ;  after the l loop e = IFFT_P(acc) and the group adds
//     conj(e^{j 2 pi n f/N}) e[n] into its per-(r, m) gradient partial (a8B).
//   Step A adjoint (MODE_ADJ_A), group (r, l, chunk of k), loop over (k, m):
//     X, r, G, G_hat as above and acc += X . conj(G_hat); at the end of the chunk
//     d = IFFT_P(acc) is the group's dL/dw_l^* partial (a8A).
//
// The cotangent needs the LSE / p-norm normalizer of the *whole* loss, so the
// adjoint kernels accumulate with a group-uniform running shift m (online
// rescaling): phi = e^{beta (v - m)} (LSE) or (v / m)^{p-1} (PNORM), and the
// combine kernel rescales every group to the global shift, so one pass is exact.
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
  int loss_mode;    // 0 MAX, 1 LSE, 2 PNORM
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
  float2* g;                // [Gtot][N] adjoint partial (time domain)
};

__device__ __forceinline__ unsigned long long pack_key(float val, uint32_t idx) {
  return ((unsigned long long)__float_as_uint(val) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}

// Group-level helpers: T <= 32 -> shuffles inside the group's lanes; T > 32 -> shuffles
// + one smem slot per warp + a group barrier.
template <int T>
struct Group {
  GroupSync sync;
  unsigned mask;
  float* red;  // 2 * 32 floats (double-buffered)
  unsigned long long* redk;
  int par;
  int t;

  __device__ __forceinline__ float max_f(float x) {
    const int W = T < 32 ? T : 32;
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
  // Fixed-order sums (bitwise identical across runs).
  __device__ __forceinline__ float sum_f(float x) {
    const int W = T < 32 ? T : 32;
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
    const int W = T < 32 ? T : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(mask, x, o);
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
  static constexpr int XBUF = PL::NP > 1 ? 2 * PL::P : 0;
  static constexpr int GACC = MODE == MODE_ADJ_B ? PL::P / 2 : 0;  // N <= P/2
  static constexpr int RED = 64;                                    // 64 float2 = 2x32 u64 / 2x32 f32
  static constexpr int TOTAL = XBUF + GACC + 2 * RED;
};

// phi for the surrogate sums, with a shift m: LSE e^{beta (v - m)}, PNORM (v/m)^p (0 if m <= 0).
__device__ __forceinline__ float surrogate_term(int mode, float v, float m, float bp) {
  if (mode == 1) return __expf(bp * (v - m));
  return m > 0.f ? __powf(v / m, bp) : 0.f;
}

// Epilogue on one IFFT output slice r[j] (j = t + i T) of map (m, l, k).
// Returns per-element v = w |A| / N (or -1 outside the ROI) in vv[], updates keys,
// writes the optional |A| map.
template <class PL>
__device__ __forceinline__ void epilogue_cells(const KP& kp, const float2 (&v)[PL::E], float (&vv)[PL::E],
                                               float (&rs)[PL::E], int t, int r, int m, int l, int k,
                                               unsigned long long& key_a, unsigned long long& key_c,
                                               float* __restrict__ af_mag) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  const int N = kp.N;
  const bool is_auto = (m == l);
  const uint32_t base_idx = (uint32_t)((m * kp.M + l) * kp.L);
  float* mrow = af_mag ? af_mag + ((((size_t)r * kp.M + m) * kp.M + l) * kp.K + k) * (size_t)kp.L : nullptr;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int j = t + i * T;
    const int tau = (j < N) ? -j : (j > P - N ? P - j : (1 << 24));
    const float a2 = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
    const float rsq = a2 > 0.f ? rsqrtf(a2) : 0.f;
    const float mag = a2 * rsq;
    rs[i] = rsq;
    if (mrow && tau != (1 << 24)) mrow[tau + N - 1] = mag;
    bool in = tau >= kp.tau_lo && tau <= kp.tau_hi && !(is_auto && kp.excl0 && tau == 0);
    float wt = 1.f;
    if (in && kp.weights) {
      wt = __ldg(kp.weights + (size_t)k * kp.L + tau + N - 1);
      in = wt > 0.f;
    }
    vv[i] = in ? wt * mag * kp.invN : -1.f;
    if (in) {
      const uint32_t idx = (base_idx + (uint32_t)(tau + N - 1)) * (uint32_t)kp.K + (uint32_t)k;
      const unsigned long long key = pack_key(wt * wt * a2, idx);
      if (is_auto) key_a = key > key_a ? key : key_a;
      else key_c = key > key_c ? key : key_c;
    }
  }
}

template <class PL, int G, int MODE>
__global__ void __launch_bounds__(PL::T* G)
    k_af(const KP kp, const float2* __restrict__ s, const float2* __restrict__ Hh,
         const float2* __restrict__ dtw, float* __restrict__ af_mag, Part part) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  using GS = GroupSmem<PL, MODE>;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int gg = kp.g_lo + blockIdx.x * G + grp;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * GS::TOTAL;
  float2* xbuf = gsm;
  float2* gacc = gsm + GS::XBUF;
  float* red = reinterpret_cast<float*>(gsm + GS::XBUF + GS::GACC);
  unsigned long long* redk = reinterpret_cast<unsigned long long*>(gsm + GS::XBUF + GS::GACC + GS::RED);

  Group<T> grpops;
  grpops.sync.id = 1 + grp;
  grpops.sync.nthreads = T;
  grpops.sync.mask = T >= 32 ? 0xffffffffu : (((1u << T) - 1u) << ((threadIdx.x & 31) & ~(T - 1)));
  grpops.mask = grpops.sync.mask;
  grpops.red = red;
  grpops.redk = redk;
  grpops.par = 0;
  grpops.t = t;

  const bool active = gg < kp.g_hi;
  const int M = kp.M, N = kp.N;
  const int ra = active ? gg / kp.C : 0, c = active ? gg % kp.C : 0;
  const int r = ra / M, a = ra % M;
  const int k0 = c * kp.chunk;
  const int k1 = active ? min(kp.K, k0 + kp.chunk) : k0;

  float2 tw[PL::NTW];
  init_twiddles<PL>(tw, t);
  int par = 0;

  unsigned long long key_a = 0ull, key_c = 0ull;
  const int mode = kp.loss_mode;
  const float bp = kp.beta_or_p;
  // forward: per-thread shift; adjoint: group-uniform shift (starts at -inf / 0)
  float shift = (mode == 2) ? 0.f : -INFINITY;
  float Ssum = 0.f;

  float2 v[E], xh[E], acc[E];
  float vv[E], rs[E];
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
      // ---- a3: Doppler modulation (Eq. 33) + forward FFT of the zero-padded code
      const float2* sr = s + ((size_t)r * M + m) * N;
      const float2* twr = dtw + (size_t)k * N;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int n = t + i * T;
        v[i] = n < N ? cmul(__ldg(sr + n), __ldg(twr + n)) : make_float2(0.f, 0.f);
      }
      fft<PL, -1>(v, tw, xbuf, t, par, grpops.sync);
#pragma unroll
      for (int i = 0; i < E; ++i) xh[i] = v[i];
      if constexpr (MODE == MODE_ADJ_B) {
#pragma unroll
        for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
      }
      const int l_lo = (MODE == MODE_ADJ_A) ? a : 0, l_hi = (MODE == MODE_ADJ_A) ? a + 1 : M;
      for (int l = l_lo; l < l_hi; ++l) {
        const float2* Hl = Hh + ((size_t)r * M + l) * P;
        // ---- a4: cross-spectrum + IFFT (Eq. 36); H is stored pre-scaled by 1/P
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = cmulc(xh[i], __ldg(Hl + t + i * T));
        fft<PL, +1>(v, tw, xbuf, t, par, grpops.sync);
        // ---- a5: fused cell epilogue
        epilogue_cells<PL>(kp, v, vv, rs, t, r, m, l, k, key_a, key_c, af_mag);
        if constexpr (MODE == MODE_FWD) {
          if (kp.want_S) {
#pragma unroll
            for (int i = 0; i < E; ++i) {
              if (vv[i] < 0.f) continue;
              if (vv[i] > shift) {  // per-thread online rescale
                if (Ssum > 0.f) Ssum *= (mode == 1) ? __expf(bp * (shift - vv[i])) : __powf(shift / vv[i], bp);
                shift = vv[i];
              }
              Ssum += surrogate_term(mode, vv[i], shift, bp);
            }
          }
        } else {
          // ---- a7: cotangent with a group-uniform running shift
          float lmax = -INFINITY;
#pragma unroll
          for (int i = 0; i < E; ++i) lmax = fmaxf(lmax, vv[i]);
          const float gmax = grpops.max_f(lmax);
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
#pragma unroll
          for (int i = 0; i < E; ++i) {
            float phi = 0.f, gphi = 0.f;
            if (vv[i] >= 0.f) {
              if (mode == 1) {
                phi = __expf(bp * (vv[i] - shift));
                gphi = phi;
              } else if (shift > 0.f) {
                const float q = vv[i] / shift;
                gphi = __powf(q, bp - 1.f);
                phi = gphi * q;
              }
            }
            Ssum += phi;
            // unnormalized G = gphi * w * A / |A|; w |A| / N = vv  ->  w / |A| = vv * N / |A|^2
            const float wfac = vv[i] >= 0.f ? gphi * vv[i] * (float)N * rs[i] * rs[i] : 0.f;
            v[i] = make_float2(v[i].x * wfac, v[i].y * wfac);
          }
          // ---- a7: G_hat = FFT(G placed at (-tau) mod P) -- same positions as r
          fft<PL, -1>(v, tw, xbuf, t, par, grpops.sync);
          if constexpr (MODE == MODE_ADJ_B) {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmul(v[i], __ldg(Hl + t + i * T)));
          } else {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmulc(xh[i], v[i]));  // X . conj(G_hat)
          }
        }
      }  // l
      if constexpr (MODE == MODE_ADJ_B) {
        // ---- a8B: e = IFFT(sum_l G_hat H_l / P), demodulate, accumulate over the chunk's bins
        fft<PL, +1>(acc, tw, xbuf, t, par, grpops.sync);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int n = t + i * T;
          if (n < N) {
            float2 g = gacc[n];
            gacc[n] = cadd(g, cmulc(acc[i], __ldg(twr + n)));
          }
        }
      }
    }  // m (Step A)
  }    // k

  // ---- group partials
  key_a = grpops.max_u64(key_a);
  key_c = grpops.max_u64(key_c);
  float gshift = shift;
  float gS;
  if constexpr (MODE == MODE_FWD) {
    // combine per-thread shifts inside the group
    gshift = grpops.max_f(shift);
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
    // ---- a8A: d = IFFT(sum X conj(G_hat)) -> the group's dL/dw_l^* partial (x 1/P later)
    fft<PL, +1>(acc, tw, xbuf, t, par, grpops.sync);
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
    k_filter_fft(int RM, int N, const float2* __restrict__ w, float2* __restrict__ Hh) {
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int id = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (PL::NP > 1 ? 2 * P : 0);
  GroupSync sync;
  sync.id = 1 + grp;
  sync.nthreads = T;
  sync.mask = T >= 32 ? 0xffffffffu : (((1u << T) - 1u) << ((threadIdx.x & 31) & ~(T - 1)));
  float2 tw[PL::NTW];
  init_twiddles<PL>(tw, t);
  const int rl = id < RM ? id : RM - 1;
  float2 v[E];
  const float2* wr = w + (size_t)rl * N;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    v[i] = n < N ? __ldg(wr + n) : make_float2(0.f, 0.f);
  }
  int par = 0;
  fft<PL, -1>(v, tw, xbuf, t, par, sync);
  if (id >= RM) return;
  const float sc = 1.0f / (float)P;
#pragma unroll
  for (int i = 0; i < E; ++i) Hh[(size_t)rl * P + t + i * T] = make_float2(v[i].x * sc, v[i].y * sc);
}

}  // namespace sq
