// Fused AF/CAF forward + adjoint kernels.
//
// A *group* of T = P/E threads owns one evaluation unit at a time and keeps its
// spectra in registers (strided ownership, fft.cuh).
//
//   k_xhat, unit (r, m, k):                        a3
//     x_hat = s_m . e^{j 2 pi n f_k / N}            Eq. 33 (twiddle table built in fp64)
//     X_{m,k} = FFT_P(x_hat_pad)  -> X cache [R][M][K][P] (L2-resident for C1-C4)
//   The fused kernel is persistent: each group pulls units (r, a, k) from an atomic
//   counter and writes that unit's partials into the unit's own slot, so the load is
//   balanced across SMs while every sum stays in a fixed order (deterministic).
//   forward (MODE_FWD), unit (r, m, k):              a4-a5
//     for l: r = IFFT_P(X . conj(H_l)/P)            Eq. 36; A(tau) = r[(-tau) mod P] (Q1)
//            fused epilogue: |A|, ROI mask, (value, index) max keys for WAPSL /
//            WCPSL (Eqs. 7-9), LSE / p-norm partial sums, optional |A| map.
//   Step B adjoint (MODE_ADJ_B), unit (r, m, k):     a4-a7, a8B
//     per l: r, then G = dL/dA^* (unnormalized: phi * w * A / |A|) in place,
//     G_hat = FFT_P(G), acc += G_hat . H_l/P;  after the l loop e = IFFT_P(acc),
//     demodulated by conj(e^{j 2 pi n f/N}) -> the unit's time-domain slot.
//   Step A adjoint (MODE_ADJ_A), unit (r, l, k), loop over m:   a4-a7, a8A
//     r, G, G_hat as above and acc += X . conj(G_hat) -> the unit's spectral slot;
//     the combine sums the slots over k and one IFFT_P per filter gives dL/dw_l^*.
//   Every transform of a unit runs through ONE inlined forward FFT (a phase loop):
//   IFFT(x) = conj(FFT(conj x)), the conjugations folded into the adjacent products.
//
// The cotangent needs the LSE / p-norm normalizer of the *whole* loss, so each unit
// accumulates with a unit-uniform running shift m (online rescaling):
// phi = e^{beta (v - m)} (LSE) or (v / m)^{p-1} (PNORM); the combine rescales every
// unit to the restart's global shift, so one pass is exact.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "fft.cuh"

namespace sq {

enum { MODE_FWD = 0, MODE_ADJ_A = 1, MODE_ADJ_B = 2 };

#ifndef SQNGD_AF_TWS
#define SQNGD_AF_TWS 0  // shared-memory twiddles: measured no gain (C3 FFT engine, C4)
#endif

struct KP {
  int R, M, N, K, L, P;
  int tau_lo, tau_hi, excl0;
  int loss_mode;  // 0 MAX, 1 LSE, 2 PNORM
  float beta_or_p;
  float invN;
  const float* weights;  // [K][L] or nullptr
  int u_lo, u_hi;        // units evaluated by this rank (multi-GPU slice of R*M*K)
  int want_S;            // forward: accumulate surrogate sums
  int* counter;          // dynamic unit counter (zeroed before the launch)
  uint32_t* tiew;        // [R][2] 1 + float bits of the largest value at which a group saw two cells tie (zeroed with counter)
  int track_tie;         // 1: track ties (SQNGD_FLAG_TIE requested)
  int mld;               // |A| map row pitch (floats)
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
  // fixed-order fp64 sum of a (re, im) pair; smem slots reuse the u64 area
  __device__ __forceinline__ double2 sum_d2(double2 x) {
    constexpr int W = T < 32 ? T : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      x.x += __shfl_xor_sync(mask, x.x, o);
      x.y += __shfl_xor_sync(mask, x.y, o);
    }
    if constexpr (T > 32) {
      double* b = reinterpret_cast<double*>(redk) + (par ? 32 : 0);
      par ^= 1;
      if ((t & 31) == 0) {
        b[(t >> 5)] = x.x;
        b[(t >> 5) + 16] = x.y;
      }
      sync();
      x = make_double2(b[0], b[16]);
#pragma unroll
      for (int w = 1; w < T / 32; ++w) {
        x.x += b[w];
        x.y += b[w + 16];
      }
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

// Per-group shared memory of the single-FFT kernels (exchange buffers + reduction slots).
template <class PL>
struct FftSmem {
  static constexpr int XBUF = PL::NP > 1 ? 2 * PL::PADDED : 0;
  static constexpr int TOTAL = XBUF + 32 + 64;
};

// Per-group shared memory (float2 units).
template <class PL, int MODE>
struct GroupSmem {
  static constexpr int XBUF = PL::NP > 1 ? 2 * PL::PADDED : 0;
  static constexpr int RED = 32;    // 64 floats (2 x 32)
  static constexpr int REDK = 64;   // 64 u64 (2 x 32)
  static constexpr int GRAB = 1;    // 2 ints: the unit index broadcast (double-buffered)
  static constexpr int TOTAL = XBUF + RED + REDK + GRAB;
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

// MUFU approximations (no denormal fix-up code): 2^x and 1/sqrt(x), |rel err| ~ 2^-22.
__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2a(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqa(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Per-slice constants of the epilogue.
struct SliceCtx {
  uint32_t roi;         // ROI bitmask of this thread's elements for this map (auto / cross)
  const float* wrow;    // weights row (HW) centred at tau = 0
  uint32_t base_idx;    // (m M + l) L + N - 1
  int k;
};

// Lowest cell index among this thread's in-ROI elements whose key value equals kv
// (the rare path of the running argmax: taken only when a slice reaches the running max).
template <class PL, bool HW>
__device__ __forceinline__ uint32_t argmax_index(const float2 (&v)[PL::E], float kv, const SliceCtx& sc, int t, int N,
                                              int K, int& cnt) {
  uint32_t best = 0xFFFFFFFFu;
  cnt = 0;  // cells of value kv (SQNGD_FLAG_TIE)
#pragma unroll
  for (int i = 0; i < PL::E; ++i) {
    if (!((sc.roi >> i) & 1u)) continue;
    const int lag = lag_of(t + i * PL::T, N, PL::P);
    float x = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
    if (HW) {
      const float wt = __ldg(sc.wrow + lag);
      if (!(wt > 0.f)) continue;
      x *= wt * wt;
    }
    if (x == kv) {
      ++cnt;
      const uint32_t idx = (sc.base_idx + (uint32_t)lag) * (uint32_t)K + (uint32_t)sc.k;
      best = idx < best ? idx : best;
    }
  }
  return best;
}

// Pass 1 of the cell epilogue: max over the thread's in-ROI cells of w^2 |A|^2 (-1 if none).
template <class PL, bool HW>
__device__ __forceinline__ float slice_max2(const float2 (&v)[PL::E], const SliceCtx& sc, int t, int N) {
  float lmax2 = -1.f;
#pragma unroll
  for (int i = 0; i < PL::E; ++i) {
    float kv = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
    if (HW) {
      const float wt = ((sc.roi >> i) & 1u) ? __ldg(sc.wrow + lag_of(t + i * PL::T, N, PL::P)) : 0.f;
      kv = wt > 0.f ? kv * wt * wt : -1.f;
    } else {
      kv = ((sc.roi >> i) & 1u) ? kv : -1.f;
    }
    lmax2 = fmaxf(lmax2, kv);
  }
  return lmax2;
}

// Pass 2: surrogate terms phi with shift `shift` (LSE: e^{b(v-m)}, PNORM: (v/m)^p), summed
// into Ssum; if GRAD, v <- G = gphi w A / |A| (v holds conj(A) on entry, hence the sign).
// v = w |A| / N.  Cells outside the ROI get phi = 0 and G = 0; |A| = 0 gives G = 0.
template <class PL, bool HW, int LM, bool GRAD>
__device__ __forceinline__ void slice_terms(float2 (&v)[PL::E], const SliceCtx& sc, int t, int N, float invN,
                                            float shift, float bp, float& Ssum) {
  const float lb = bp * 1.4426950408889634f;
  const float lbN = lb * invN, lbs = lb * shift;        // LSE: phi = 2^{lbN |A| w - lb m}
  const float qN = shift > 0.f ? invN / shift : 0.f;    // PNORM: q = w |A| / (N m)
#pragma unroll
  for (int i = 0; i < PL::E; ++i) {
    const float a2 = fmaf(v[i].x, v[i].x, v[i].y * v[i].y);
    const float rsq = rsqa(fmaxf(a2, 1e-30f));
    const float mag = a2 * rsq;
    float wt = 1.f;
    if (HW) wt = ((sc.roi >> i) & 1u) ? __ldg(sc.wrow + lag_of(t + i * PL::T, N, PL::P)) : 0.f;
    const bool in = HW ? (wt > 0.f) : (((sc.roi >> i) & 1u) != 0u);
    float phi, gphi;
    if (LM == 1) {
      phi = ex2a(fmaf(lbN, HW ? wt * mag : mag, -lbs));
      gphi = phi;
    } else {
      const float q = (HW ? wt * mag : mag) * qN;
      gphi = ex2a((bp - 1.f) * lg2a(q));  // q^(p-1); 0 at q = 0
      phi = gphi * q;
    }
    phi = in ? phi : 0.f;
    Ssum += phi;
    if (GRAD) {
      const float gfac = in ? gphi * (HW ? wt * rsq : rsq) : 0.f;
      v[i] = make_float2(v[i].x * gfac, -v[i].y * gfac);
    }
  }
}

// a3: X_{m,k} = FFT_P(s_m e^{j 2 pi n f_k / N}) for every unit (r, m, k) -> X cache.
template <class PL, int G, int MINB>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_xhat(int u0, int units, int M, int N, int K, const float2* __restrict__ s, const float2* __restrict__ dtw,
           const float2* __restrict__ ftw, float2* __restrict__ Xc, const float2* __restrict__ w, double2* cm) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int u = blockIdx.x * G + grp;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  float2* xbuf = gsm;
  Group<T> gops;
  gops.sync = GroupSync{1 + grp, T, group_mask(T)};
  gops.mask = gops.sync.mask;
  gops.red = reinterpret_cast<float*>(gsm + FftSmem<PL>::XBUF);
  gops.redk = reinterpret_cast<unsigned long long*>(gsm + FftSmem<PL>::XBUF + 32);
  gops.par = 0;
  gops.t = t;
  const int uu = u0 + (u < units ? u : units - 1);  // units [u0, u0 + units): this rank's shard
  const int k = uu % K, rm = uu / K;
  const float2* sr = s + (size_t)rm * N;
  const float2* twr = dtw + (size_t)k * N;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    v[i] = n < N ? cmul(__ldg(sr + n), __ldg(twr + n)) : make_float2(0.f, 0.f);
  }
  if (w != nullptr && k == 0) {  // a6: c_m = sum_n s_m(n) conj(w_m(n)) = A_mm(0,0) (Eq. 38), fp64
    const float2* wr = w + (size_t)rm * N;
    double2 acc = make_double2(0.0, 0.0);
    for (int n = t; n < N; n += T) {
      const float2 a = __ldg(sr + n), b = __ldg(wr + n);
      acc.x += (double)a.x * b.x + (double)a.y * b.y;
      acc.y += (double)a.y * b.x - (double)a.x * b.y;
    }
    acc = gops.sum_d2(acc);
    if (t == 0 && u < units) cm[rm] = acc;
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, gops.sync);
  if (u >= units) return;
  float2* out = Xc + (size_t)uu * P;
#pragma unroll
  for (int i = 0; i < E; ++i) out[t + i * T] = v[i];
}

template <class PL, int G, int MINB, int MODE>
__global__ void __launch_bounds__(PL::T* G, MINB)
    k_af(const KP kp, const float2* __restrict__ Xc, const float2* __restrict__ Hh,
         const float2* __restrict__ dtw, const float2* __restrict__ ftw, float* __restrict__ af_mag, Part part) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  using GS = GroupSmem<PL, MODE>;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * GS::TOTAL;
  float2* xbuf = gsm;
  int* grab = reinterpret_cast<int*>(gsm + GS::XBUF + GS::RED + GS::REDK);

  Group<T> grpops;
  grpops.sync = GroupSync{1 + grp, T, group_mask(T)};
  grpops.mask = grpops.sync.mask;
  grpops.red = reinterpret_cast<float*>(gsm + GS::XBUF);
  grpops.redk = reinterpret_cast<unsigned long long*>(gsm + GS::XBUF + GS::RED);
  grpops.par = 0;
  grpops.t = t;

#if SQNGD_AF_TWS
  // the plan's Stockham twiddles, staged once per (persistent) CTA in shared memory
  float2* tws = reinterpret_cast<float2*>(smem_raw) + G * GS::TOTAL;
  for (int i = threadIdx.x; i < PL::TWSIZE; i += blockDim.x) tws[i] = __ldg(ftw + i);
  __syncthreads();
  const float2* twt = tws;
#else
  const float2* twt = ftw;
#endif
  const int M = kp.M, N = kp.N, K = kp.K;
  const int mode = kp.loss_mode;
  const float bp = kp.beta_or_p;
  const float lb = bp * 1.4426950408889634f;  // e^{b x} = 2^{lb x}
  uint32_t roi_auto, roi_cross;
  roi_masks<PL>(kp, t, roi_auto, roi_cross);
  const bool has_w = kp.weights != nullptr;
  int par = 0, gpar = 0;
  int cur_r = -1;
  unsigned long long key_a = 0ull, key_c = 0ull;  // packed (w^2 |A|^2, ~index) maxima
  uint32_t tie_a = 0u, tie_c = 0u;                 // largest value at which two of the group's cells tied
  float2 v[E];
  float2 acc[MODE == MODE_FWD ? 1 : E];

  for (;;) {
    // ---- dynamic unit scheduling: one atomic per unit, broadcast through smem
    if (t == 0) grab[gpar] = atomicAdd(kp.counter, 1);
    grpops.sync();
    const int u = kp.u_lo + grab[gpar];
    gpar ^= 1;
    if (u >= kp.u_hi) break;
    const int k = u % K, ra = u / K;
    const int r = ra / M, a = ra % M;
    const float* wrow = has_w ? kp.weights + (size_t)k * kp.L + N - 1 : nullptr;

    float shift = (mode == 2) ? 0.f : -INFINITY;  // unit-uniform running shift of the sums
    float Ssum = 0.f;
    if (r != cur_r) {  // group-uniform running (value, index) maxima, kept across units of one restart
      cur_r = r;
      key_a = key_c = 0ull;
      tie_a = tie_c = 0u;
    }
    if constexpr (MODE != MODE_FWD) {
#pragma unroll
      for (int i = 0; i < E; ++i) acc[i] = make_float2(0.f, 0.f);
    }

    // Phases: FWD: M slices; ADJ_A: (slice, G) x M; ADJ_B: (slice, G) x M + final IFFT(acc).
    const int nph = (MODE == MODE_FWD) ? M : (MODE == MODE_ADJ_B ? 2 * M + 1 : 2 * M);
#pragma unroll 1
    for (int ph = 0; ph < nph; ++ph) {
      const bool final_ph = (MODE == MODE_ADJ_B) && ph == 2 * M;
      const bool slice_ph = (MODE == MODE_FWD) || (!final_ph && (ph & 1) == 0);
      const int li = (MODE == MODE_FWD) ? ph : (ph >> 1);
      const int m = (MODE == MODE_ADJ_A) ? li : a;
      const int l = (MODE == MODE_ADJ_A) ? a : li;
      const float2* Xr = Xc + (((size_t)r * M + m) * K + k) * P;
      const float2* Hl = Hh + ((size_t)r * M + (final_ph ? 0 : l)) * P;
      // ---- pre: the transform's input
      if (slice_ph) {
        // a4: conj(X . conj(H_l)/P) = conj(X) . H_l/P ; FFT of the conjugate = conj(IFFT) (Eq. 36)
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = cmulc(__ldg(Hl + t + i * T), __ldg(Xr + t + i * T));
      } else if (final_ph) {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_float2(acc[i].x, -acc[i].y);
      }  // G phase: v already holds G
      fft<PL, -1, SQNGD_AF_TWS != 0>(v, twt, xbuf, t, par, grpops.sync);
      // ---- post
      if (slice_ph) {
        // v[i] = conj(r[j]), j = t + i T, A(tau) = r[(-tau) mod P]  (a5: fused epilogue)
        const bool is_auto = (m == l);
        SliceCtx sc;
        sc.roi = is_auto ? roi_auto : roi_cross;
        sc.wrow = wrow;
        sc.base_idx = (uint32_t)((m * M + l) * kp.L + N - 1);
        sc.k = k;
        if constexpr (MODE == MODE_FWD) {
          if (af_mag) {
            float* mrow = af_mag + ((((size_t)r * M + m) * M + l) * K + k) * (size_t)kp.mld + N - 1;
#pragma unroll
            for (int i = 0; i < E; ++i) {
              const int j = t + i * T;
              if (j < N || j > P - N) mrow[lag_of(j, N, P)] = sqrtf(fmaf(v[i].x, v[i].x, v[i].y * v[i].y));
            }
          }
        }
        const float lmax2 = has_w ? slice_max2<PL, true>(v, sc, t, N) : slice_max2<PL, false>(v, sc, t, N);
        const float gmax2 = grpops.max_f(lmax2);
        // running argmax per map type (group-uniform branch, taken only when the running max is
        // reached): the threads holding the max find their lowest cell index, one more reduction
        unsigned long long& kcat = is_auto ? key_a : key_c;
        if (gmax2 >= 0.f && __float_as_uint(gmax2) >= (uint32_t)(kcat >> 32)) {
          uint32_t idx = 0xFFFFFFFFu;
          int cnt = 0;
          if (lmax2 == gmax2)
            idx = has_w ? argmax_index<PL, true>(v, lmax2, sc, t, N, K, cnt)
                        : argmax_index<PL, false>(v, lmax2, sc, t, N, K, cnt);
          const unsigned long long cand = grpops.max_u64(lmax2 == gmax2 ? pack_key(gmax2, idx) : 0ull);
          // SQNGD_FLAG_TIE: two cells of this slice, or a cell of an earlier slice, at the value gmax2
          if (MODE == MODE_FWD && kp.track_tie) {  // (uniform; forward only: the adjoints keep their code)
            const float ncell = grpops.sum_f((float)cnt);
            if (ncell >= 2.f || (kcat != 0ull && (uint32_t)(kcat >> 32) == __float_as_uint(gmax2))) {
              uint32_t& tcat = is_auto ? tie_a : tie_c;
              tcat = max(tcat, __float_as_uint(gmax2) + 1u);
            }
          }
          kcat = cand > kcat ? cand : kcat;
        }
        // ---- surrogate sums (and a7: the cotangent) with a unit-uniform running shift
        const float gmax = gmax2 >= 0.f ? sqrtf(gmax2) * kp.invN : -1.f;
        if (mode != 0 && gmax >= 0.f && gmax > shift) {
          float sc_S = 0.f, sc_G = 0.f;  // PNORM with shift 0: nothing accumulated yet (0^p = 0)
          if (mode == 1) {
            if (shift > -INFINITY) sc_S = sc_G = ex2a(lb * (shift - gmax));
          } else if (shift > 0.f) {
            sc_G = ex2a((bp - 1.f) * lg2a(shift / gmax));
            sc_S = sc_G * (shift / gmax);
          }
          Ssum *= sc_S;
          if constexpr (MODE != MODE_FWD) {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = make_float2(acc[i].x * sc_G, acc[i].y * sc_G);
          }
          shift = gmax;
        }
        constexpr bool GRAD = MODE != MODE_FWD;
        if (mode == 1 && (GRAD || kp.want_S)) {
          if (has_w) slice_terms<PL, true, 1, GRAD>(v, sc, t, N, kp.invN, shift, bp, Ssum);
          else slice_terms<PL, false, 1, GRAD>(v, sc, t, N, kp.invN, shift, bp, Ssum);
        } else if (mode == 2 && (GRAD || kp.want_S)) {
          if (has_w) slice_terms<PL, true, 2, GRAD>(v, sc, t, N, kp.invN, shift, bp, Ssum);
          else slice_terms<PL, false, 2, GRAD>(v, sc, t, N, kp.invN, shift, bp, Ssum);
        }
      } else if (final_ph) {
        // a8B: v = conj(e), e = IFFT(sum_l G_hat H_l / P); slot <- e conj(tw) = conj(v tw)
        const float2* twr = dtw + (size_t)k * N;
        float2* gout = part.g + (size_t)u * P;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int n = t + i * T;
          if (n < N) {
            const float2 q = cmul(v[i], __ldg(twr + n));
            gout[n] = make_float2(q.x, -q.y);
          }
        }
      } else {
        // G phase: v = G_hat
        if constexpr (MODE == MODE_ADJ_B) {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmul(v[i], __ldg(Hl + t + i * T)));
        } else if constexpr (MODE == MODE_ADJ_A) {
#pragma unroll
          for (int i = 0; i < E; ++i) acc[i] = cadd(acc[i], cmulc(__ldg(Xr + t + i * T), v[i]));  // X conj(G_hat)
        }
      }
    }  // phases

    // ---- unit partials (keys: the group's running maxima of this restart)
    const float uS = grpops.sum_f(Ssum);
    const float ushift = shift;
    if (t == 0) {
      part.key[2 * (size_t)u] = key_a;
      part.key[2 * (size_t)u + 1] = key_c;
      if (MODE == MODE_FWD && tie_a) atomicMax(kp.tiew + 2 * r, tie_a);
      if (MODE == MODE_FWD && tie_c) atomicMax(kp.tiew + 2 * r + 1, tie_c);
      part.m[u] = ushift;
      part.S[u] = uS;
    }
    if constexpr (MODE == MODE_ADJ_A) {
      float2* gout = part.g + (size_t)u * P;  // spectral partial of dL/dw_l^* (unscaled)
#pragma unroll
      for (int i = 0; i < E; ++i) gout[t + i * T] = acc[i];
    }
  }
}

// Step A combine, second half: d_l = IFFT_P(spectral sum)[0..N) for each (r, l) row,
// via the forward FFT of the conjugate.
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_rows_ifft(int rows, int N, const float2* __restrict__ in, const float2* __restrict__ ftw, float2* __restrict__ out) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int id = blockIdx.x * G + grp;
  float2* xbuf = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  GroupSync sync{1 + grp, T, group_mask(T)};
  const int row = id < rows ? id : rows - 1;
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const float2 x = __ldg(in + (size_t)row * P + t + i * T);
    v[i] = make_float2(x.x, -x.y);
  }
  int par = 0;
  fft<PL, -1>(v, ftw, xbuf, t, par, sync);
  if (id >= rows) return;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    if (n < N) out[(size_t)row * N + n] = make_float2(v[i].x, -v[i].y);
  }
}

// a2: H_l = FFT_P([w_l; 0]) / P for every (r, l); one group per filter.
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_filter_fft(int RM, int N, const float2* __restrict__ w, const float2* __restrict__ ftw, float2* __restrict__ Hh,
                 const float2* __restrict__ s, double2* cm) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int id = blockIdx.x * G + grp;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  float2* xbuf = gsm;
  Group<T> gops;
  gops.sync = GroupSync{1 + grp, T, group_mask(T)};
  gops.mask = gops.sync.mask;
  gops.red = reinterpret_cast<float*>(gsm + FftSmem<PL>::XBUF);
  gops.redk = reinterpret_cast<unsigned long long*>(gsm + FftSmem<PL>::XBUF + 32);
  gops.par = 0;
  gops.t = t;
  const GroupSync& sync = gops.sync;
  const int rl = id < RM ? id : RM - 1;
  if (s != nullptr) {  // a6: c_m = sum_n s_m(n) conj(w_m(n)) (Eq. 38), fp64
    const float2* sr = s + (size_t)rl * N;
    const float2* wr = w + (size_t)rl * N;
    double2 acc = make_double2(0.0, 0.0);
    for (int n = t; n < N; n += T) {
      const float2 a = __ldg(sr + n), b = __ldg(wr + n);
      acc.x += (double)a.x * b.x + (double)a.y * b.y;
      acc.y += (double)a.y * b.x - (double)a.x * b.y;
    }
    acc = gops.sum_d2(acc);
    if (t == 0 && id < RM) cm[rl] = acc;
  }
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
