// Small kernels around the fused AF path: quantizer (a1), mainlobe (a6),
// deterministic partial combines (a5/a8), loss / metric finalization (a6),
// the sparse MAX-mode adjoint, the chain through Q_A (a8B), Adam and the two
// projections (a9).
#pragma once
#include <stdint.h>

#include "af_kernels.cuh"  // (+ common.cuh)

namespace sq {

// ------------------------------------------------------------------ a1 quantizer
// fp64 table of the hard levels: lut[i*] = k with y_hard = k / B for i* = #{rho <= z}
// (Eq. 43 with the nearest-level snap of Q12; decision in fp64 like the oracle).
__global__ void k_hard_lut(int B, int BR, double c, const float* __restrict__ rho, int* __restrict__ lut,
                           int* __restrict__ status) {
  SQ_PDL_WAIT();
  extern __shared__ float rr[];  // the restart's thresholds (the searches below are dependent chains)
  const int r = blockIdx.y;
  {
    const float* rg = rho + (size_t)r * BR;
    for (int base = 0; base < BR; base += 8 * (int)blockDim.x) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = base + k * blockDim.x + threadIdx.x;
        v[k] = i < BR ? __ldg(rg + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = base + k * blockDim.x + threadIdx.x;
        if (i < BR) rr[i] = v[k];
      }
    }
    __syncthreads();
  }
  int* out = lut + (size_t)r * (BR + 1);
  const double W = 20.0 / c;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // one warp per entry
  if (i > BR) return;
  if (i == 0 || i == BR) {
    if (lane == 0) out[i] = i == 0 ? 0 : (int)floor(B * (2.0 * BR / (2.0 * B)) + 0.5);
    return;
  }
  if (lane == 0 && rr[i - 1] > rr[i]) atomicOr(status, ST_INVALID);
  const double x = 0.5 * ((double)rr[i - 1] + (double)rr[i]);
  int lo = 0, hi = BR;  // cnt = #{rho_j <= x}
  while (lo < hi) { int mid = (lo + hi) >> 1; if ((double)rr[mid] <= x) lo = mid + 1; else hi = mid; }
  const int cnt = lo;
  // window [i0, i1): |c (x - rho)| < 20 ; outside, tanh + 1 is 0 or 2 to < 1e-17
  lo = 0; hi = cnt;
  while (lo < hi) { int mid = (lo + hi) >> 1; if ((double)rr[mid] < x - W) lo = mid + 1; else hi = mid; }
  const int i0 = lo;
  lo = cnt; hi = BR;
  while (lo < hi) { int mid = (lo + hi) >> 1; if ((double)rr[mid] <= x + W) lo = mid + 1; else hi = mid; }
  const int i1 = lo;
  double resid = 0.0;  // y = cnt/B + a * resid
  for (int j = i0 + lane; j < i1; j += 32) {
    const double u = c * (x - (double)rr[j]);
    const double e2 = exp(-2.0 * fabs(u));
    const double tt = 2.0 * e2 / (1.0 + e2);  // 1 - tanh|u|
    resid += (j >= cnt) ? tt : -tt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) resid += __shfl_xor_sync(0xffffffffu, resid, o);
  if (lane == 0) out[i] = cnt + (int)floor(0.5 * resid + 0.5);  // floor(B y + 1/2), B a = 1/2
}

// y_soft = Q_A(z) (Eq. 24) as cnt/B + a*resid (integer plateau count + small residual, so the
// phase 2 pi y keeps fp32 precision although y reaches r_n), s_soft = e^{j 2 pi y} (Eq. 23),
// dq = Q_A'(z); hard: s_hard = e^{j 2 pi b / B}, b = lut[cnt] mod B.
// 8 lanes per element split the tanh window; fixed xor-shuffle order (deterministic).
__global__ void k_quantize(int MN, int B, int BR, float c, const float* __restrict__ z,
                           const float* __restrict__ rho, const int* __restrict__ lut, float2* s_soft,
                           float2* s_hard, uint8_t* b_hard, float* dq) {
  SQ_PDL_WAIT();
  extern __shared__ float rs[];
  constexpr int LPE = 8;
  const int r = blockIdx.y;
  const float* rr = rho + (size_t)r * BR;
  for (int base = 0; base < BR; base += 8 * (int)blockDim.x) {  // 8 loads in flight per thread
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + k * blockDim.x + threadIdx.x;
      v[k] = i < BR ? __ldg(rr + i) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + k * blockDim.x + threadIdx.x;
      if (i < BR) rs[i] = v[k];
    }
  }
  __syncthreads();
  const int sub = threadIdx.x & (LPE - 1);
  const int e0 = blockIdx.x * (blockDim.x / LPE) + threadIdx.x / LPE;
  const bool ok = e0 < MN;
  const size_t e = (size_t)r * MN + (ok ? e0 : 0);
  const float x = z[e];
  // counts #{rs < v} (strict) or #{rs <= v} over the ascending thresholds: a guess from the
  // near-uniform spacing (rho_i ~ (i + 1/2) / BR), corrected by a short walk, with a binary
  // search if the walk would be long -- the same exact count as a plain binary search
  auto count = [&](float v, bool le) -> int {
    int i = (int)floorf(v * (float)BR + 0.5f);
    i = i < 0 ? 0 : (i > BR ? BR : i);
    for (int step = 0; step < 6; ++step) {
      const bool below = i > 0 && (le ? rs[i - 1] > v : rs[i - 1] >= v);   // count too high
      const bool above = i < BR && (le ? rs[i] <= v : rs[i] < v);          // count too low
      if (!below && !above) return i;
      i += above ? 1 : -1;
    }
    int lo = 0, hi = BR;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (le ? rs[mid] <= v : rs[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int cnt = count(x, true);
  if (s_soft || dq) {
    const float W = 12.0f / c;
    const int i0 = count(x - W, false);
    const int i1 = count(x + W, true);
    float resid = 0.f, sech = 0.f;
    for (int j = i0 + sub; j < i1; j += LPE) {
      const float u = c * (x - rs[j]);
      const float e2 = ex2a_m(-2.8853900817779268f * fabsf(u));  // e^{-2|u|}
      const float inv = rcp_m(1.f + e2);
      const float tt = 2.f * e2 * inv;
      resid += (j >= cnt) ? tt : -tt;
      sech += 4.f * e2 * inv * inv;
    }
#pragma unroll
    for (int o = LPE / 2; o > 0; o >>= 1) {
      resid += __shfl_xor_sync(0xffffffffu, resid, o);
      sech += __shfl_xor_sync(0xffffffffu, sech, o);
    }
    const float a = 1.f / (2.f * B);
    if (ok && sub == 0) {
      if (dq) dq[e] = a * c * sech;
      if (s_soft) {
        float ph = (float)(cnt % B) / (float)B + a * resid;
        ph -= floorf(ph);
        float sn, cs;
        sincospif(2.f * ph, &sn, &cs);
        s_soft[e] = make_float2(cs, sn);
      }
    }
  }
  if (ok && sub == 0 && (s_hard || b_hard)) {
    const int k = lut[(size_t)r * (BR + 1) + cnt];
    const int b = ((k % B) + B) % B;
    if (b_hard) b_hard[e] = (uint8_t)b;
    if (s_hard) {
      float sn, cs;
      sincospif(2.f * (float)b / (float)B, &sn, &cs);
      s_hard[e] = make_float2(cs, sn);
    }
  }
}

// ------------------------------------------------------------------ a6 metrics / loss
// ------------------------------------------------------------------ combines
// Per restart: max keys, global shift and the rescaled sum S over the restart's units
// [r * GPR, (r+1) * GPR) intersected with [g_lo, g_hi); per-unit rescale factors for the
// gradient combine.  One block of 1024 threads per restart, fixed order (deterministic).
__global__ void k_reduce_groups(int GPR, int g_lo, int g_hi, int mode, double bp, Part part, Red* red,
                                MetricsArgs ma, int* status, const uint32_t* tiew) {
  SQ_PDL_WAIT();
  __shared__ double shd[32];
  __shared__ unsigned long long shk[32];
  reduce_restart(blockIdx.x, GPR, g_lo, g_hi, mode, bp, part, red, ma, status, shd, shk, tiew);
}

// Multi-GPU: the shift m arrived from the all-reduce; refresh the per-group scales.
__global__ void k_group_scales(int GPR, int g_lo, int g_hi, int mode, double bp, Part part, const Red* red) {
  SQ_PDL_WAIT();
  const int r = blockIdx.x;
  const int lo = max(g_lo, r * GPR), hi = min(g_hi, (r + 1) * GPR);
  const double m = red[r].m;
  for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    float sc = 0.f;
    if (part.S[g] > 0.f && m > -INFINITY) {
      const float mg = part.m[g], mf = (float)m;
      sc = mode == 1 ? exp2f((float)(bp * 1.4426950408889634) * (mg - mf)) : exp2f((float)(bp - 1.0) * log2f(mg / mf));
    }
    part.scale[g] = sc;
  }
}

// Unit slots -> per-row sums in true units of dL_wpsl / d(.)^*:
// out[ra][q] = norm_r * sum_k scale[u] slot[u][q],  u = ra K + k  (fixed order),
// norm_r = eps/(2N) * extra * (LSE: 1/S_r, PNORM: S_r^{1/p-1}).  Block: 32 q x 8 k-lanes.
// ------------------------------------------------------------------ MAX-mode sparse adjoint
// Eq. 37's subgradient goes to the unique argmax cell (Q17): recompute A there by the O(N)
// correlation and write the whole red_grad[r] (zero elsewhere).
// wrt 1 (filters): dL/dw_l*^*(n) = conj(G) x_hat_{m*,k*}(n - tau*);
// wrt 2 (transmit): dL/ds_m*^*(n) = G e^{-j2pi n f/N} w_l*(n + tau*).
__global__ void k_sparse_adj(int M, int N, int K, int L, int wrt, double eps, const float* __restrict__ weights,
                             const float2* __restrict__ s, const float2* __restrict__ w,
                             const float2* __restrict__ dtw, const Red* __restrict__ red, float2* red_grad) {
  SQ_PDL_WAIT();
  __shared__ double sre[256], sim[256];
  const int r = blockIdx.x;
  const unsigned long long ka = red[r].key_a, kc = red[r].key_c;
  const unsigned long long key = ka > kc ? ka : kc;
  const bool any = key != 0ull;
  const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
  const int k = idx % K;
  const int ti = (idx / K) % L;
  const int l = (idx / K / L) % M;
  const int m = idx / K / L / M;
  const int tau = ti - (N - 1);
  const float2* sm = s + ((size_t)r * M + m) * N;
  const float2* wl = w + ((size_t)r * M + l) * N;
  const float2* tw = dtw + (size_t)k * N;
  double re = 0.0, im = 0.0;
  if (any) {
    for (int n = max(0, -tau) + threadIdx.x; n < min(N, N - tau); n += blockDim.x) {
      const float2 xh = cmul(sm[n], tw[n]);
      const float2 p = cmulc(xh, wl[n + tau]);
      re += p.x;
      im += p.y;
    }
  }
  sre[threadIdx.x] = re;
  sim[threadIdx.x] = im;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sre[threadIdx.x] += sre[threadIdx.x + o];
      sim[threadIdx.x] += sim[threadIdx.x + o];
    }
    __syncthreads();
  }
  const double Ar = sre[0], Ai = sim[0];
  const double mag = sqrt(Ar * Ar + Ai * Ai);
  const double wt = weights ? (double)weights[(size_t)k * L + ti] : 1.0;
  double Gr = 0.0, Gi = 0.0;  // G = eps * (w/N) * A / (2|A|)
  if (any && mag > 0.0) {
    Gr = eps * wt / N * Ar / (2.0 * mag);
    Gi = eps * wt / N * Ai / (2.0 * mag);
  }
  const float2 G = make_float2((float)Gr, (float)Gi);
  for (int e = threadIdx.x; e < M * N; e += blockDim.x) {
    const int a = e / N, n = e % N;
    float2 out = make_float2(0.f, 0.f);
    if (any) {
      if (wrt == 1 && a == l) {
        const int nn = n - tau;
        if (nn >= 0 && nn < N) out = cmulc(cmul(sm[nn], tw[nn]), G) ;  // x_hat conj(G)
      } else if (wrt == 2 && a == m) {
        const int nn = n + tau;
        if (nn >= 0 && nn < N) out = cmul(cmulc(G, tw[n]), wl[nn]);    // G conj(tw) w
      }
    }
    red_grad[((size_t)r * M) * N + e] = out;
  }
}

__global__ void k_metrics(MetricsArgs a, int* status) {
  SQ_PDL_WAIT();
  metrics_warp(a, blockIdx.x, status);
}

// ------------------------------------------------------------------ finalize gradients
// Step A: grad_w = 2 (red_grad + conj(Gc_l) s_l)           (Q16)
// Step B: g = red_grad + Gc_m w_m = dL/ds^*; optional grad_s; dy = 4 pi Im(g conj(s)),
//         grad_z = dq * dy (Eqs. 23-24 chain).
// Gc_m = (1-eps)(2/M)(p_m - p_tar)/N * c_m / (2|c_m|)   (Eq. 41 on c_m = A_mm(0,0)).
struct FinArgs {
  int R, M, N, wrt;
  double eps, ptar;
  const double2* cm;
  const float2* s;
  const float2* w;
  const float* dq;
  float2* grad_w;
  float2* grad_s;
  float* dy;
  float* grad_z;
};

// Element e = (row, n) of the final gradient from the WPSL part rg (true units):
// Step A: grad_w = 2 (rg + conj(Gc_l) s_l)           (Q16)
// Step B: g = rg + Gc_m w_m = dL/ds^*; dy = 4 pi Im(g conj(s)), grad_z = dq * dy (Eqs. 23-24)
// Gc_m = (1-eps)(2/M)(p_m - p_tar)/N * c_m / (2|c_m|)   (Eq. 41 on c_m = A_mm(0,0)).
__device__ __forceinline__ double2 snrl_coef(const FinArgs& f, size_t row) {
  const double2 c = f.cm[row];
  const double mag = sqrt(c.x * c.x + c.y * c.y);
  if (!(mag > 0.0)) return make_double2(0.0, 0.0);
  const double q = (1.0 - f.eps) * (2.0 / f.M) * (mag / f.N - f.ptar) / f.N / (2.0 * mag);
  return make_double2(q * c.x, q * c.y);
}

// The element's inputs (s, w, dq), loaded ahead of the arithmetic by callers that batch them.
struct FinIn {
  float2 s, w;
  float dq;
};
__device__ __forceinline__ FinIn finalize_load(const FinArgs& f, size_t e) {
  FinIn in;
  in.s = f.s[e];
  in.w = f.wrt == 1 ? make_float2(0.f, 0.f) : f.w[e];
  in.dq = (f.wrt != 1 && f.grad_z) ? f.dq[e] : 0.f;
  return in;
}
__device__ __forceinline__ void finalize_pre(const FinArgs& f, size_t e, float2 rg, double2 gc, const FinIn& in,
                                             int* status) {
  const float gr = (float)gc.x, gi = (float)gc.y;
  bool bad;
  if (f.wrt == 1) {
    const float2 sv = in.s;
    const float re = rg.x + (gr * sv.x + gi * sv.y);
    const float im = rg.y + (gr * sv.y - gi * sv.x);
    if (f.grad_w) f.grad_w[e] = make_float2(2.f * re, 2.f * im);
    bad = !isfinite(re) || !isfinite(im);
  } else {
    const float2 wv = in.w;
    const float re = rg.x + (gr * wv.x - gi * wv.y);
    const float im = rg.y + (gr * wv.y + gi * wv.x);
    if (f.grad_s) f.grad_s[e] = make_float2(re, im);
    const float2 sv = in.s;
    const float d = 4.f * 3.14159265358979f * (im * sv.x - re * sv.y);  // Im(g conj(s))
    if (f.dy) f.dy[e] = d;
    if (f.grad_z) f.grad_z[e] = in.dq * d;
    bad = !isfinite(re) || !isfinite(im);
  }
  if (bad) atomicOr(status, ST_NONFINITE);
}

__device__ __forceinline__ void finalize_elem(const FinArgs& f, size_t e, float2 rg, double2 gc, int* status) {
  const float gr = (float)gc.x, gi = (float)gc.y;
  bool bad;
  if (f.wrt == 1) {
    const float2 sv = f.s[e];  // conj(Gc) s
    const float re = rg.x + (gr * sv.x + gi * sv.y);
    const float im = rg.y + (gr * sv.y - gi * sv.x);
    if (f.grad_w) f.grad_w[e] = make_float2(2.f * re, 2.f * im);
    bad = !isfinite(re) || !isfinite(im);
  } else {
    const float2 wv = f.w[e];  // Gc w
    const float re = rg.x + (gr * wv.x - gi * wv.y);
    const float im = rg.y + (gr * wv.y + gi * wv.x);
    if (f.grad_s) f.grad_s[e] = make_float2(re, im);
    const float2 sv = f.s[e];
    const float d = 4.f * 3.14159265358979f * (im * sv.x - re * sv.y);  // Im(g conj(s))
    if (f.dy) f.dy[e] = d;
    if (f.grad_z) f.grad_z[e] = f.dq[e] * d;
    bad = !isfinite(re) || !isfinite(im);
  }
  if (bad) atomicOr(status, ST_NONFINITE);
}

__global__ void k_finalize_grad(FinArgs f, const float2* __restrict__ red_grad, int* status, MetricsArgs ma) {
  SQ_PDL_WAIT();
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x < 32 && blockIdx.x < (unsigned)f.R && (ma.out || ma.loss_hist)) metrics_warp(ma, blockIdx.x, status);
  if (e >= (size_t)f.R * f.M * f.N) return;
  finalize_elem(f, e, red_grad[e], snrl_coef(f, e / f.N), status);
}

// Step A tail: d_l = IFFT_P(spectral sum)[0..N) per (r, l) row (forward FFT of the conjugate),
// then finalize.
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_rows_ifft_fin(int rows, const float2* __restrict__ in, const float2* __restrict__ ftw, FinArgs f, int* status) {
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
  const double2 gc = snrl_coef(f, row);
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    if (n < f.N) finalize_elem(f, (size_t)row * f.N + n, make_float2(v[i].x, -v[i].y), gc, status);
  }
}

struct CombineArgs {
  int M, N, K, len, slot_stride, u_lo, u_hi, mode;
  double bp, eps, extra;
  Part part;
  const Red* red;     // restart shift / sum (from k_reduce_groups or the multi-GPU all-reduce)
  float2* out;        // [R*M][len] (when !fin)
  int fin;            // 1: apply finalize_elem to each output (len == N)
  FinArgs f;
};

// Unit slots -> per-row sums in true units of dL_wpsl / d(.)^*:
// out[ra][q] = norm_r * sum_k scale_u slot_u[q],  u = ra K + k  (fixed order),
// norm_r = eps/(2N) * extra * (LSE: 1/S_r, PNORM: S_r^{1/p-1}).
// Block: 32 lanes x 2 complex (q) x KL k-lanes (16 for the long slot lists: one load round trip per lane).
template <int KL>
__global__ void __launch_bounds__(32 * KL) k_combine_rows(CombineArgs a, int* status) {
  SQ_PDL_WAIT();
  __shared__ float4 sh[KL][33];
  const int ra = blockIdx.y;
  const int r = ra / a.M;
  const double m = a.red[r].m, S = a.red[r].S;
  const bool live = m > -INFINITY && S > 0.0;
  double norm = 0.0;  // (fp64 divide / pow issued now, off the critical path of the slot sums)
  if (live) norm = a.eps / (2.0 * a.N) * a.extra * ((a.mode == 1) ? 1.0 / S : pow(S, 1.0 / a.bp - 1.0));
  const int q = 2 * (blockIdx.x * 32 + (threadIdx.x & 31));  // two complex values per thread
  const int kl = threadIdx.x >> 5;                              // KL k-lanes
  FinIn fin0{}, fin1{};
  double2 gcf = make_double2(0.0, 0.0);
  if (a.fin && kl == 0 && q < a.len) {  // finalize inputs fetched now, overlapping the slot sums
    fin0 = finalize_load(a.f, (size_t)ra * a.N + q);
    if (q + 1 < a.len) fin1 = finalize_load(a.f, (size_t)ra * a.N + q + 1);
    gcf = snrl_coef(a.f, ra);
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live && q < a.len) {
    const int klo = max(0, a.u_lo - ra * a.K), khi = min(a.K, a.u_hi - ra * a.K);
#pragma unroll 8
    for (int k = klo + kl; k < khi; k += KL) {
      const int u = ra * a.K + k;
      const float sc = a.part.scale ? __ldg(a.part.scale + u) : 1.f;  // null: slots pre-scaled (Chebyshev engine)
      const float4 v = __ldg(reinterpret_cast<const float4*>(a.part.g + (size_t)u * a.slot_stride + q));
      acc.x = fmaf(sc, v.x, acc.x);
      acc.y = fmaf(sc, v.y, acc.y);
      acc.z = fmaf(sc, v.z, acc.z);
      acc.w = fmaf(sc, v.w, acc.w);
    }
  }
  sh[kl][threadIdx.x & 31] = acc;
  __syncthreads();
  if (kl == 0 && q < a.len) {
    float4 t = sh[0][threadIdx.x];
#pragma unroll
    for (int j = 1; j < KL; ++j) {
      t.x += sh[j][threadIdx.x].x;
      t.y += sh[j][threadIdx.x].y;
      t.z += sh[j][threadIdx.x].z;
      t.w += sh[j][threadIdx.x].w;
    }
    const float nf = (float)norm;
    const float2 g0 = make_float2(t.x * nf, t.y * nf), g1 = make_float2(t.z * nf, t.w * nf);
    if (a.fin) {
      finalize_pre(a.f, (size_t)ra * a.N + q, g0, gcf, fin0, status);
      if (q + 1 < a.len) finalize_pre(a.f, (size_t)ra * a.N + q + 1, g1, gcf, fin1, status);
    } else {
      float2* o = a.out + (size_t)ra * a.len + q;
      o[0] = g0;
      if (q + 1 < a.len) o[1] = g1;
    }
  }
}

// Step A tail for the optimizer step, one group per filter row (r, l):
//   d = IFFT_P(spectral sum)[0..N), grad_w = 2 (d + conj(Gc_l) s_l) (finalize), Adam on
//   (Re w, Im w), Pi_H (Eq. 32, fp64 energy), then the next inner step's H_l = FFT_P(w_l)/P and
//   c_l = sum_n s_l conj(w_l).  A row whose gradient is non-finite is not updated (status latched).
template <class PL, int G>
__global__ void __launch_bounds__(PL::T* G)
    k_rows_adam_w(int rows, const float2* __restrict__ in, const float2* __restrict__ ftw, FinArgs f, AdamP ap,
                  float2* w, float* mw, float* vw, float2* Hh, double2* cm, int* status) {
  SQ_PDL_WAIT();
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  extern __shared__ float4 smem_raw[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int id = blockIdx.x * G + grp;
  float2* gsm = reinterpret_cast<float2*>(smem_raw) + grp * (FftSmem<PL>::TOTAL);
  Group<T> gops;
  gops.sync = GroupSync{1 + grp, T, group_mask(T)};
  gops.mask = gops.sync.mask;
  gops.red = reinterpret_cast<float*>(gsm + FftSmem<PL>::XBUF);
  gops.redk = reinterpret_cast<unsigned long long*>(gsm + FftSmem<PL>::XBUF + 32);
  gops.par = 0;
  gops.t = t;
  const int row = id < rows ? id : rows - 1;
  const int N = f.N;
  const bool skip_all = (*status & ST_NONFINITE) != 0;  // uniform
  float2 v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const float2 x = __ldg(in + (size_t)row * P + t + i * T);
    v[i] = make_float2(x.x, -x.y);
  }
  // the row's s, w and Adam moments, loaded up front: their latency hides behind the IFFT (inside
  // the update loop the moment stores would otherwise serialize one round trip per element)
  float2 sv[E], wv[E], mv[E], vv[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int n = t + i * T;
    const size_t j = (size_t)row * N + (n < N ? n : 0);
    sv[i] = f.s[j];
    wv[i] = w[j];
    mv[i] = reinterpret_cast<const float2*>(mw)[j];
    vv[i] = reinterpret_cast<const float2*>(vw)[j];
  }
  const double2 gc = snrl_coef(f, row);
  float c1, c2;
  ap.corr(c1, c2);
  int par = 0;
  double2 cacc = make_double2(0.0, 0.0);
  // one inlined FFT instance for both transforms (IFFT of the spectral sum, then FFT of the new
  // w): half the code, which matters on the few SMs this row kernel runs on (instruction cache)
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    fft<PL, -1>(v, ftw, gsm, t, par, gops.sync);
    if (ph == 1) break;
    float bad = 0.f;
    double e = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int n = t + i * T;
      float2 wn = make_float2(0.f, 0.f);
      if (n < N) {
        const size_t j = (size_t)row * N + n;
        const float re = 2.f * (v[i].x + ((float)gc.x * sv[i].x + (float)gc.y * sv[i].y));   // d = conj(v)
        const float im = 2.f * (-v[i].y + ((float)gc.x * sv[i].y - (float)gc.y * sv[i].x));
        if (!isfinite(re) || !isfinite(im)) bad = 1.f;
        if (f.grad_w && id < rows) f.grad_w[j] = make_float2(re, im);
        const float g2[2] = {re, im};
        float x2[2] = {wv[i].x, wv[i].y};
        const float m2[2] = {mv[i].x, mv[i].y}, v2[2] = {vv[i].x, vv[i].y};
        float mo[2], vo[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {  // Adam on the real parameters (Re w, Im w)
          mo[q] = ap.b1 * m2[q] + (1.f - ap.b1) * g2[q];
          vo[q] = ap.b2 * v2[q] + (1.f - ap.b2) * g2[q] * g2[q];
          x2[q] -= ap.lr * (mo[q] / c1) / (sqrtf(vo[q] / c2) + ap.eps);
        }
        if (!skip_all && id < rows) {  // (a padding group duplicates the last row: no stores)
          reinterpret_cast<float2*>(mw)[j] = make_float2(mo[0], mo[1]);
          reinterpret_cast<float2*>(vw)[j] = make_float2(vo[0], vo[1]);
        }
        wn = make_float2(x2[0], x2[1]);
        e += (double)wn.x * wn.x + (double)wn.y * wn.y;
      }
      v[i] = wn;
    }
    const float gbad = gops.max_f(bad);
    const double en = gops.sum_d2(make_double2(e, 0.0)).x;
    if (skip_all || gbad > 0.f || !(en > 0.0)) {
      if (t == 0 && id < rows) atomicOr(status, gbad > 0.f ? ST_NONFINITE : (en > 0.0 ? 0 : ST_DEGENERATE));
      return;  // uniform across the group
    }
    const float sc = (float)sqrt((double)N / en);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int n = t + i * T;
      v[i] = make_float2(v[i].x * sc, v[i].y * sc);
      if (n < N) {
        const size_t j = (size_t)row * N + n;
        if (id < rows) w[j] = v[i];
        // c_l = sum_n s_l(n) conj(w_l(n)) for the next evaluation
        cacc.x += (double)sv[i].x * v[i].x + (double)sv[i].y * v[i].y;
        cacc.y += (double)sv[i].y * v[i].x - (double)sv[i].x * v[i].y;
      }
    }
    cacc = gops.sum_d2(cacc);
  }  // next H_l = FFT_P(w_l) / P
  if (id >= rows) return;
  if (t == 0) cm[row] = cacc;
  const float inv = 1.0f / (float)P;
#pragma unroll
  for (int i = 0; i < E; ++i) Hh[(size_t)row * P + t + i * T] = make_float2(v[i].x * inv, v[i].y * inv);
}

// dL/drho_i = -a c sum_e sech^2(c (z_e - rho_i)) dy_e, gathered per threshold over a chunk of
// elements (partials [R][nchunk][BR], then a fixed-order sum).  sech^2 via MUFU, culled
// outside |c (z - rho)| < 12 where it is < 1.6e-10: per element, a warp whose 32 (sorted)
// thresholds all lie farther than 12/c from z skips it (warp-uniform test), so only the
// ~2 x 12/c x B r_n thresholds near each z do the work.
__device__ void adam_project_rho_dev(int r, int BR, float* rho, float* mr, float* vr, const float* g, const AdamP& ap,
                                     float lo, float hi, float gap, float* sr);

// Finishing work done by last-arriving blocks (arrival counters, self-resetting; fixed-order sums):
//   per (r, threshold block): grad_rho[i] = coef * sum_ch part[ch][i]  (when gsum != nullptr);
//   per (r, element chunk):   Adam on the chunk's z (when zad.z != nullptr) -- after every
//                             threshold block has read that chunk's old z.
// Adam on z (direct parameterization), by the blocks 1.. of k_adam_project_rho (after k_grad_rho read z).
struct ZAdam {
  float *z, *mz, *vz;  // z == nullptr: none (generator mode)
  const float* gz;     // grad_z [R][MN]
  int MN;
  AdamP ap;
};

// dL/drho_i = coef sum_n sech^2(c (z_n - rho_i)) dy_n over the window |c (z_n - rho_i)| < 12 (the chain of
// Eq. 25 through Q_A; the oracle's chain()), in one pass without sorting.  Block = TB
// consecutive thresholds x TPT lanes each (rho ascending, so their union window is one z interval).  Per
// chunk of CH elements the block compacts, in a fixed order (thread, then element), the (z, dy) whose z lies
// in the union window (block-wide exclusive scan of the per-thread counts), and lane `sub` of a threshold
// sums every TPT-th compacted element; the TPT lanes combine by a fixed xor tree.  Deterministic.
template <int TB>
__global__ void __launch_bounds__(256) k_grad_rho(int MN, int BR, float c, float coef, const float* __restrict__ z,
                                                  const float* __restrict__ rho, const float* __restrict__ dy,
                                                  float* __restrict__ gsum) {
  SQ_PDL_WAIT();
  constexpr int TPT = 256 / TB, EPT = 16, CH = 256 * EPT;
  static_assert(TPT >= 1 && (TPT & (TPT - 1)) == 0 && TPT <= 32, "TPT lanes per threshold, within a warp");
  __shared__ float2 buf[CH];
  __shared__ int wsum[8];
  const int r = blockIdx.y, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int i0 = blockIdx.x * TB;
  const int i = min(i0 + t / TPT, BR - 1);
  const int sub = t % TPT;
  const float* rr = rho + (size_t)r * BR;
  const float ri = __ldg(rr + i);
  const float W = 12.f / c;
  const float zlo = __ldg(rr + i0) - W, zhi = __ldg(rr + min(i0 + TB, BR) - 1) + W;
  const float* zr = z + (size_t)r * MN;
  const float* dr = dy + (size_t)r * MN;
  const float k2 = -2.f * 1.4426950408889634f;
  float acc4[4] = {0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < MN; base += CH) {
    float zv[EPT];
    unsigned inm = 0u;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = base + k * 256 + t;
      zv[k] = e < MN ? __ldg(zr + e) : 0.f;
      const bool in = e < MN && zv[k] >= zlo && zv[k] <= zhi;
      inm |= in ? (1u << k) : 0u;
      cnt += in ? 1 : 0;
    }
    // block-wide exclusive scan of cnt
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int off = x - cnt, n = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int v = wsum[w];
      off += w < wid ? v : 0;
      n += v;
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (inm & (1u << k)) buf[off++] = make_float2(zv[k], __ldg(dr + base + k * 256 + t));
    __syncthreads();
    // four independent partial sums per lane (element e + j TPT, j < 4, of each group of 4 TPT)
    for (int e = sub; e < n; e += 4 * TPT) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ej = e + j * TPT;
        const float2 p = ej < n ? buf[ej] : make_float2(ri + 2.f * W, 0.f);
        const float au = c * fabsf(p.x - ri);
        const float e2 = ex2a_m(k2 * au);
        const float inv = rcp_m(1.f + e2);
        const float sech2 = 4.f * e2 * inv * inv;
        acc4[j] = fmaf(au < 12.f ? sech2 : 0.f, p.y, acc4[j]);
      }
    }
    __syncthreads();  // (buf and wsum are rewritten by the next chunk)
  }
  float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
#pragma unroll
  for (int o = 1; o < TPT; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (sub == 0 && i0 + t / TPT < BR) gsum[(size_t)r * BR + i0 + t / TPT] = coef * acc;
}


// ------------------------------------------------------------------ a9 optimizer
// Adam step counters and the bias corrections (c1, c2) = (1 - b1^t, 1 - b2^t) of every inner step of
// the coming sqngd_step (t = t_a + k + 1 for Step A, t_b + k + 1 for Step B), computed in fp64 exactly
// as AdamP::corr does, so the update kernels read one table entry instead of two pow chains.
__global__ void k_set_t(long long* dt, long long ta, long long tb, float2* ct, int cts, int nh, int nx, double b1,
                        double b2) {
  SQ_PDL_WAIT();
  if (threadIdx.x == 0) {
    dt[0] = ta;
    dt[1] = tb;
  }
  for (int k = threadIdx.x; k < cts; k += blockDim.x) {
    if (k < nh) {
      const double t = (double)(ta + k + 1);
      ct[k] = make_float2((float)(1.0 - pow(b1, t)), (float)(1.0 - pow(b2, t)));
    }
    if (k < nx) {
      const double t = (double)(tb + k + 1);
      ct[cts + k] = make_float2((float)(1.0 - pow(b1, t)), (float)(1.0 - pow(b2, t)));
    }
  }
}

__global__ void k_adam(size_t n, float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, AdamP ap, const int* __restrict__ status) {
  SQ_PDL_WAIT();
  if (*status & ST_NONFINITE) return;  // keep the last finite iterate
  float c1, c2;
  ap.corr(c1, c2);
  const float lr = ap.lr, b1 = ap.b1, b2 = ap.b2, eps = ap.eps;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = b1 * m[i] + (1.f - b1) * gi;
  const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  x[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
}

// Adam on (Re w, Im w) of one filter row, then Eq. 32: h_m <- sqrt(N / ||h_m||^2) h_m (fp64 energy).
// One block per row; skipped entirely when a non-finite value is latched.
__global__ void k_adam_project_w(int N, float* w, float* mw, float* vw, const float* __restrict__ g, AdamP ap,
                                 int* status) {
  SQ_PDL_WAIT();
  __shared__ double sh[32];
  if (*status & ST_NONFINITE) return;
  float c1, c2;
  ap.corr(c1, c2);
  const float lr = ap.lr, b1 = ap.b1, b2 = ap.b2, eps = ap.eps;
  const size_t base = (size_t)blockIdx.x * 2 * N;
  double e = 0.0;
  for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
    const size_t j = base + i;
    const float gi = g[j];
    const float mi = b1 * mw[j] + (1.f - b1) * gi;
    const float vi = b2 * vw[j] + (1.f - b2) * gi * gi;
    mw[j] = mi;
    vw[j] = vi;
    const float x = w[j] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    w[j] = x;
    e += (double)x * x;
  }
  auto dsum = [](double x, double y) { return x + y; };
  const double en = block_reduce(e, dsum, sh);
  if (en == 0.0) {
    if (threadIdx.x == 0) atomicOr(status, ST_DEGENERATE);
    return;
  }
  const float sc = (float)sqrt((double)N / en);
  for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) w[base + i] *= sc;
}

// Threshold projection: sort ascending, clamp to [lo, hi], forward min-gap sweep.
// Adam on rho of restart r, then the projection; called by one whole block (any size with
// BR <= 32 blockDim), sr = 2 n2 floats of shared memory (n2 = next power of two >= BR).
// g: the restart's gradient (read with ld.cg: it may come from other blocks of this launch).
__device__ void adam_project_rho_dev(int r, int BR, float* rho, float* mr, float* vr, const float* g, const AdamP& ap,
                                     float lo, float hi, float gap, float* sr) {
  __shared__ int flag, swapped;
  float c1, c2;
  ap.corr(c1, c2);
  const float lr = ap.lr, b1 = ap.b1, b2 = ap.b2, eps = ap.eps;
  float* p = rho + (size_t)r * BR;
  int n2 = 1;
  while (n2 < BR) n2 <<= 1;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int base = 0; base < n2; base += 8 * blockDim.x) {  // Adam step (all loads issued first), then the projection
    float gv[8], mv[8], vv[8], pv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + k * blockDim.x + threadIdx.x;
      if (i < BR) {
        const size_t j = (size_t)r * BR + i;
        gv[k] = __ldcg(g + i);
        mv[k] = mr[j];
        vv[k] = vr[j];
        pv[k] = p[i];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + k * blockDim.x + threadIdx.x;
      if (i >= n2) break;
      float x = INFINITY;
      if (i < BR) {
        const size_t j = (size_t)r * BR + i;
        const float mi = b1 * mv[k] + (1.f - b1) * gv[k];
        const float vi = b2 * vv[k] + (1.f - b2) * gv[k] * gv[k];
        mr[j] = mi;
        vr[j] = vi;
        x = pv[k] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
      }
      sr[i] = x;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i + 1 < BR; i += blockDim.x)
    if (sr[i] > sr[i + 1]) flag = 1;
  __syncthreads();
  if (flag) {
    // nearly sorted (Adam moves each threshold by ~lr per step): odd-even transposition
    // rounds with early exit; a full bitonic sort only if that does not converge.
    int rounds = 0;
    do {
      __syncthreads();
      if (threadIdx.x == 0) swapped = 0;
      __syncthreads();
      for (int ph = 0; ph < 2; ++ph) {
        for (int i = 2 * threadIdx.x + ph; i + 1 < BR; i += 2 * blockDim.x) {
          const float a = sr[i], b = sr[i + 1];
          if (a > b) { sr[i] = b; sr[i + 1] = a; swapped = 1; }
        }
        __syncthreads();
      }
    } while (swapped && ++rounds < 2);  // clusters of near-equal thresholds need many rounds: bitonic then
    if (swapped && n2 == 2 * (int)blockDim.x && n2 >= 128) {
      // bitonic sort with two elements per thread (2t, 2t+1) in registers: partner distances j <= 32
      // stay inside the warp (xor shuffles, no barrier), larger ones go through shared memory
      const int t = threadIdx.x;
      float x0 = sr[2 * t], x1 = sr[2 * t + 1];
      for (int kk = 2; kk <= n2; kk <<= 1) {
        const bool up = ((2 * t) & kk) == 0;  // direction of this thread's pairs (both slots)
        int j = kk >> 1;
        if (j >= 64) {
          sr[2 * t] = x0;
          sr[2 * t + 1] = x1;
          __syncthreads();
          for (; j >= 64; j >>= 1) {
            const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // pair t: i has bit j clear
            const bool upi = (i & kk) == 0;
            const float a = sr[i], b = sr[i | j];
            if ((a > b) == upi) { sr[i] = b; sr[i | j] = a; }
            __syncthreads();
          }
          x0 = sr[2 * t];
          x1 = sr[2 * t + 1];
        }
        for (; j >= 2; j >>= 1) {  // partner of element 2t + b is 2 (t ^ j/2) + b: lane t ^ j/2
          const int h = j >> 1;
          const float y0 = __shfl_xor_sync(0xffffffffu, x0, h), y1 = __shfl_xor_sync(0xffffffffu, x1, h);
          const bool keep_min = ((t & h) == 0) == up;  // lower index of an ascending pair keeps the min
          x0 = keep_min ? fminf(x0, y0) : fmaxf(x0, y0);
          x1 = keep_min ? fminf(x1, y1) : fmaxf(x1, y1);
        }
        if ((x0 > x1) == up) {  // j = 1: the thread's own pair
          const float tmp = x0;
          x0 = x1;
          x1 = tmp;
        }
      }
      sr[2 * t] = x0;
      sr[2 * t + 1] = x1;
    } else if (swapped) {
      for (int kk = 2; kk <= n2; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
          for (int i = threadIdx.x; i < n2; i += blockDim.x) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const bool up = (i & kk) == 0;
              const float a = sr[i], b = sr[ixj];
              if ((a > b) == up) { sr[i] = b; sr[ixj] = a; }
            }
          }
          __syncthreads();
        }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BR; i += blockDim.x) sr[i] = fminf(fmaxf(sr[i], lo), hi);
  __syncthreads();
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int i = threadIdx.x + 1; i < BR; i += blockDim.x)
    if (sr[i] < sr[i - 1] + gap) flag = 1;
  __syncthreads();
  if (flag) {
    // forward sweep rho_i = max(rho_i, rho_{i-1} + gap) == max_{j<=i}(rho_j + (i-j) gap):
    // inclusive prefix max of q_j = rho_j - j gap (Hillis-Steele), value kept exact where inactive.
    float* q = sr + n2;
    if (n2 == 2 * (int)blockDim.x && blockDim.x % 32 == 0 && blockDim.x <= 1024) {
      // two elements per thread; warp scans with shuffles, one shared-memory pass over the warp
      // totals (max is exact, so this equals the Hillis-Steele result bit for bit)
      __shared__ float wtot[32];
      const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
      const int i0 = 2 * t, i1 = 2 * t + 1;
      const float a0 = i0 < BR ? sr[i0] - (float)i0 * gap : -INFINITY;
      const float a1 = i1 < BR ? sr[i1] - (float)i1 * gap : -INFINITY;
      float inc = fmaxf(a0, a1);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = fmaxf(inc, v);
      }
      float exc = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) exc = -INFINITY;
      if (lane == 31) wtot[wp] = inc;
      __syncthreads();
      if (wp == 0) {
        const int nw = blockDim.x >> 5;
        float x = lane < nw ? wtot[lane] : -INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float v = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x = fmaxf(x, v);
        }
        const float xe = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane < nw) wtot[lane] = lane == 0 ? -INFINITY : xe;  // exclusive warp offsets
      }
      __syncthreads();
      const float base = fmaxf(wtot[wp], exc);
      const float p0 = fmaxf(base, a0), p1 = fmaxf(p0, a1);
      if (i0 < BR) q[i0] = p0;
      if (i1 < BR) q[i1] = p1;
      __syncthreads();
    } else {
    for (int i = threadIdx.x; i < BR; i += blockDim.x) q[i] = sr[i] - (float)i * gap;
    __syncthreads();
    for (int off = 1; off < BR; off <<= 1) {
      float tmp[32];
      int cnt = 0;
      for (int i = threadIdx.x; i < BR; i += blockDim.x) tmp[cnt++] = (i >= off) ? fmaxf(q[i], q[i - off]) : q[i];
      __syncthreads();
      cnt = 0;
      for (int i = threadIdx.x; i < BR; i += blockDim.x) q[i] = tmp[cnt++];
      __syncthreads();
    }
    }
    for (int i = threadIdx.x; i < BR; i += blockDim.x) {
      const float qi = sr[i] - (float)i * gap;
      if (q[i] > qi) sr[i] = q[i] + (float)i * gap;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BR; i += blockDim.x) p[i] = sr[i];
}

// Step-B update: block (0, r) Adam(rho) + projection of restart r; blocks (1.., r) Adam(z), 4096 elements each.
__global__ void __launch_bounds__(1024) k_adam_project_rho(int BR, float* rho, float* mr, float* vr, const float* __restrict__ g, AdamP ap,
                                   float lo, float hi, float gap, const int* status, ZAdam za) {
  SQ_PDL_WAIT();
  extern __shared__ float sr[];
  if (*status & ST_NONFINITE) return;  // keep the last finite iterate
  if (blockIdx.x > 0) {  // Adam(z): 4 elements per thread of chunk blockIdx.x - 1 (grid (1 + chunks, R))
    float c1, c2;
    za.ap.corr(c1, c2);
    const int r = blockIdx.y;
    float gv[4], mv[4], vv[4], zv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = (blockIdx.x - 1) * 4 * blockDim.x + k * blockDim.x + threadIdx.x;
      const size_t j = (size_t)r * za.MN + (e < za.MN ? e : 0);
      gv[k] = za.gz[j]; mv[k] = za.mz[j]; vv[k] = za.vz[j]; zv[k] = za.z[j];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = (blockIdx.x - 1) * 4 * blockDim.x + k * blockDim.x + threadIdx.x;
      if (e < za.MN) {
        const size_t j = (size_t)r * za.MN + e;
        const float mi = za.ap.b1 * mv[k] + (1.f - za.ap.b1) * gv[k];
        const float vi = za.ap.b2 * vv[k] + (1.f - za.ap.b2) * gv[k] * gv[k];
        za.mz[j] = mi;
        za.vz[j] = vi;
        za.z[j] = zv[k] - za.ap.lr * (mi / c1) / (sqrtf(vi / c2) + za.ap.eps);
      }
    }
    return;
  }
  adam_project_rho_dev(blockIdx.y, BR, rho, mr, vr, g + (size_t)blockIdx.y * BR, ap, lo, hi, gap, sr);
}

// a6 reporting: SNRL_m = 10 log10(||s_m||^2 ||w_m||^2 / |s_m^H w_m|^2) (Eq. 10) from
// the literal fp64 norms, one block per restart and one warp per channel (fixed-order lane sums, xor
// shuffles); the restart's maximum goes into metrics[r].snrl_db_max and / or worst_out[r].  A zero
// s_m^H w_m gives +inf and latches ST_DEGENERATE.  Launch with blockDim = 32 * min(M, 32).
__global__ void __launch_bounds__(1024) k_snrl(int M, int N, const float2* __restrict__ s,
                                               const float2* __restrict__ w, double* snrl_out, MetricsOut* met,
                                               int* status, double* worst_out) {
  SQ_PDL_WAIT();
  __shared__ double wmax[32];
  const int r = blockIdx.x, lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double worst = -INFINITY;
  for (int m = wp; m < M; m += nw) {
    const float2* sr = s + ((size_t)r * M + m) * N;
    const float2* wr = w + ((size_t)r * M + m) * N;
    double ss = 0.0, ww = 0.0, cr = 0.0, ci = 0.0;
#pragma unroll 8
    for (int n = lane; n < N; n += 32) {  // (unrolled: 8 loads in flight per lane)
      const float2 a = __ldg(sr + n), b = __ldg(wr + n);
      ss += (double)a.x * a.x + (double)a.y * a.y;
      ww += (double)b.x * b.x + (double)b.y * b.y;
      cr += (double)a.x * b.x + (double)a.y * b.y;  // s conj(w)
      ci += (double)a.y * b.x - (double)a.x * b.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      ww += __shfl_xor_sync(0xffffffffu, ww, o);
      cr += __shfl_xor_sync(0xffffffffu, cr, o);
      ci += __shfl_xor_sync(0xffffffffu, ci, o);
    }
    const double c2 = cr * cr + ci * ci;
    const double db = c2 > 0.0 ? 10.0 * log10(ss * ww / c2) : INFINITY;
    if (lane == 0) {
      if (snrl_out) snrl_out[(size_t)r * M + m] = db;
      if (!(c2 > 0.0)) atomicOr(status, ST_DEGENERATE);
    }
    worst = fmax(worst, db);
  }
  if (lane == 0) wmax[wp] = worst;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; ++i) worst = fmax(worst, wmax[i]);
    if (met) met[r].snrl_db_max = worst;
    if (worst_out) worst_out[r] = worst;
  }
}

// ------------------------------------------------------------------ a10 multi-GPU (comm.h)
// c_m = sum_n s_m(n) conj(w_m(n)) (fp64) for every row: the sharded forward computes it only for the rows
// it owns, but the metrics and the SNRL term need all of them on every rank.  One warp per row.
__global__ void k_cm_rows(int RM, int N, const float2* __restrict__ s, const float2* __restrict__ w, double2* cm) {
  SQ_PDL_WAIT();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= RM) return;
  const float2* sr = s + (size_t)row * N;
  const float2* wr = w + (size_t)row * N;
  double cr = 0.0, ci = 0.0;
  for (int n = lane; n < N; n += 32) {
    const float2 a = __ldg(sr + n), b = __ldg(wr + n);
    cr += (double)a.x * b.x + (double)a.y * b.y;
    ci += (double)a.y * b.x - (double)a.x * b.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    ci += __shfl_xor_sync(0xffffffffu, ci, o);
  }
  if (lane == 0) cm[row] = make_double2(cr, ci);
}

struct WorldArgs {
  int R, M, N, mode, with_grad;
  double bp;
  Red* red;                   // per restart: local (m, S, keys) in, global out
  double* mref;               // [R] reference shift, identical on every rank
  float2* grad;               // [R][M][N] local normalised gradient partial in, global out (or nullptr)
  double* pay;                // [R][1 + 2 M N]
  unsigned long long* key;    // [R][3]: key_a, key_c, bits(m_r)
};

__device__ __forceinline__ void world_weights(const WorldArgs& a, int r, double& wS, double& wG, double& m) {
  const Red rr = a.red[r];
  m = rr.m;
  wS = wG = 0.0;
  if (a.mode == 0 || !(rr.S > 0.0) || !(rr.m > -INFINITY)) return;
  const double mr = a.mref[r];
  if (a.mode == 1) {
    wS = wG = exp(a.bp * (rr.m - mr)) * rr.S;
  } else {
    const double rho = rr.m / mr;
    wS = pow(rho, a.bp) * rr.S;
    wG = pow(rho, a.bp - 1.0) * pow(rr.S, 1.0 - 1.0 / a.bp);
  }
}

// Pack: grid (blocks, R); block (0, r) writes the scalars, every block a slice of the weighted gradient.
__global__ void __launch_bounds__(256) k_world_pack(WorldArgs a) {
  SQ_PDL_WAIT();
  const int r = blockIdx.y;
  double wS, wG, m;
  world_weights(a, r, wS, wG, m);
  const size_t n = a.with_grad ? (size_t)2 * a.M * a.N : 0, stride = 1 + n;
  double* p = a.pay + (size_t)r * stride;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p[0] = wS;
    const Red rr = a.red[r];
    a.key[3 * r] = rr.key_a;
    a.key[3 * r + 1] = rr.key_c;
    a.key[3 * r + 2] = (rr.m > 0.0) ? (unsigned long long)__double_as_longlong(rr.m) : 0ull;  // m >= 0: bits order
    if (!isfinite(wS) || !isfinite(wG)) p[0] = INFINITY;  // fp64 weight overflow (beta |m_r - m_ref| > ~700)
  }
  const float* g = reinterpret_cast<const float*>(a.grad) + (size_t)r * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[1 + i] = wG * (double)g[i];
}

// Unpack: the global record (m = m_ref, S = sum wS, max keys) and the normalised global gradient; block
// (0, r) then advances m_ref to the global maximum of the ranks' shifts for the next evaluation.
__global__ void __launch_bounds__(256) k_world_unpack(WorldArgs a, int* status) {
  SQ_PDL_WAIT();
  const int r = blockIdx.y;
  const size_t n = a.with_grad ? (size_t)2 * a.M * a.N : 0, stride = 1 + n;
  const double* p = a.pay + (size_t)r * stride;
  const double S = p[0];
  double norm = 0.0;
  if (a.mode != 0 && S > 0.0) norm = a.mode == 1 ? 1.0 / S : pow(S, 1.0 / a.bp - 1.0);
  float* g = reinterpret_cast<float*>(a.grad) + (size_t)r * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    g[i] = (float)(p[1 + i] * norm);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double mr = a.mref[r];
    Red rr;
    rr.m = (a.mode != 0 && S > 0.0) ? mr : -INFINITY;
    rr.S = a.mode != 0 ? S : 0.0;
    rr.key_a = a.key[3 * r];
    rr.key_c = a.key[3 * r + 1];
    rr.tie = rr.pad = 0u;  // (ties between ranks are not tracked)
    a.red[r] = rr;
    if (!isfinite(S)) atomicOr(status, ST_NONFINITE);
    const unsigned long long mb = a.key[3 * r + 2];
    if (mb && a.mode != 0) a.mref[r] = __longlong_as_double((long long)mb);
  }
}

// Reference shifts at create: 0 (LSE) or 1 (p-norm); v = w |A| / N is O(1).
__global__ void k_world_init(int R, int mode, double* mref) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) mref[r] = mode == 2 ? 1.0 : 0.0;
}

}  // namespace sq
