// Small kernels around the fused AF path: quantizer (a1), mainlobe (a6),
// deterministic partial combines (a5/a8), loss / metric finalization (a6),
// the sparse MAX-mode adjoint, the chain through Q_A (a8B), Adam and the two
// projections (a9).
#pragma once
#include <stdint.h>

#include "af_kernels.cuh"

namespace sq {

enum : int { ST_INVALID = 1, ST_DEGENERATE = 2, ST_NONFINITE = 4 };

struct Red {               // per restart, after combining all groups
  double m;                // shift of S and of the gradient partials
  double S;                // sum of phi at shift m
  unsigned long long key_a, key_c;
};

// ------------------------------------------------------------------ a1 quantizer
// fp64 table of the hard levels: lut[i*] = k with y_hard = k / B for i* = #{rho <= z}
// (Eq. 43 with the nearest-level snap of Q12; decision in fp64 like the oracle).
__global__ void k_hard_lut(int B, int BR, double c, const float* __restrict__ rho, int* __restrict__ lut,
                           int* __restrict__ status) {
  const int r = blockIdx.y;
  const float* rr = rho + (size_t)r * BR;
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
  extern __shared__ float rs[];
  constexpr int LPE = 8;
  const int r = blockIdx.y;
  const float* rr = rho + (size_t)r * BR;
  for (int i = threadIdx.x; i < BR; i += blockDim.x) rs[i] = rr[i];
  __syncthreads();
  const int sub = threadIdx.x & (LPE - 1);
  const int e0 = blockIdx.x * (blockDim.x / LPE) + threadIdx.x / LPE;
  const bool ok = e0 < MN;
  const size_t e = (size_t)r * MN + (ok ? e0 : 0);
  const float x = z[e];
  int lo = 0, hi = BR;
  while (lo < hi) { int mid = (lo + hi) >> 1; if (rs[mid] <= x) lo = mid + 1; else hi = mid; }
  const int cnt = lo;
  if (s_soft || dq) {
    const float W = 12.0f / c;
    lo = 0; hi = cnt;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (rs[mid] < x - W) lo = mid + 1; else hi = mid; }
    const int i0 = lo;
    lo = cnt; hi = BR;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (rs[mid] <= x + W) lo = mid + 1; else hi = mid; }
    const int i1 = lo;
    float resid = 0.f, sech = 0.f;
    for (int j = i0 + sub; j < i1; j += LPE) {
      const float u = c * (x - rs[j]);
      const float e2 = __expf(-2.f * fabsf(u));
      const float inv = __frcp_rn(1.f + e2);
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

// ------------------------------------------------------------------ a6 mainlobe
// c_m = sum_n s_m(n) conj(w_m(n)) = A_mm(0,0) (Eq. 38), fp64 fixed-order tree.
__global__ void k_mainlobe(int N, const float2* __restrict__ s, const float2* __restrict__ w, double2* cm) {
  __shared__ double sre[256], sim[256];
  const size_t row = blockIdx.x;
  double re = 0.0, im = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    const float2 a = s[row * N + n], b = w[row * N + n];
    re += (double)a.x * b.x + (double)a.y * b.y;
    im += (double)a.y * b.x - (double)a.x * b.y;
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
  if (threadIdx.x == 0) cm[row] = make_double2(sre[0], sim[0]);
}

// ------------------------------------------------------------------ combines
// Per restart: max keys, global shift and the rescaled sum S over the restart's groups
// [r * GPR, (r+1) * GPR) intersected with [g_lo, g_hi).  Block of 256, fixed order.
__global__ void k_reduce_groups(int GPR, int g_lo, int g_hi, int mode, double bp, Part part, Red* red) {
  __shared__ double sh[256];
  __shared__ unsigned long long ka[256], kc[256];
  const int r = blockIdx.x;
  const int lo = max(g_lo, r * GPR), hi = min(g_hi, (r + 1) * GPR);
  double mloc = -INFINITY;
  unsigned long long a = 0, cc = 0;
  for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    if (part.S[g] > 0.f) mloc = fmax(mloc, (double)part.m[g]);
    a = max(a, part.key[2 * g]);
    cc = max(cc, part.key[2 * g + 1]);
  }
  sh[threadIdx.x] = mloc;
  ka[threadIdx.x] = a;
  kc[threadIdx.x] = cc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
      ka[threadIdx.x] = max(ka[threadIdx.x], ka[threadIdx.x + o]);
      kc[threadIdx.x] = max(kc[threadIdx.x], kc[threadIdx.x + o]);
    }
    __syncthreads();
  }
  const double m = sh[0];
  __syncthreads();
  double S = 0.0;
  if (mode != 0 && m > -INFINITY) {
    for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
      const double Sg = part.S[g];
      if (Sg > 0.0) S += Sg * (mode == 1 ? exp(bp * ((double)part.m[g] - m)) : pow((double)part.m[g] / m, bp));
    }
  }
  sh[threadIdx.x] = S;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    red[r].m = m;
    red[r].S = sh[0];
    red[r].key_a = ka[0];
    red[r].key_c = kc[0];
  }
  // per-group rescale of the gradient partials to the restart's shift (used by the combine)
  if (part.scale && mode != 0) {
    for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
      float sc = 0.f;
      if (part.S[g] > 0.f && m > -INFINITY)
        sc = (float)(mode == 1 ? exp(bp * ((double)part.m[g] - m)) : pow((double)part.m[g] / m, bp - 1.0));
      part.scale[g] = sc;
    }
  }
}

// Multi-GPU: the shift m arrived from the all-reduce; refresh the per-group scales.
__global__ void k_group_scales(int GPR, int g_lo, int g_hi, int mode, double bp, Part part, const Red* red) {
  const int r = blockIdx.x;
  const int lo = max(g_lo, r * GPR), hi = min(g_hi, (r + 1) * GPR);
  const double m = red[r].m;
  for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    float sc = 0.f;
    if (part.S[g] > 0.f && m > -INFINITY)
      sc = (float)(mode == 1 ? exp(bp * ((double)part.m[g] - m)) : pow((double)part.m[g] / m, bp - 1.0));
    part.scale[g] = sc;
  }
}

// Unit slots -> per-row sums in true units of dL_wpsl / d(.)^*:
// out[ra][q] = norm_r * sum_k scale[u] slot[u][q],  u = ra K + k  (fixed order),
// norm_r = eps/(2N) * extra * (LSE: 1/S_r, PNORM: S_r^{1/p-1}).  Block: 32 q x 8 k-lanes.
__global__ void k_combine_rows(int M, int N, int K, int len, int slot_stride, int u_lo, int u_hi, int mode,
                               double bp, double eps, double extra, Part part, const Red* __restrict__ red,
                               float2* out) {
  __shared__ float2 sh[8][33];
  const int ra = blockIdx.y;
  const int r = ra / M;
  const int q = blockIdx.x * 32 + (threadIdx.x & 31);
  const int kl = threadIdx.x >> 5;  // 0..7
  const double S = red[r].S;
  const bool live = red[r].m > -INFINITY && S > 0.0;
  float re = 0.f, im = 0.f;
  if (live && q < len) {
    for (int k = kl; k < K; k += 8) {
      const int u = ra * K + k;
      if (u < u_lo || u >= u_hi) continue;
      const float sc = part.scale[u];
      const float2 v = part.g[(size_t)u * slot_stride + q];
      re = fmaf(sc, v.x, re);
      im = fmaf(sc, v.y, im);
    }
  }
  sh[kl][threadIdx.x & 31] = make_float2(re, im);
  __syncthreads();
  if (kl == 0 && q < len) {
    float2 t = sh[0][threadIdx.x];
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      t.x += sh[j][threadIdx.x].x;
      t.y += sh[j][threadIdx.x].y;
    }
    double norm = 0.0;
    if (live) {
      norm = eps / (2.0 * N) * extra;
      norm *= (mode == 1) ? 1.0 / S : pow(S, 1.0 / bp - 1.0);
    }
    out[(size_t)ra * len + q] = make_float2((float)(t.x * norm), (float)(t.y * norm));
  }
}

// ------------------------------------------------------------------ MAX-mode sparse adjoint
// Eq. 37's subgradient goes to the unique argmax cell (Q17): recompute A there by the O(N)
// correlation and write the whole red_grad[r] (zero elsewhere).
// wrt 1 (filters): dL/dw_l*^*(n) = conj(G) x_hat_{m*,k*}(n - tau*);
// wrt 2 (transmit): dL/ds_m*^*(n) = G e^{-j2pi n f/N} w_l*(n + tau*).
__global__ void k_sparse_adj(int M, int N, int K, int L, int wrt, double eps, const float* __restrict__ weights,
                             const float2* __restrict__ s, const float2* __restrict__ w,
                             const float2* __restrict__ dtw, const Red* __restrict__ red, float2* red_grad) {
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

// ------------------------------------------------------------------ a6 metrics / loss
__device__ __forceinline__ void decode_key(unsigned long long key, int M, int N, int K, int L, int32_t out[4],
                                           double* vsq) {
  if (key == 0ull) {
    out[0] = out[1] = out[2] = out[3] = -1;
    *vsq = 0.0;
    return;
  }
  const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
  out[3] = idx % K;
  out[2] = (int)((idx / K) % L) - (N - 1);
  out[1] = (idx / K / L) % M;
  out[0] = idx / K / L / M;
  *vsq = (double)__uint_as_float((uint32_t)(key >> 32));
}

struct MetricsOut {       // mirrors sqngd_metrics (include/sqngd.h)
  double loss, loss_wpsl, loss_snrl, wapsl, wcpsl, wpsl;
  int32_t argmax_auto[4], argmax_cross[4];
  uint32_t flags, n_cells;
};

__global__ void k_metrics(int M, int N, int K, int L, int mode, double bp, double eps, double ptar,
                          uint32_t n_cells, uint32_t flags, const Red* __restrict__ red,
                          const double2* __restrict__ cm, MetricsOut* out, double* p_out, double* loss_hist,
                          int hist_stride, int hist_col, int* status) {
  const int r = blockIdx.x;
  if (threadIdx.x != 0) return;
  MetricsOut o;
  double va, vc;
  decode_key(red[r].key_a, M, N, K, L, o.argmax_auto, &va);
  decode_key(red[r].key_c, M, N, K, L, o.argmax_cross, &vc);
  o.wapsl = sqrt(va) / N;
  o.wcpsl = sqrt(vc) / N;
  o.wpsl = fmax(o.wapsl, o.wcpsl);
  if (mode == 0) o.loss_wpsl = o.wpsl;
  else if (red[r].m > -INFINITY && red[r].S > 0.0)
    o.loss_wpsl = mode == 1 ? red[r].m + log(red[r].S) / bp : red[r].m * pow(red[r].S, 1.0 / bp);
  else o.loss_wpsl = 0.0;
  double lsn = 0.0;
  for (int m = 0; m < M; ++m) {
    const double2 c = cm[(size_t)r * M + m];
    const double p = sqrt(c.x * c.x + c.y * c.y) / N;
    if (p_out) p_out[(size_t)r * M + m] = p;
    if (p == 0.0) atomicOr(status, ST_DEGENERATE);
    lsn += (p - ptar) * (p - ptar);
  }
  o.loss_snrl = lsn / M;
  o.loss = eps * o.loss_wpsl + (1.0 - eps) * o.loss_snrl;
  o.flags = flags;
  o.n_cells = n_cells;
  if (!isfinite(o.loss)) atomicOr(status, ST_NONFINITE);
  if (out) out[r] = o;
  if (loss_hist) loss_hist[(size_t)r * hist_stride + hist_col] = o.loss;
}

// ------------------------------------------------------------------ finalize gradients
// Step A: grad_w = 2 (red_grad + conj(Gc_l) s_l)           (Q16)
// Step B: g = red_grad + Gc_m w_m = dL/ds^*; optional grad_s; dy = 4 pi Im(g conj(s)),
//         grad_z = dq * dy (Eqs. 23-24 chain).
// Gc_m = (1-eps)(2/M)(p_m - p_tar)/N * c_m / (2|c_m|)   (Eq. 41 on c_m = A_mm(0,0)).
__global__ void k_finalize_grad(int R, int M, int N, int wrt, double eps, double ptar,
                                const double2* __restrict__ cm, const float2* __restrict__ red_grad,
                                const float2* __restrict__ s, const float2* __restrict__ w,
                                const float* __restrict__ dq, float2* grad_w, float2* grad_s, float* dy,
                                float* grad_z, int* status) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)R * M * N) return;
  const size_t row = e / N;
  const int m = (int)(row % M);
  const double2 c = cm[row];
  const double mag = sqrt(c.x * c.x + c.y * c.y);
  double gr = 0.0, gi = 0.0;
  if (mag > 0.0) {
    const double f = (1.0 - eps) * (2.0 / M) * (mag / N - ptar) / N / (2.0 * mag);
    gr = f * c.x;
    gi = f * c.y;
  }
  (void)m;
  const float2 rg = red_grad[e];
  bool bad = false;
  if (wrt == 1) {
    const float2 sv = s[e];  // conj(Gc) s
    const float re = rg.x + (float)(gr * sv.x + gi * sv.y);
    const float im = rg.y + (float)(gr * sv.y - gi * sv.x);
    if (grad_w) grad_w[e] = make_float2(2.f * re, 2.f * im);
    bad = !isfinite(re) || !isfinite(im);
  } else {
    const float2 wv = w[e];  // Gc w
    const float re = rg.x + (float)(gr * wv.x - gi * wv.y);
    const float im = rg.y + (float)(gr * wv.y + gi * wv.x);
    if (grad_s) grad_s[e] = make_float2(re, im);
    const float2 sv = s[e];
    const float d = 4.f * 3.14159265358979f * (im * sv.x - re * sv.y);  // Im(g conj(s))
    if (dy) dy[e] = d;
    if (grad_z) grad_z[e] = dq[e] * d;
    bad = !isfinite(re) || !isfinite(im);
  }
  if (bad) atomicOr(status, ST_NONFINITE);
}

// dL/drho_i = -a c sum_e sech^2(c (z_e - rho_i)) dy_e, gathered per threshold over a chunk of
// elements (partials [R][nchunk][BR], then a fixed-order sum).  Culled outside |c(z - rho)| < 12.
__global__ void k_grad_rho_part(int MN, int BR, int chunk, float c, const float* __restrict__ z,
                                const float* __restrict__ rho, const float* __restrict__ dy, float* part) {
  __shared__ float zs[256], ds[256];  // chunk <= 256
  const int r = blockIdx.z;
  const int ch = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float ri = i < BR ? rho[(size_t)r * BR + i] : 0.f;
  const int e0 = ch * chunk, e1 = min(MN, e0 + chunk);
  float acc = 0.f;
  for (int base = e0; base < e1; base += 256) {
    __syncthreads();
    const int e = base + threadIdx.x;
    if (threadIdx.x < 256) {
      zs[threadIdx.x] = e < e1 ? z[(size_t)r * MN + e] : 1e30f;
      ds[threadIdx.x] = e < e1 ? dy[(size_t)r * MN + e] : 0.f;
    }
    __syncthreads();
    const int n = min(256, e1 - base);
    for (int q = 0; q < n; ++q) {
      const float u = c * (zs[q] - ri);
      if (fabsf(u) < 12.f) {
        const float e2 = __expf(-2.f * fabsf(u));
        const float inv = 1.f / (1.f + e2);
        acc += 4.f * e2 * inv * inv * ds[q];
      }
    }
  }
  if (i < BR) part[((size_t)r * gridDim.y + ch) * BR + i] = acc;
}

__global__ void k_grad_rho_sum(int BR, int nchunk, float coef, const float* __restrict__ part, float* grad_rho) {
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BR) return;
  float acc = 0.f;
  for (int ch = 0; ch < nchunk; ++ch) acc += part[((size_t)r * nchunk + ch) * BR + i];
  grad_rho[(size_t)r * BR + i] = coef * acc;
}

// ------------------------------------------------------------------ a9 optimizer
__global__ void k_adam(size_t n, float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, float lr, float b1, float b2, float eps, float c1, float c2,
                       const int* __restrict__ status) {
  if (*status & ST_NONFINITE) return;  // keep the last finite iterate
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = b1 * m[i] + (1.f - b1) * gi;
  const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  x[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
}

// Eq. 32: h_m <- sqrt(N / ||h_m||^2) h_m, one block per row, fp64 energy.
__global__ void k_project_w(int N, float2* w, int* status) {
  __shared__ double sh[256];
  if (*status & ST_NONFINITE) return;
  float2* row = w + (size_t)blockIdx.x * N;
  double e = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) e += (double)row[n].x * row[n].x + (double)row[n].y * row[n].y;
  sh[threadIdx.x] = e;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double en = sh[0];
  if (en == 0.0) {
    if (threadIdx.x == 0) atomicOr(status, ST_DEGENERATE);
    return;
  }
  const float sc = (float)sqrt((double)N / en);
  for (int n = threadIdx.x; n < N; n += blockDim.x) row[n] = make_float2(row[n].x * sc, row[n].y * sc);
}

// Threshold projection: sort ascending, clamp to [lo, hi], forward min-gap sweep.
// One block (1024 threads) per restart; BR <= 8192.
__global__ void k_project_rho(int BR, float* rho, float lo, float hi, float gap, const int* status) {
  extern __shared__ float sr[];
  __shared__ int flag;
  if (*status & ST_NONFINITE) return;
  float* p = rho + (size_t)blockIdx.x * BR;
  int n2 = 1;
  while (n2 < BR) n2 <<= 1;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n2; i += blockDim.x) sr[i] = i < BR ? p[i] : INFINITY;
  __syncthreads();
  for (int i = threadIdx.x; i + 1 < BR; i += blockDim.x)
    if (sr[i] > sr[i + 1]) flag = 1;
  __syncthreads();
  if (flag) {
    // nearly sorted (Adam moves each threshold by ~lr per step): odd-even transposition
    // rounds with early exit; a full bitonic sort only if that does not converge.
    __shared__ int swapped;
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
    } while (swapped && ++rounds < 64);
    if (swapped) {
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
    for (int i = threadIdx.x; i < BR; i += blockDim.x) q[i] = sr[i] - (float)i * gap;
    __syncthreads();
    for (int off = 1; off < BR; off <<= 1) {
      float tmp[8];
      int cnt = 0;
      for (int i = threadIdx.x; i < BR; i += blockDim.x) tmp[cnt++] = (i >= off) ? fmaxf(q[i], q[i - off]) : q[i];
      __syncthreads();
      cnt = 0;
      for (int i = threadIdx.x; i < BR; i += blockDim.x) q[i] = tmp[cnt++];
      __syncthreads();
    }
    for (int i = threadIdx.x; i < BR; i += blockDim.x) {
      const float qi = sr[i] - (float)i * gap;
      if (q[i] > qi) sr[i] = q[i] + (float)i * gap;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BR; i += blockDim.x) p[i] = sr[i];
}

}  // namespace sq
