// Definitions shared by the fused kernels and the small kernels: status bits, MUFU helpers,
// Adam parameters, the per-restart reduction record and metrics (a6), block reductions.
#pragma once
#include <stdint.h>

#include "adam.cuh"

namespace sq {


__device__ __forceinline__ float ex2a_m(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_m(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


struct Red {               // per restart, after combining all groups
  double m;                // shift of S and of the gradient partials
  double S;                // sum of phi at shift m
  unsigned long long key_a, key_c;
  uint32_t tie, pad;       // tie: SQNGD_FLAG_TIE of this restart's maxima (0 after a multi-GPU combine)
};

// The packed key with its index part un-inverted: the max over these gives the HIGHEST index among
// the keys of the maximal value, the max over the keys themselves the lowest -- two different indices
// of one value mean a tie between two slots (SQNGD_FLAG_TIE).
__device__ __forceinline__ unsigned long long key_hi_index(unsigned long long k) {
  return k ? ((k & 0xFFFFFFFF00000000ull) | (~k & 0xFFFFFFFFull)) : 0ull;
}
// Tie of a category's maximum: between two slots (lowest-index key k vs highest-index key kh of the
// same value) or inside one (tv: 1 + the float bits of the largest value at which a unit saw two of its
// cells tie; 0: none).
__device__ __forceinline__ bool key_tied(unsigned long long k, unsigned long long kh, uint32_t tv) {
  if (!k) return false;
  const uint32_t v = (uint32_t)(k >> 32);
  return ((uint32_t)(kh >> 32) == v && kh != key_hi_index(k)) || tv == v + 1u;
}


struct Part {                // one slot per unit u = (r * M + a) * K + k
  unsigned long long* key;  // [U][2]  (auto, cross)
  float* m;                 // [U] shift of the unit's sums
  float* S;                 // [U] sum of phi (LSE: e^{b(v-m)}, PNORM: (v/m)^p)
  float* scale;             // [U] rescale to the restart's global shift (combine)
  float2* g;                // [U][P] adjoint partial: Step B time domain (N used), Step A spectral
};

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
  double apslr_db, cpslr_db, pslr_db;  // Eq. 48 of WAPSL, WCPSL, WPSL
  double snrl_db_max;                  // max_m Eq. 10 (k_snrl; NaN where not computed)
};

struct MetricsArgs {
  int M, N, K, L, mode;
  double bp, eps, ptar;
  uint32_t n_cells, flags;
  const Red* red;
  const double2* cm;
  MetricsOut* out;
  double* p_out;
  double* loss_hist;
  int hist_stride, hist_col;
  const double* snrl_in;  // [R] max_m SNRL_m (k_snrl) for the record, or nullptr (NaN in the record)
  int tie_scan;           // 1: compute SQNGD_FLAG_TIE (a record the caller reads); 0: flag left clear
};

// Eqs. 7-10, 37-42 for restart r from the combined partials.  Called by one whole warp
// (all 32 lanes): lane m computes p_m (Eq. 38) for m = lane, lane + 32, ...; the fixed-order
// xor-shuffle sum of (p_m - p_tar)^2 is deterministic; lane 0 writes the record.
__device__ void metrics_warp(const MetricsArgs& a, int r, int* status) {
  const int lane = threadIdx.x & 31;
  double lsn = 0.0;
  for (int m = lane; m < a.M; m += 32) {
    const double2 c = a.cm[(size_t)r * a.M + m];
    const double p = sqrt(c.x * c.x + c.y * c.y) / a.N;
    if (a.p_out) a.p_out[(size_t)r * a.M + m] = p;
    if (p == 0.0) atomicOr(status, ST_DEGENERATE);
    lsn += (p - a.ptar) * (p - a.ptar);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsn += __shfl_xor_sync(0xffffffffu, lsn, o);
  if (lane != 0) return;
  MetricsOut o;
  double va, vc;
  const Red rr = a.red[r];
  decode_key(rr.key_a, a.M, a.N, a.K, a.L, o.argmax_auto, &va);
  decode_key(rr.key_c, a.M, a.N, a.K, a.L, o.argmax_cross, &vc);
  o.wapsl = sqrt(va) / a.N;
  o.wcpsl = sqrt(vc) / a.N;
  o.wpsl = fmax(o.wapsl, o.wcpsl);
  if (a.mode == 0) o.loss_wpsl = o.wpsl;
  else if (rr.m > -INFINITY && rr.S > 0.0)
    o.loss_wpsl = a.mode == 1 ? rr.m + log(rr.S) / a.bp : rr.m * exp(log(rr.S) / a.bp);
  else o.loss_wpsl = 0.0;
  o.loss_snrl = lsn / a.M;
  o.loss = a.eps * o.loss_wpsl + (1.0 - a.eps) * o.loss_snrl;
  o.flags = a.flags | (rr.tie ? 2u : 0u);  // 2 = SQNGD_FLAG_TIE
  o.n_cells = a.n_cells;
  // Eq. 48: PSLR = 20 log10(PSL / N); the maxima above are already normalised by N (Q5)
  o.apslr_db = 20.0 * log10(o.wapsl);
  o.cpslr_db = 20.0 * log10(o.wcpsl);
  o.pslr_db = 20.0 * log10(o.wpsl);
  o.snrl_db_max = a.snrl_in ? a.snrl_in[r] : __longlong_as_double(0x7ff8000000000000ll);
  if (!isfinite(o.loss)) atomicOr(status, ST_NONFINITE);
  if (a.out) a.out[r] = o;
  if (a.loss_hist) a.loss_hist[(size_t)r * a.hist_stride + a.hist_col] = o.loss;
}

// Block-wide fixed-order reductions (warp shuffles, then the warps in index order).
template <class T_, class Op>
__device__ __forceinline__ T_ block_reduce(T_ x, Op op, T_* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = x;
  __syncthreads();
  x = sh[0];
  for (int i = 1; i < nw; ++i) x = op(x, sh[i]);
  return x;
}

// Per restart r: max keys, global shift and the rescaled sum S over the restart's units
// [r * GPR, (r+1) * GPR) intersected with [g_lo, g_hi); per-unit rescale factors for the
// gradient combine; the metrics.  Called by a whole block (fixed order, deterministic).
// Partials are read with ld.global.cg: in the fused kernel's last CTA they were written by
// other SMs in the same launch.
__device__ void reduce_restart(int r, int GPR, int g_lo, int g_hi, int mode, double bp, Part part, Red* red,
                               const MetricsArgs& ma, int* status, double* shd, unsigned long long* shk,
                               const uint32_t* tiew) {
  const int lo = max(g_lo, r * GPR), hi = min(g_hi, (r + 1) * GPR);
  double mloc = -INFINITY;
  unsigned long long a = 0, cc = 0, ah = 0, ch = 0;  // ah, ch: highest-index keys (ties, SQNGD_FLAG_TIE)
  for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    if (__ldcg(part.S + g) > 0.f) mloc = fmax(mloc, (double)__ldcg(part.m + g));
    const unsigned long long ka = __ldcg(part.key + 2 * g), kc = __ldcg(part.key + 2 * g + 1);
    a = max(a, ka);
    cc = max(cc, kc);
    if (ma.tie_scan) {
      ah = max(ah, key_hi_index(ka));
      ch = max(ch, key_hi_index(kc));
    }
  }
  auto dmax = [](double x, double y) { return fmax(x, y); };
  auto umax = [](unsigned long long x, unsigned long long y) { return x > y ? x : y; };
  const double m = block_reduce(mloc, dmax, shd);
  a = block_reduce(a, umax, shk);
  cc = block_reduce(cc, umax, shk);
  if (ma.tie_scan) {  // (uniform)
    ah = block_reduce(ah, umax, shk);
    ch = block_reduce(ch, umax, shk);
  }
  double S = 0.0;
  const float mf = (float)m;
  const float lb = (float)(bp * 1.4426950408889634);
  for (int g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    float sc = 0.f;
    const float Sg = __ldcg(part.S + g);
    if (mode != 0 && Sg > 0.f && m > -INFINITY) {
      const float mg = __ldcg(part.m + g);
      sc = mode == 1 ? exp2f(lb * (mg - mf)) : exp2f((float)(bp - 1.0) * log2f(mg / mf));
      S += (double)Sg * (mode == 1 ? sc : sc * (mg / mf));
    }
    if (part.scale) part.scale[g] = sc;
  }
  auto dsum = [](double x, double y) { return x + y; };
  S = block_reduce(S, dsum, shd);
  if (threadIdx.x == 0) {
    red[r].m = m;
    red[r].S = S;
    red[r].key_a = a;
    red[r].key_c = cc;
    red[r].tie = ma.tie_scan && (key_tied(a, ah, tiew ? tiew[2 * r] : 0u) || key_tied(cc, ch, tiew ? tiew[2 * r + 1] : 0u) ||
                  (a && (a >> 32) == (cc >> 32))) ? 1u : 0u;
  }
  __syncthreads();
  if (threadIdx.x < 32 && (ma.out || ma.loss_hist || ma.p_out)) metrics_warp(ma, r, status);
  __syncthreads();
}

}  // namespace sq
