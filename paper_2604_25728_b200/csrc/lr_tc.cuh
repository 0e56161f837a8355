// Forward-only Chebyshev contraction on the 5th-generation tensor cores (tcgen05 / TMEM), SURVEY §8(f)
// NEXT-1 (forward part: sqngd_af_forward, the MAX loss, the hard metrics):
//
//   At(tau, f_p) = Pe + Po,  At(tau, f_{K-1-p}) = Pe - Po,  Pe = sum_j alpha_j(p) E_j(tau),
//   Po = sum_j beta_j(p) O_j(tau)   (DESIGN.md §3 "Grid symmetry"; E, O from the exact node AFs)
//
// A CTA owns 128 lags of one (restart, channel, channel) pair and all K bins.  The node sums of its
// lags are staged once in shared memory as FP16 hi / lo parts in the canonical K-major layout (the
// 3-term split packed along K = 16, as in k_lrt: x_hi c_hi + x_lo c_hi + x_hi c_lo, with the per-lag
// power-of-two prescale); the Lagrange tables come pre-laid-out from the host, one 128-column image
// per 64 bin pairs: columns [A0 of the 64 pairs | A1 of the 64 pairs], i.e. B_E = [alpha | alpha],
// B_O = [beta | -beta].  One thread issues four kind::f16 MMAs per 64-pair chunk (M = 128, N = 128,
// K = 16): D_re = Er B_E + Or B_O, D_im = Ei B_E + Oi B_O, so the tensor core forms A0 and A1
// directly; the accumulators (256 TMEM columns) are read by 8 epilogue warps with tcgen05.ld
// (32 consecutive bins of one lag row per instruction), which run the same cell epilogue as k_lrt
// (keys with the lowest-bin tie rule, the LSE / p-norm sum, the optional |A| map -- one lag row per
// lane, so a warp's map store is 32 consecutive lags of one bin).  Two CTAs per SM (256 columns each).
//
// The adjoint stays on k_lrt (mma.sync): its products have N = 16 nodes, where one tcgen05 instruction
// costs ~100-145 cycles (profiles/r02_tcgen05_study.md).
#pragma once
#include <stdint.h>

#include "lr_kernels.cuh"

namespace sq {

namespace umma {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared-memory matrix descriptor: K-major, no swizzle, core matrices of 8 rows x 16 bytes
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;
}
// instruction descriptor, kind::f16: D f32, A / B f16, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// Wait for the phase of `bar` with the given parity to complete.  A watchdog traps after ~2^31 cycles
// (about a second) so a broken hand-off fails the launch loudly instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (1ll << 31)) asm volatile("trap;");
  }
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 consecutive fp32 columns of this lane's TMEM row
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
}  // namespace umma

// Byte offset of element (row, k) in a canonical K-major, no-swizzle image with K = 16 fp16 columns:
// core matrices of 8 rows x 16 B, LBO = 128 B along K, SBO = 256 B along the rows.
__host__ __device__ constexpr uint32_t lrf_off(int row, int k) {
  return (uint32_t)((row & 7) * 16 + (row >> 3) * 256 + (k >> 3) * 128 + (k & 7) * 2);
}
constexpr int kLrfRows = 128;       // lags per CTA (M of the MMA, TMEM lanes)
constexpr int kLrfPairs = 32;       // bin pairs per MMA chunk (N = 64: A0 and A1 columns)
constexpr int kLrfImg = 4096;       // bytes of one 128-row x 16 fp16 A image
constexpr int kLrfImgB = 2048;      // bytes of one 64-row x 16 fp16 B image (one chunk)
constexpr int kLrfThreads = 256;    // 8 epilogue warps (two per TMEM lane quarter)

struct LrfArgs {
  int M, N, L, K, Kp, Q, nc, npc, row0;  // nc: 128-lag chunks per pair; npc: 64-pair MMA chunks
  int tau_lo, tau_hi, excl0, LS, mld;
  float bp, invN;
  const float* weights;  // [K][L] or nullptr
  const float* wmax;     // [L]
  const float* coefm;    // [Q/2] middle-bin coefficients (odd K)
  const uint4* tabB;     // [npc][2][kLrfImgB / 16]: B_E, B_O images per chunk
  const float2* Rn;      // [R M M][Q][LS] node AFs
  float* af_mag;         // [R][M][M][K][mld] or nullptr
  Part part;             // unit slots, u = pair nc + chunk
  LrRed* lred;           // [R]
};

inline size_t lrf_smem_bytes(int npc, int QH) {
  return (size_t)4 * kLrfImg + (size_t)npc * 2 * kLrfImgB + (size_t)kLrfRows * QH * sizeof(float2) + 1024;
}

template <int LM, bool HW, bool MAP>
__global__ void __launch_bounds__(kLrfThreads, 2) k_lrf(const LrfArgs a) {
  SQ_PDL_WAIT();
  extern __shared__ __align__(1024) uint8_t lrf_smem[];
  // 1 KiB-aligned base for the UMMA images
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lrf_smem) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                              // Er, Ei, Or, Oi images
  uint8_t* sB = sm + 4 * kLrfImg;                // npc x (B_E, B_O)
  float2* sE = reinterpret_cast<float2*>(sB + (size_t)a.npc * 2 * kLrfImgB);  // [128][QH] fp32 E (middle bin)
  __shared__ uint64_t full[2], empty[2];  // TMEM double buffer: MMA -> epilogue, epilogue warps -> MMA
  __shared__ uint32_t tbase;
  __shared__ float s_isc[kLrfRows], s_shift[kLrfRows];
  __shared__ int s_valid[kLrfRows];
  __shared__ unsigned long long s_key[kLrfThreads / 32];
  __shared__ float s_red[kLrfThreads / 32];
  __shared__ int s_bad;
  const int QH = a.Q / 2;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int lq = wp & 3, half = wp >> 2;  // TMEM lane quarter; 0: A0 columns, 1: A1 columns
  const int ch = blockIdx.x;
  const int rm = a.row0 + (int)blockIdx.z;
  const int l = blockIdx.y;
  const int M = a.M;
  const int pr = rm * M + l;
  const int r = rm / M, m = rm - (rm / M) * M;
  const bool is_auto = m == l;
  const int u = pr * a.nc + ch;
  const float lb = a.bp * 1.4426950408889634f;

  // ---- staging: node sums of this CTA's lags (two threads per lag row: E images and row constants,
  // O images), FP16 split images in the canonical layout, per-row constants
  {
    const int row = tid & (kLrfRows - 1), part = tid >> 7, idx = ch * kLrfRows + row;
    const bool inL = idx < a.L;
    const float2* Rp = a.Rn + (size_t)pr * a.Q * a.LS + idx;
    float2 xq[10];  // Q <= 10 (F16 split): every node load in flight at once
#pragma unroll
    for (int q = 0; q < 10; ++q) xq[q] = (q < a.Q && inL) ? __ldg(Rp + (size_t)q * a.LS) : make_float2(0.f, 0.f);
    float nm2 = 0.f;
#pragma unroll
    for (int q = 0; q < 10; ++q) nm2 = fmaxf(nm2, fmaf(xq[q].x, xq[q].x, xq[q].y * xq[q].y));
    int ex = 0;  // per-lag power-of-two prescale: 2 max_q |R_q| -> <= 8192 (k_lrt)
    if (nm2 > 0.f) {
      const float t = 8192.f / (2.f * sqrtf(nm2));
      ex = (int)((__float_as_uint(t) >> 23) & 0xFFu) - 127;
      ex = ex < -100 ? -100 : (ex > 100 ? 100 : ex);
    }
    const float sc = __uint_as_float((uint32_t)(127 + ex) << 23);
    if (part == 0) {
      s_isc[row] = __uint_as_float((uint32_t)(127 - ex) << 23);
      const int tau = idx - (a.N - 1);
      const bool valid = inL && tau >= a.tau_lo && tau <= a.tau_hi && !(is_auto && a.excl0 && tau == 0);
      s_valid[row] = valid ? 1 : 0;
      const float wm = HW ? (inL ? __ldg(a.wmax + idx) : 0.f) : 1.f;
      float shift = 0.f;
      if (LM == 1) shift = sqrtf(nm2) * a.invN * wm + 40.f / a.bp;
      if (LM == 2) shift = fmaxf(sqrtf(nm2) * a.invN * wm, 1e-30f);
      s_shift[row] = shift;
    }
    uint16_t im[2][16];
#pragma unroll
    for (int mtx = 0; mtx < 2; ++mtx)
#pragma unroll
      for (int k = 0; k < 16; ++k) im[mtx][k] = 0;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      if (j >= QH) break;
      const float2 xa = xq[j];
      float2 xb = xq[0];  // x[Q - 1 - j] (Q <= 10, compile-time selects)
#pragma unroll
      for (int q = 1; q < 10; ++q) xb = (q == a.Q - 1 - j) ? xq[q] : xb;
      const float2 v = part == 0 ? make_float2(xa.x + xb.x, xa.y + xb.y) : make_float2(xa.x - xb.x, xa.y - xb.y);
      if (part == 0) sE[row * QH + j] = v;  // unscaled fp32 E (middle bin)
      const float vv[2] = {v.x * sc, v.y * sc};
#pragma unroll
      for (int mtx = 0; mtx < 2; ++mtx) {
        const __half h = __float2half_rn(vv[mtx]);
        const __half lo = __float2half_rn(vv[mtx] - __half2float(h));
        im[mtx][j] = __half_as_ushort(h);
        im[mtx][5 + j] = __half_as_ushort(lo);
        im[mtx][10 + j] = __half_as_ushort(h);
      }
    }
#pragma unroll
    for (int mtx = 0; mtx < 2; ++mtx)
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        uint4 v;
        v.x = (uint32_t)im[mtx][8 * kb + 0] | ((uint32_t)im[mtx][8 * kb + 1] << 16);
        v.y = (uint32_t)im[mtx][8 * kb + 2] | ((uint32_t)im[mtx][8 * kb + 3] << 16);
        v.z = (uint32_t)im[mtx][8 * kb + 4] | ((uint32_t)im[mtx][8 * kb + 5] << 16);
        v.w = (uint32_t)im[mtx][8 * kb + 6] | ((uint32_t)im[mtx][8 * kb + 7] << 16);
        *reinterpret_cast<uint4*>(sA + (2 * part + mtx) * kLrfImg + lrf_off(row, 8 * kb)) = v;
      }
  }
  {  // the B images of every chunk (static tables)
    const int n16 = a.npc * 2 * (kLrfImgB / 16);
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (int i = tid; i < n16; i += kLrfThreads) dst[i] = __ldg(a.tabB + i);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core reads
  if (wp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(umma::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    umma::mbar_init(&full[0], 1);
    umma::mbar_init(&full[1], 1);
    umma::mbar_init(&empty[0], kLrfThreads / 32);
    umma::mbar_init(&empty[1], kLrfThreads / 32);
    s_bad = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tb = tbase;

  // ---- per-thread row state
  const int row = 32 * lq + lane, idx = ch * kLrfRows + row;
  const bool inL = idx < a.L;
  const bool valid = s_valid[row] != 0;
  const float isc = s_isc[row];
  float shift = s_shift[row];
  float* mrow = (MAP && a.af_mag && inL) ? a.af_mag + (size_t)pr * a.K * a.mld + idx : nullptr;
  const uint32_t idesc = umma::idesc_f16(128, 2 * kLrfPairs);
  const uint32_t aE_r = umma::smem_u32(sA), aE_i = aE_r + kLrfImg, aO_r = aE_r + 2 * kLrfImg,
                 aO_i = aE_r + 3 * kLrfImg;
  // TMEM buffer b (128 columns): re [A0 | A1] at 128 b + [0, 64), im at 128 b + [64, 128)
  auto issue = [&](int c, int n) {  // chunk c into TMEM buffer n & 1 (n: issue count, continues over passes)
    const int b = n & 1;
    const uint32_t bE = umma::smem_u32(sB) + (uint32_t)(2 * c) * kLrfImgB, bO = bE + kLrfImgB;
    const uint32_t d = tb + 128u * b;
    umma::mma_f16(d, umma::desc(aE_r, 128, 256), umma::desc(bE, 128, 256), idesc, 0);
    umma::mma_f16(d, umma::desc(aO_r, 128, 256), umma::desc(bO, 128, 256), idesc, 1);
    umma::mma_f16(d + 64, umma::desc(aE_i, 128, 256), umma::desc(bE, 128, 256), idesc, 0);
    umma::mma_f16(d + 64, umma::desc(aO_i, 128, 256), umma::desc(bO, 128, 256), idesc, 1);
    umma::commit(&full[b]);
  };
  float best = -1.f, S = 0.f;
  int bk = 0;
  int nissued = 0, nconsumed = 0;  // chunk counters across passes (mbarrier phases)
  for (int pass = 0; pass < 2; ++pass) {
    const float lbN = lb * a.invN * isc;
    const float nlbs = valid ? -lb * shift : -INFINITY;
    const float qN = valid ? a.invN / shift * isc : 0.f;
    best = -1.f;
    bk = 0;
    S = 0.f;
    // one Doppler cell (a5): key value, LSE / p-norm term, optional map; H = 1: the A1 half (bins
    // descend with the pair index, so ties keep the later pair, i.e. the lower bin)
    auto cell = [&](float re, float im, int k, float& bv) {
      const float a2 = fmaf(re, re, fmaf(im, im, 1e-30f));
      float wt = 1.f, kv = a2;
      if (HW) {
        wt = valid ? __ldg(a.weights + (size_t)k * a.L + idx) : 0.f;
        kv = wt > 0.f ? a2 * wt * wt : -1.f;
      }
      bv = kv;
      if (LM == 0) {
        if (MAP && mrow && pass == 0) mrow[(size_t)k * a.mld] = sqrtf(a2) * isc;
        return;
      }
      const float rsq = rsqa(a2);
      const float mag = a2 * rsq;
      if (MAP && mrow && pass == 0) mrow[(size_t)k * a.mld] = mag * isc;
      float phi;
      if (LM == 1) {
        phi = ex2a(fmaf(lbN, HW ? wt * mag : mag, nlbs));
        if (HW) phi = wt > 0.f ? phi : 0.f;
      } else {
        const float q = (HW ? wt * mag : mag) * qN;
        phi = ex2a((a.bp - 1.f) * lg2a(q)) * q;
      }
      S += phi;
    };
    auto block = [&](auto hc, const float (&re)[32], const float (&imv)[32], int p0) {
      constexpr int H = decltype(hc)::value;
      const int nv = min(32, a.Kp - p0);
      float bb = -1.f;
      int bi = 0;
      if (nv == 32) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float kv;
          cell(re[i], imv[i], H ? a.K - 1 - p0 - i : p0 + i, kv);
          const bool upd = H ? (kv >= bb) : (kv > bb);
          bb = upd ? kv : bb;
          bi = upd ? i : bi;
        }
      } else {  // the last, partial chunk (predicated, indices stay compile-time: re / imv in registers)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i >= nv) break;
          float kv;
          cell(re[i], imv[i], H ? a.K - 1 - p0 - i : p0 + i, kv);
          const bool upd = H ? (kv >= bb) : (kv > bb);
          bb = upd ? kv : bb;
          bi = upd ? i : bi;
        }
      }
      // blocks run in pair order: A0 bins ascend (keep the first max), A1 bins descend (keep the last)
      const bool upd = H ? (bb >= best) : (bb > best);
      if (upd && nv > 0) {
        best = bb;
        bk = H ? a.K - 1 - p0 - bi : p0 + bi;
      }
    };
    if (wp == 0) {  // the first two chunks of this pass (warp 0 reconverges before its tcgen05.ld)
      if (lane == 0)
        for (int c = 0; c < 2 && c < a.npc; ++c) {
          const int n = nissued;
          if (n >= 2) umma::mbar_wait(&empty[n & 1], ((n >> 1) - 1) & 1);
          umma::fence_after();
          issue(c, n);
          ++nissued;
        }
      __syncwarp();
    }
    for (int c = 0; c < a.npc; ++c) {
      const int n = nconsumed++;
      umma::mbar_wait(&full[n & 1], (n >> 1) & 1);
      umma::fence_after();
      float re[32], imv[32];
      const uint32_t ta = tb + ((uint32_t)(32 * lq) << 16) + 128u * (n & 1) + (uint32_t)(half * kLrfPairs);
      umma::ld32(ta, re);
      umma::ld32(ta + 64, imv);
      umma::ld_wait();
      umma::fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(&empty[n & 1])) : "memory");
      if (wp == 0 && c + 2 < a.npc) {  // refill the buffer just released, once every warp has read it
        if (lane == 0) {
          const int ni = nissued;
          umma::mbar_wait(&empty[ni & 1], ((ni >> 1) - 1) & 1);
          umma::fence_after();
          issue(c + 2, ni);
        }
        ++nissued;
        __syncwarp();
      }
      const int p0 = c * kLrfPairs;
      if (half) block(std::integral_constant<int, 1>{}, re, imv, p0);
      else block(std::integral_constant<int, 0>{}, re, imv, p0);
    }
    // middle bin of an odd K (beta = 0): At = sum_j alpha_j E_j in fp32 from the unscaled node sums
    if ((a.K & 1) && half == 0) {
      float xr = 0.f, xi = 0.f;
      for (int j = 0; j < QH; ++j) {
        const float cj = __ldg(a.coefm + j);
        const float2 e = sE[row * QH + j];
        xr = fmaf(cj, e.x, xr);
        xi = fmaf(cj, e.y, xi);
      }
      float kv;
      cell(xr / isc, xi / isc, a.Kp, kv);  // (the prescaled value, as the other cells)
      if (kv > best) { best = kv; bk = a.Kp; }
    }
    if (LM == 0) break;
    // a row whose largest cell exceeds its node-based shift by too much redoes its sums at the exact max
    // (the two halves of a row see different cells: combine through shared memory)
    {
      const float vb = sqrtf(fmaxf(best, 0.f)) * isc * a.invN;
      const bool bd = valid && (LM == 1 ? lb * (vb - shift) > 96.f : (vb > shift && (a.bp * log2f(vb / shift)) > 96.f));
      if (bd) {
        atomicMax(reinterpret_cast<unsigned int*>(&s_shift[row]), __float_as_uint(vb));  // (positive floats)
        s_bad = 1;
      }
    }
    __syncthreads();
    const int any_bad = s_bad;
    if (!any_bad || pass == 1) break;
    shift = s_shift[row];
  }

  // ---- unit reduction: key (max over the CTA), shift m_u = max valid row shift, S rescaled to it
  unsigned long long key = 0ull;
  {
    const float bu = best * isc * isc;  // exact: sigma is a power of two
    const uint32_t cell = ((uint32_t)((m * M + l) * a.L + idx)) * (uint32_t)a.K + (uint32_t)bk;
    key = (valid && best >= 0.f) ? pack_key(bu, cell) : 0ull;
  }
  uint32_t tv = 0u;  // SQNGD_FLAG_TIE (ties between lanes and between warps of the unit)
  key = warp_key_max_tie(key, tv);
  if (lane == 0) s_key[wp] = key;
  if (lane == 0 && tv) atomicMax(is_auto ? &a.lred[r].tie_a : &a.lred[r].tie_c, tv);
  float mw = 0.f;
  if (LM != 0) {
    mw = valid ? shift : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    if (lane == 0) s_red[wp] = mw;
  }
  __syncthreads();
  if (LM != 0) {
    mw = s_red[0];
    for (int w = 1; w < kLrfThreads / 32; ++w) mw = fmaxf(mw, s_red[w]);
  }
  float Su = 0.f;
  if (LM != 0 && valid) {
    float fS, fG;
    lr_rescale<LM == 0 ? 1 : LM>(shift, mw, lb, a.bp, fS, fG);
    Su = S * fS;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Su += __shfl_xor_sync(0xffffffffu, Su, o);
  __syncthreads();  // (s_red reused for the sums)
  if (lane == 0) s_red[wp] = Su;
  umma::fence_before();
  __syncthreads();
  if (tid == 0) {
    unsigned long long kk = s_key[0];
    float St = s_red[0];
    uint32_t tw = 0u;
    for (int w = 1; w < kLrfThreads / 32; ++w) {
      if (s_key[w] && kk && (s_key[w] >> 32) == (kk >> 32) && s_key[w] != kk) tw = max(tw, (uint32_t)(kk >> 32) + 1u);
      kk = s_key[w] > kk ? s_key[w] : kk;
      St += s_red[w];
    }
    if (tw) atomicMax(is_auto ? &a.lred[r].tie_a : &a.lred[r].tie_c, tw);
    a.part.key[2 * (size_t)u] = is_auto ? kk : 0ull;
    a.part.key[2 * (size_t)u + 1] = is_auto ? 0ull : kk;
    a.part.m[u] = mw;
    a.part.S[u] = St;
    if (kk) atomicMax(is_auto ? &a.lred[r].key_a : &a.lred[r].key_c, kk);
    if (LM != 0 && mw > 0.f) atomicMax(&a.lred[r].mbits, __float_as_uint(mw));
  }
  if (wp == 0) {
    umma::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
  }
}

}  // namespace sq
