// In-CTA complex FFTs for sm_100a: registers + swizzled shared memory.
//
// The paper's Eq. 36 evaluates every Doppler bin's aperiodic
// correlation as IFFT(FFT(x_pad) . conj(FFT(h_pad))).  Here one FFT of length P
// (power of two, P >= 2N-1, Q23) is carried by a *group* of T = P/E threads; each
// thread owns E elements in "strided ownership": v[i] <-> element t + i*T.
//
// A transform is a sequence of Stockham autosort passes (radix E, the last one
// radix P / E^(passes-1)).  Pass p (span Ns = E^p) takes butterfly j's inputs
// x[j + r P/R], multiplies by W^{(j mod Ns) r / (Ns R)}, does an R-point DFT in
// registers and writes y[(j/Ns) Ns R + (j mod Ns) + r Ns].  With the strided
// ownership the first pass reads registers and the last pass writes registers,
// so a P-point transform costs (passes - 1) shared-memory exchanges and the
// output lands in the same strided ownership as the input: an IFFT can follow an
// FFT (or an epilogue + FFT can follow an IFFT) with no extra data movement.
//
// Shared-memory addresses are padded (one float2 after every 16: i + i/16) so that
// every write pattern (stride-R for the first pass, contiguous afterwards) and
// every strided read is bank-conflict free for 64-bit accesses, and the unrolled
// offsets stay compile-time constants.  Exchanges double-buffer (two padded
// P-element buffers) so one barrier per exchange.
// Stockham twiddles come from a per-P table in global memory (L1-resident,
// [pass][r-1][j mod Ns] so a warp's loads coalesce), built in fp64 on the host.
#pragma once
#include <cuda_runtime.h>
#include <type_traits>

namespace sq {

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

template <int I, int N, class Fn>
__device__ __forceinline__ void static_for(Fn&& fn) {
  if constexpr (I < N) {
    fn(std::integral_constant<int, I>{});
    static_for<I + 1, N>(fn);
  }
}

// Packed FP32 pairs (PTX .f32x2, sm_100a FADD2 / FMUL2 / FFMA2): one issue slot for the same
// operation on two lanes' values.  Measured on B200 (tools/ubench_ffma2.cu): FFMA2 runs at the FP32
// pipe's lane rate (127 lane-FMA/clk/SM, as scalar FFMA), so it does not raise the FP32 peak; it
// halves the issue slots of the FP32 work (the k_lrt epilogue and the FFT kernels are issue-bound,
// DESIGN.md §6).  Each lane is an IEEE fp32 operation with round-to-nearest, as the scalar op.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 v) {
  float a;
  asm("mov.b64 {%0, _}, %1;" : "=f"(a) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi2(f32x2 v) {
  float b;
  asm("mov.b64 {_, %0}, %1;" : "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

#ifndef SQNGD_CPACKED
#define SQNGD_CPACKED 1
#endif
__device__ __forceinline__ f32x2 f2p(float2 a) { return pk2(a.x, a.y); }
__device__ __forceinline__ float2 p2f(f32x2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// Complex arithmetic on (re, im) pairs.  Packed: an add is one FADD2; a product is one FMUL2 and one FFMA2
//   a b = (a.x, a.y) b.x + (-a.y, a.x) b.y,   a conj(b) = (a.x, a.y) b.x + (a.y, -a.x) b.y
// (ptxas folds the swap, the one-sided negation and the broadcasts of b.x / b.y into operand modifiers).
template <bool PK>
__device__ __forceinline__ float2 cadd_p(float2 a, float2 b) {
  if (PK) return p2f(add2(f2p(a), f2p(b)));
  return make_float2(a.x + b.x, a.y + b.y);
}
template <bool PK>
__device__ __forceinline__ float2 csub_p(float2 a, float2 b) {
  if (PK) return p2f(sub2(f2p(a), f2p(b)));
  return make_float2(a.x - b.x, a.y - b.y);
}
template <bool PK>
__device__ __forceinline__ float2 cmul_p(float2 a, float2 b) {
  if (PK) return p2f(fma2(pk2(-a.y, a.x), pk2(b.y, b.y), mul2(f2p(a), pk2(b.x, b.x))));
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
template <bool PK>
__device__ __forceinline__ float2 cmulc_p(float2 a, float2 b) {
  if (PK) return p2f(fma2(pk2(a.y, -a.x), pk2(b.y, b.y), mul2(f2p(a), pk2(b.x, b.x))));
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return cadd_p<SQNGD_CPACKED>(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return csub_p<SQNGD_CPACKED>(a, b); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return cmul_p<SQNGD_CPACKED>(a, b); }
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return cmulc_p<SQNGD_CPACKED>(a, b); }

// cos(2 pi i / 64), i = 0..16, to full float precision (first quadrant).
__host__ __device__ constexpr double kCos64(int i) {
  constexpr double t[17] = {1.0,
                            0.99518472667219688624,
                            0.98078528040323044913,
                            0.95694033573220886494,
                            0.92387953251128675613,
                            0.88192126434835502971,
                            0.83146961230254523708,
                            0.77301045336273696081,
                            0.70710678118654752440,
                            0.63439328416364549822,
                            0.55557023301960222474,
                            0.47139673682599764856,
                            0.38268343236508977173,
                            0.29028467725446236764,
                            0.19509032201612826785,
                            0.09801714032956060199,
                            0.0};
  return t[i];
}
// cos / sin of 2 pi k / 64 for any k (exact table symmetries).
__host__ __device__ constexpr double cos64(int k) {
  k &= 63;
  return k <= 16 ? kCos64(k) : k <= 32 ? -kCos64(32 - k) : k <= 48 ? -kCos64(k - 32) : kCos64(64 - k);
}
__host__ __device__ constexpr double sin64(int k) { return cos64(k - 16); }

// x * W_R^{DIR*k}, W_R = e^{2 pi i / R}; DIR = -1 forward transform.
template <int R, int DIR, int k, bool PK = SQNGD_CPACKED>
__device__ __forceinline__ float2 twc(float2 x) {
  constexpr int kk = ((k % R) + R) % R;
  constexpr int q = kk * (64 / R);  // angle in units of 2 pi / 64
  if constexpr (kk == 0) {
    return x;
  } else if constexpr (q == 16) {  // i^DIR
    return DIR < 0 ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  } else if constexpr (q == 32) {
    return make_float2(-x.x, -x.y);
  } else if constexpr (q == 48) {
    return DIR < 0 ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  } else if constexpr (q == 8 || q == 24 || q == 40 || q == 56) {  // odd multiples of pi/4
    constexpr float h = 0.70710678118654752440f;
    constexpr float c = (float)cos64(q) > 0 ? h : -h;
    constexpr float s = (float)(DIR * sin64(q)) > 0 ? h : -h;
    // (x.x + i x.y)(c + i s) with |c| = |s| = h
    return make_float2(h * ((c > 0 ? x.x : -x.x) - (s > 0 ? x.y : -x.y)),
                       h * ((s > 0 ? x.x : -x.x) + (c > 0 ? x.y : -x.y)));
  } else {
    constexpr float c = (float)cos64(q);
    constexpr float s = (float)(DIR * sin64(q));
    if (PK) return cmul_p<true>(x, make_float2(c, s));
    return make_float2(fmaf(x.x, c, -x.y * s), fmaf(x.x, s, x.y * c));
  }
}

// R-point DFT in registers (natural order in and out), radix-2 decimation in time.
// DIR = -1: X[q] = sum_n x[n] e^{-2 pi i q n / R};  DIR = +1: unnormalized inverse.
template <int R, int DIR, bool PK = SQNGD_CPACKED>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    float2 a = v[0], b = v[1];
    v[0] = cadd_p<PK>(a, b);
    v[1] = csub_p<PK>(a, b);
  } else {
    float2 ev[R / 2], od[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      ev[i] = v[2 * i];
      od[i] = v[2 * i + 1];
    }
    dft<R / 2, DIR, PK>(ev);
    dft<R / 2, DIR, PK>(od);
    static_for<0, R / 2>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      float2 t = twc<R, DIR, k, PK>(od[k]);
      v[k] = cadd_p<PK>(ev[k], t);
      v[k + R / 2] = csub_p<PK>(ev[k], t);
    });
  }
}

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

// Plan of a P-point transform carried by T = P/E threads.
template <int P_, int E_>
struct Plan {
  static constexpr int P = P_, E = E_, T = P_ / E_;
  static constexpr int LP = ilog2c(P_), LE = ilog2c(E_);
  static constexpr int NP = (LP + LE - 1) / LE;  // passes
  static constexpr int LAST_R = 1 << (LP - LE * (NP - 1));
  static constexpr int PADDED = P_ + P_ / 16;  // float2 per exchange buffer
  static_assert((1 << LP) == P_ && (1 << LE) == E_ && E_ <= P_, "power-of-two sizes");
  __host__ __device__ static constexpr int R(int p) { return p < NP - 1 ? E : LAST_R; }
  __host__ __device__ static constexpr int NS(int p) { return 1 << (LE * p); }
  // twiddle table: pass p >= 1 occupies NS(p) * (R(p) - 1) entries starting at twoff(p)
  __host__ __device__ static constexpr int twoff(int p) {
    int n = 0;
    for (int q = 1; q < p; ++q) n += NS(q) * (R(q) - 1);
    return n;
  }
  static constexpr int TWSIZE = twoff(NP) > 0 ? twoff(NP) : 1;
};

// Host-side builder of the Stockham twiddle table (fp64 -> fp32):
// tw[twoff(p) + (r-1) * Ns + jm] = e^{-2 pi i jm r / (Ns R)}.
template <class PL>
inline void build_twiddle_table(float2* out) {
  for (int p = 1; p < PL::NP; ++p) {
    const int R = PL::R(p), Ns = PL::NS(p);
    for (int r = 1; r < R; ++r)
      for (int jm = 0; jm < Ns; ++jm) {
        const double a = -2.0 * 3.14159265358979323846 * (double)jm * r / ((double)Ns * R);
        out[PL::twoff(p) + (r - 1) * Ns + jm] = make_float2((float)cos(a), (float)sin(a));
      }
  }
}

// Barrier among the threads of one FFT group.
struct GroupSync {
  int id, nthreads;
  unsigned mask;  // lanes of the group when nthreads <= 32
  __device__ __forceinline__ void operator()() const {
    if (nthreads <= 32) {
      __syncwarp(mask);
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
    }
  }
};

// In-place P-point transform of the group's data v (strided ownership in and out).
// DIR = -1 forward, +1 unnormalized inverse.  sbuf: 2 * PADDED float2 of group-private
// smem; tw: the plan's twiddle table (global, read through L1).
// par: exchange parity (alternates the two buffers); must start equal in all threads.
// TWS: the twiddle table `tw` is in shared memory (plain loads) instead of global (__ldg).
// PK: complex arithmetic on packed FP32 pairs (fewer issue slots, more registers: per kernel, measured).
template <class PL, int DIR, bool TWS = false, bool PK = SQNGD_CPACKED>
__device__ __forceinline__ void fft(float2 (&v)[PL::E], const float2* __restrict__ tw, float2* sbuf, int t,
                                    int& par, const GroupSync& sync) {
  constexpr int E = PL::E, T = PL::T;
  static_for<0, PL::NP>([&](auto pc) {
    constexpr int p = decltype(pc)::value;
    constexpr int R = PL::R(p), Ns = PL::NS(p), NB = E / R;
    float2* buf = sbuf + (par ? PL::PADDED : 0);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float2 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = v[b + r * NB];
      const int j = t + b * T;
      if constexpr (p > 0) {
        const float2* twp = tw + PL::twoff(p) + (j & (Ns - 1));
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const float2 w = TWS ? twp[(r - 1) * Ns] : __ldg(twp + (r - 1) * Ns);
          x[r] = DIR < 0 ? cmul_p<PK>(x[r], w) : cmulc_p<PK>(x[r], w);
        }
      }
      dft<R, DIR, PK>(x);
      if constexpr (p == PL::NP - 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[b + r * NB] = x[r];
      } else {
        const int base = (j / Ns) * Ns * R + (j & (Ns - 1));
        float2* wb = buf + pad16(base);
#pragma unroll
        for (int r = 0; r < R; ++r) wb[r * Ns + (r * Ns) / 16] = x[r];  // pad16(base + r Ns), Ns % 16 == 0 or Ns == 1
      }
    }
    if constexpr (p < PL::NP - 1) {
      sync();
      const float2* rb = buf + pad16(t);
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = rb[i * T + (i * T) / 16];  // pad16(t + i T), T % 16 == 0
      par ^= 1;
    }
  });
}

}  // namespace sq
