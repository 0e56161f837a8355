// SQNGD oracle -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, fp64 CPU implementation of what the SQNGD hot path computes,
// written from PAPER.md (arXiv 2604.25728).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header, table or constant generator with the CUDA path
// (paper_2604_25728_b200/csrc); it is built separately by g++.
//
// Every quantity is evaluated from its plain definition:
//   * the AF by the direct two-branch sum of Eq. 6 (no FFT),
//   * the loss by Eqs. 7-9, 37-42 (plus the LSE / p-norm surrogates of the
//     north star),
//   * the gradients by the closed-form adjoint sums written out by direct
//     summation (Wirtinger calculus on Eq. 6), no FFT,
//   * the quantizers by the full sums of Eq. 24 and the literal Eq. 43.
// Readings of the paper are listed in DESIGN.md.
//
// Pins (tests/test_oracle_*.py): numpy.correlate, the Dirichlet closed form,
// the Parseval volume identity, Barker-13, Eq. 25's level set, finite
// differences of every gradient, SPEC per-op examples.  No function here is
// "parity unpinned".
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>

typedef std::complex<double> cd;

extern "C" {

// Plain parameter block (mirrored by oracle/oracle.py with ctypes).
typedef struct {
  int32_t R, M, N, B, r_n;
  double c;                      // quantizer steepness (Eq. 21/24)
  int32_t K;                     // Doppler bins
  double f_lo, f_hi;             // inclusive uniform Doppler grid, paper units
  int32_t tau_lo, tau_hi;        // ROI delays
  int32_t exclude_auto_zero_delay;  // Eq. 8 "tau != 0" (whole column)
  int32_t loss_mode;             // 0 MAX (Eq. 37), 1 LSE, 2 PNORM
  double beta_or_p;
  double eps_w, mu_db;           // Eq. 42 epsilon, SNRL target (dB, Eq. 39)
  const double* weights;         // [K][2N-1] w(tau,f) >= 0, or NULL (=> 1)
} oracle_cfg;

typedef struct {
  double loss, loss_wpsl, loss_snrl;   // Eq. 42, surrogate-or-max, Eq. 41
  double wapsl, wcpsl, wpsl;           // exact maxima of w|A|/N (Eqs. 7-9, /N per Q5)
  int32_t argmax_auto[4];              // (m, l, tau, k)
  int32_t argmax_cross[4];
  int32_t n_cells;                     // |S|, sidelobe cells in the ROI
  int32_t flags;                       // 1: M == 1 (no cross terms); 2: tied maximum (Q17)
} oracle_metrics;

}  // extern "C"

namespace {

const double kPi = 3.14159265358979323846;

// f_k of the inclusive uniform grid.
double doppler_bin(const oracle_cfg& c, int k) {
  if (c.K == 1) return c.f_lo;
  return c.f_lo + (c.f_hi - c.f_lo) * (double)k / (double)(c.K - 1);
}

// e^{j 2 pi n f / N} with the phase n f / N reduced mod 1 in fp64 (Eq. 33).
cd doppler_phasor(int n, double f, int N) {
  double cyc = (double)n * f / (double)N;
  cyc -= std::floor(cyc);
  return cd(std::cos(2.0 * kPi * cyc), std::sin(2.0 * kPi * cyc));
}

double roi_weight(const oracle_cfg& c, int tau, int k, bool is_auto) {
  if (tau < c.tau_lo || tau > c.tau_hi) return 0.0;
  if (is_auto && c.exclude_auto_zero_delay && tau == 0) return 0.0;
  if (c.weights) return c.weights[(size_t)k * (2 * c.N - 1) + (tau + c.N - 1)];
  return 1.0;
}

// Eq. 33: x_hat_{m,f}(n) = x_m(n) e^{j 2 pi n f / N}, n = 1..N.
void modulate(const cd* x, int N, double f, cd* out) {
  for (int n = 1; n <= N; ++n) out[n - 1] = x[n - 1] * doppler_phasor(n, f, N);
}

// Eq. 34 (= Eq. 6 with Eq. 33 substituted): the aperiodic correlation
//   A_ml(tau, f) = sum_n x_hat_{m,f}(n) h_l^*(n + tau),
// the two branches merged as n in [max(1, 1 - tau), min(N, N - tau)].
cd af_cell(const cd* xhat, const cd* h, int N, int tau) {
  cd acc(0.0, 0.0);
  int n0 = std::max(1, 1 - tau), n1 = std::min(N, N - tau);
  for (int n = n0; n <= n1; ++n) acc += xhat[n - 1] * std::conj(h[n + tau - 1]);
  return acc;
}

// Lexicographic (m, l, tau, k) order for argmax ties.
bool lex_less(const int a[4], const int b[4]) {
  for (int i = 0; i < 4; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}

// All Doppler-modulated waveforms of one restart, [M][K][N] (Eq. 33).
void modulate_all(const oracle_cfg& c, const cd* s, std::vector<cd>& xhat) {
  xhat.assign((size_t)c.M * c.K * c.N, cd(0, 0));
#pragma omp parallel for collapse(2) schedule(static)
  for (int m = 0; m < c.M; ++m)
    for (int k = 0; k < c.K; ++k)
      modulate(s + (size_t)m * c.N, c.N, doppler_bin(c, k), &xhat[((size_t)m * c.K + k) * c.N]);
}

// Full AF cube for one restart, [M][M][K][2N-1].
void af_cube(const oracle_cfg& c, const cd* s, const cd* w, std::vector<cd>& A) {
  const int M = c.M, N = c.N, K = c.K, L = 2 * N - 1;
  std::vector<cd> xhat;
  modulate_all(c, s, xhat);
  A.assign((size_t)M * M * K * L, cd(0, 0));
#pragma omp parallel for collapse(3) schedule(dynamic)
  for (int m = 0; m < M; ++m)
    for (int l = 0; l < M; ++l)
      for (int k = 0; k < K; ++k)
        for (int tau = -(N - 1); tau <= N - 1; ++tau)
          A[(((size_t)m * M + l) * K + k) * L + (tau + N - 1)] =
              af_cell(&xhat[((size_t)m * K + k) * N], w + (size_t)l * N, N, tau);
}

struct LossParts {
  oracle_metrics met;
  std::vector<double> p;       // p_m (Eq. 38)
  std::vector<cd> cm;          // c_m = sum_n x_m(n) h_m^*(n) = A_mm(0,0)
  double vmax;                 // max v over S
  double S;                    // LSE: sum e^{beta(v - vmax)}; PNORM: sum (v/vmax)^p
  int arg[4];                  // global argmax over S (WPSL cell)
};

// Eqs. 7-9, 37-42 for one restart, from the AF cube.
LossParts loss_from_cube(const oracle_cfg& c, const cd* s, const cd* w, const std::vector<cd>& A) {
  const int M = c.M, N = c.N, K = c.K, L = 2 * N - 1;
  LossParts lp;
  std::memset(&lp.met, 0, sizeof(lp.met));
  for (int i = 0; i < 4; ++i) lp.met.argmax_auto[i] = lp.met.argmax_cross[i] = lp.arg[i] = -1;
  double wa = -1.0, wc = -1.0;
  int na = 0, nc = 0;  // cells attaining the running maxima (ties, SQNGD_FLAG_TIE)
  int n_cells = 0;
  for (int m = 0; m < M; ++m)
    for (int l = 0; l < M; ++l)
      for (int tau = -(N - 1); tau <= N - 1; ++tau)
        for (int k = 0; k < K; ++k) {   // (m, l, tau, k) lexicographic scan: first max wins ties
          bool is_auto = (m == l);
          double wt = roi_weight(c, tau, k, is_auto);
          if (!(wt > 0.0)) continue;
          ++n_cells;
          double v = wt * std::abs(A[(((size_t)m * M + l) * K + k) * L + (tau + N - 1)]) / N;
          int idx[4] = {m, l, tau, k};
          if (is_auto) {
            if (v > wa) { wa = v; na = 1; std::memcpy(lp.met.argmax_auto, idx, sizeof(idx)); }
            else if (v == wa) ++na;
          } else {
            if (v > wc) { wc = v; nc = 1; std::memcpy(lp.met.argmax_cross, idx, sizeof(idx)); }
            else if (v == wc) ++nc;
          }
        }
  lp.met.n_cells = n_cells;
  lp.met.wapsl = wa < 0 ? 0.0 : wa;
  lp.met.wcpsl = wc < 0 ? 0.0 : wc;
  if (M == 1) lp.met.flags |= 1;
  // 2: a maximum attained by more than one cell, or WAPSL == WCPSL -- the lexicographic rule decided
  // the reported argmax (Q17; the flag of the C-ABI's SQNGD_FLAG_TIE)
  if (na > 1 || nc > 1 || (wa >= 0.0 && wa == wc)) lp.met.flags |= 2;
  // WPSL = max(WAPSL, WCPSL) (Eq. 7); tie between the two -> lexicographically lower cell.
  if (wa > wc || (wa == wc && wa >= 0 && lex_less(lp.met.argmax_auto, lp.met.argmax_cross)))
    std::memcpy(lp.arg, lp.met.argmax_auto, sizeof(lp.arg));
  else
    std::memcpy(lp.arg, lp.met.argmax_cross, sizeof(lp.arg));
  lp.met.wpsl = std::max(lp.met.wapsl, lp.met.wcpsl);
  lp.vmax = lp.met.wpsl;

  // Surrogate sums over S.
  lp.S = 0.0;
  if (c.loss_mode != 0 && lp.vmax > 0.0) {
    for (int m = 0; m < M; ++m)
      for (int l = 0; l < M; ++l)
        for (int k = 0; k < K; ++k)
          for (int tau = -(N - 1); tau <= N - 1; ++tau) {
            double wt = roi_weight(c, tau, k, m == l);
            if (!(wt > 0.0)) continue;
            double v = wt * std::abs(A[(((size_t)m * M + l) * K + k) * L + (tau + N - 1)]) / N;
            if (c.loss_mode == 1) lp.S += std::exp(c.beta_or_p * (v - lp.vmax));
            else lp.S += std::pow(v / lp.vmax, c.beta_or_p);
          }
  }
  if (c.loss_mode == 0) lp.met.loss_wpsl = lp.met.wpsl;                                  // Eq. 37
  else if (c.loss_mode == 1) lp.met.loss_wpsl = lp.vmax + std::log(lp.S) / c.beta_or_p;  // (1/b) ln sum e^{b v}
  else lp.met.loss_wpsl = lp.vmax * std::pow(lp.S, 1.0 / c.beta_or_p);                  // (sum v^p)^{1/p}

  // Eqs. 38-41: p_m = |h_m^H x_m| / N,  p_tar = 10^{-mu/20},  L_SNRL = mean (p_m - p_tar)^2.
  lp.p.resize(M);
  lp.cm.resize(M);
  double ptar = std::pow(10.0, -c.mu_db / 20.0), lsn = 0.0;
  for (int m = 0; m < M; ++m) {
    cd acc(0, 0);
    for (int n = 0; n < N; ++n) acc += s[(size_t)m * N + n] * std::conj(w[(size_t)m * N + n]);
    lp.cm[m] = acc;
    lp.p[m] = std::abs(acc) / N;
    lsn += (lp.p[m] - ptar) * (lp.p[m] - ptar);
  }
  lp.met.loss_snrl = lsn / M;
  lp.met.loss = c.eps_w * lp.met.loss_wpsl + (1.0 - c.eps_w) * lp.met.loss_snrl;  // Eq. 42
  return lp;
}

// dL/dv for a sidelobe cell (the "kappa" weight of the cotangent).
double dloss_dv(const oracle_cfg& c, const LossParts& lp, double v, const int idx[4]) {
  if (c.loss_mode == 0) {  // subgradient of the max, routed to the unique argmax (Q17)
    return (idx[0] == lp.arg[0] && idx[1] == lp.arg[1] && idx[2] == lp.arg[2] && idx[3] == lp.arg[3]) ? 1.0 : 0.0;
  }
  if (lp.vmax <= 0.0) return 0.0;
  if (c.loss_mode == 1) return std::exp(c.beta_or_p * (v - lp.vmax)) / lp.S;        // softmax
  double p = c.beta_or_p;                                                              // S^{1/p-1} v^{p-1}
  return std::pow(lp.S, 1.0 / p - 1.0) * std::pow(v / lp.vmax, p - 1.0);
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- O1: quantizer
// Eq. 24: Q_A(x) = sum_{i < B r_n} a_i [tanh(c (x - rho_i)) + 1], a_i = 1/(2B) (Q10).
double oracle_QA(int B, int r_n, double c, const double* rho, double x) {
  double a = 1.0 / (2.0 * B), y = 0.0;
  for (int i = 0; i < B * r_n; ++i) y += a * (std::tanh(c * (x - rho[i])) + 1.0);
  return y;
}

// Q_A'(x) = sum_i a_i c sech^2(c (x - rho_i))  (Eq. 20 chain).
double oracle_dQA(int B, int r_n, double c, const double* rho, double x) {
  double a = 1.0 / (2.0 * B), y = 0.0;
  for (int i = 0; i < B * r_n; ++i) {
    double ch = std::cosh(c * (x - rho[i]));
    y += a * c / (ch * ch);
  }
  return y;
}

// Eq. 43 literally, then snapped to the nearest k/B (round half up).
// Returns k; y_hard = k / B, phase index b = k mod B.
int64_t oracle_QR_level(int B, int r_n, double c, const double* rho, double x) {
  int n = B * r_n, istar = 0;
  for (int i = 0; i < n; ++i) istar += (rho[i] <= x) ? 1 : 0;   // #{rho_i <= x}
  double y;
  if (istar == 0) y = 0.0;                                       // x < rho_0
  else if (istar == n) y = 2.0 * n * (1.0 / (2.0 * B));         // sum 2 a_i
  else y = oracle_QA(B, r_n, c, rho, 0.5 * (rho[istar - 1] + rho[istar]));  // rho_i <= x < rho_{i+1}
  return (int64_t)std::floor(B * y + 0.5);
}

// Quantize all R*M*N elements.  z: [R][M][N]; rho: [R][B r_n].
// Outputs (any may be NULL): y_soft, dq (= Q_A'), y_hard, b_hard (int32),
// s_soft / s_hard as interleaved (re, im) doubles (Eq. 23: x = e^{j 2 pi y}).
void oracle_quantize(const oracle_cfg* cfg, const double* z, const double* rho,
                     double* y_soft, double* dq, double* y_hard, int32_t* b_hard,
                     double* s_soft, double* s_hard) {
  const oracle_cfg& c = *cfg;
  const int BR = c.B * c.r_n;
  const size_t per = (size_t)c.M * c.N;
#pragma omp parallel for schedule(static)
  for (long long e = 0; e < (long long)(c.R * per); ++e) {
    int r = (int)(e / per);
    const double* rr = rho + (size_t)r * BR;
    double x = z[e];
    double ys = oracle_QA(c.B, c.r_n, c.c, rr, x);
    if (y_soft) y_soft[e] = ys;
    if (dq) dq[e] = oracle_dQA(c.B, c.r_n, c.c, rr, x);
    if (s_soft) {
      double fr = ys - std::floor(ys);
      s_soft[2 * e] = std::cos(2 * kPi * fr);
      s_soft[2 * e + 1] = std::sin(2 * kPi * fr);
    }
    int64_t k = oracle_QR_level(c.B, c.r_n, c.c, rr, x);
    if (y_hard) y_hard[e] = (double)k / c.B;
    int b = (int)(((k % c.B) + c.B) % c.B);
    if (b_hard) b_hard[e] = b;
    if (s_hard) {
      s_hard[2 * e] = std::cos(2 * kPi * b / c.B);
      s_hard[2 * e + 1] = std::sin(2 * kPi * b / c.B);
    }
  }
}

// ---------------------------------------------------------------- O2/O3: AF and metrics
// s, w: [R][M][N] complex (interleaved doubles).  A_out: NULL or [R][M][M][K][2N-1] complex.
// met: [R].  p_out: NULL or [R][M].
void oracle_af(const oracle_cfg* cfg, const double* s, const double* w, double* A_out,
               oracle_metrics* met, double* p_out) {
  const oracle_cfg& c = *cfg;
  const size_t per = (size_t)c.M * c.N;
  const size_t cube = (size_t)c.M * c.M * c.K * (2 * c.N - 1);
  std::vector<cd> A;
  for (int r = 0; r < c.R; ++r) {
    const cd* sr = reinterpret_cast<const cd*>(s) + r * per;
    const cd* wr = reinterpret_cast<const cd*>(w) + r * per;
    af_cube(c, sr, wr, A);
    if (A_out) std::memcpy(A_out + 2 * r * cube, A.data(), cube * sizeof(cd));
    LossParts lp = loss_from_cube(c, sr, wr, A);
    if (met) met[r] = lp.met;
    if (p_out)
      for (int m = 0; m < c.M; ++m) p_out[(size_t)r * c.M + m] = lp.p[m];
  }
}

// ---------------------------------------------------------------- O4: gradients
// Wirtinger cotangent of every cell, G = dL/dA^* (SURVEY §8(a) a7):
//   G = eps * kappa * (w/N) * A / (2|A|)  (0 at A = 0),
// plus the SNRL mainlobe term on c_m = A_mm(0,0):
//   Gc_m = (1-eps) (2/M) (p_m - p_tar) (1/N) c_m / (2|c_m|).
// Outputs (any may be NULL), all [R][M][N] complex interleaved:
//   grad_w = dL/dRe w + j dL/dIm w = 2 dL/dw^*          (Q16)
//   grad_s = dL/ds^*   (the Wirtinger derivative; Step B chains it to z, rho)
// with
//   dL/dw_l^*(k) = sum_{m,f,tau} conj(G_ml(tau,f)) s_m(k-tau) e^{j2pi(k-tau)f/N} + conj(Gc_l) s_l(k)
//   dL/ds_m^*(n) = sum_{l,f,tau} G_ml(tau,f) e^{-j2pi n f/N} w_l(n+tau)          + Gc_m w_m(n).
void oracle_loss_grad(const oracle_cfg* cfg, const double* s, const double* w,
                      oracle_metrics* met, double* grad_w, double* grad_s) {
  const oracle_cfg& c = *cfg;
  const int M = c.M, N = c.N, K = c.K, L = 2 * N - 1;
  const size_t per = (size_t)M * N;
  std::vector<cd> A, G;
  for (int r = 0; r < c.R; ++r) {
    const cd* sr = reinterpret_cast<const cd*>(s) + r * per;
    const cd* wr = reinterpret_cast<const cd*>(w) + r * per;
    af_cube(c, sr, wr, A);
    LossParts lp = loss_from_cube(c, sr, wr, A);
    if (met) met[r] = lp.met;
    G.assign(A.size(), cd(0, 0));
    for (int m = 0; m < M; ++m)
      for (int l = 0; l < M; ++l)
        for (int k = 0; k < K; ++k)
          for (int tau = -(N - 1); tau <= N - 1; ++tau) {
            double wt = roi_weight(c, tau, k, m == l);
            if (!(wt > 0.0)) continue;
            size_t id = (((size_t)m * M + l) * K + k) * L + (tau + N - 1);
            double mag = std::abs(A[id]);
            if (mag == 0.0) continue;
            int idx[4] = {m, l, tau, k};
            double kap = dloss_dv(c, lp, wt * mag / N, idx);
            G[id] = c.eps_w * kap * (wt / N) * A[id] / (2.0 * mag);
          }
    double ptar = std::pow(10.0, -c.mu_db / 20.0);
    std::vector<cd> Gc(M);
    for (int m = 0; m < M; ++m) {
      double mag = std::abs(lp.cm[m]);
      Gc[m] = mag == 0.0 ? cd(0, 0)
                         : (1.0 - c.eps_w) * (2.0 / M) * (lp.p[m] - ptar) / N * lp.cm[m] / (2.0 * mag);
    }
    if (grad_w) {
      std::vector<cd> xhat;
      modulate_all(c, sr, xhat);
      cd* gw = reinterpret_cast<cd*>(grad_w) + r * per;
#pragma omp parallel for collapse(2) schedule(dynamic)
      for (int l = 0; l < M; ++l)
        for (int kk = 1; kk <= N; ++kk) {   // filter sample h_l(kk), one-based
          cd acc(0, 0);
          for (int m = 0; m < M; ++m)
            for (int k = 0; k < K; ++k) {
              const cd* xh = &xhat[((size_t)m * K + k) * N];
              const cd* Gr = &G[(((size_t)m * M + l) * K + k) * L];
              for (int tau = -(N - 1); tau <= N - 1; ++tau) {
                int n = kk - tau;                     // x_hat sample paired with h(kk) at lag tau
                if (n < 1 || n > N) continue;
                acc += std::conj(Gr[tau + N - 1]) * xh[n - 1];
              }
            }
          acc += std::conj(Gc[l]) * sr[(size_t)l * N + kk - 1];
          gw[(size_t)l * N + kk - 1] = 2.0 * acc;
        }
    }
    if (grad_s) {
      cd* gs = reinterpret_cast<cd*>(grad_s) + r * per;
#pragma omp parallel for collapse(2) schedule(dynamic)
      for (int m = 0; m < M; ++m)
        for (int n = 1; n <= N; ++n) {
          cd acc(0, 0);
          for (int l = 0; l < M; ++l)
            for (int k = 0; k < K; ++k) {
              double f = doppler_bin(c, k);
              cd dem = std::conj(doppler_phasor(n, f, N));
              const cd* Gr = &G[(((size_t)m * M + l) * K + k) * L];
              cd part(0, 0);
              for (int tau = -(N - 1); tau <= N - 1; ++tau) {
                int kk = n + tau;
                if (kk < 1 || kk > N) continue;
                part += Gr[tau + N - 1] * wr[(size_t)l * N + kk - 1];
              }
              acc += dem * part;
            }
          acc += Gc[m] * wr[(size_t)m * N + n - 1];
          gs[(size_t)m * N + n - 1] = acc;
        }
    }
  }
}

// Chain rule through x = e^{j 2 pi y}, y = Q_A(z; rho) (Eqs. 23-24):
//   dL/dy = 4 pi Im(g conj(x)),  g = dL/dx^*
//   dL/dz = Q_A'(z) dL/dy,  dL/drho_i = -sum_{m,n} a c sech^2(c (z - rho_i)) dL/dy.
// z: [R][M][N]; rho: [R][BR]; s: x (complex); grad_s: g.  Outputs [R][M][N], [R][BR].
void oracle_chain(const oracle_cfg* cfg, const double* z, const double* rho, const double* s,
                  const double* grad_s, double* grad_z, double* grad_rho) {
  const oracle_cfg& c = *cfg;
  const int BR = c.B * c.r_n;
  const size_t per = (size_t)c.M * c.N;
  const double a = 1.0 / (2.0 * c.B);
  std::vector<double> dy(c.R * per);
  for (size_t e = 0; e < c.R * per; ++e) {
    cd g(grad_s[2 * e], grad_s[2 * e + 1]), x(s[2 * e], s[2 * e + 1]);
    dy[e] = 4.0 * kPi * std::imag(g * std::conj(x));
  }
  for (int r = 0; r < c.R; ++r) {
    const double* rr = rho + (size_t)r * BR;
    if (grad_z)
      for (size_t e = r * per; e < (r + 1) * per; ++e)
        grad_z[e] = oracle_dQA(c.B, c.r_n, c.c, rr, z[e]) * dy[e];
    if (grad_rho) {
#pragma omp parallel for schedule(static)
      for (int i = 0; i < BR; ++i) {
        double acc = 0.0;
        for (size_t e = r * per; e < (r + 1) * per; ++e) {
          double ch = std::cosh(c.c * (z[e] - rr[i]));
          acc += -a * c.c / (ch * ch) * dy[e];
        }
        grad_rho[(size_t)r * BR + i] = acc;
      }
    }
  }
}

// ---------------------------------------------------------------- O5 pieces
// Adam (bias-corrected) on n reals, in place.  t = step number after increment.
void oracle_adam(int64_t n, double* x, double* m, double* v, const double* g, int64_t t,
                 double lr, double b1, double b2, double eps) {
  double c1 = 1.0 - std::pow(b1, (double)t), c2 = 1.0 - std::pow(b2, (double)t);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    x[i] -= lr * (m[i] / c1) / (std::sqrt(v[i] / c2) + eps);
  }
}

// Eq. 32: h_m <- sqrt(N / ||h_m||^2) h_m for each of the `rows` rows of length N.
// Returns the number of zero rows (left unchanged).
int oracle_project_filters(int rows, int N, double* w) {
  int bad = 0;
  for (int r = 0; r < rows; ++r) {
    double e = 0.0;
    for (int n = 0; n < 2 * N; ++n) e += w[(size_t)r * 2 * N + n] * w[(size_t)r * 2 * N + n];
    if (e == 0.0) { ++bad; continue; }
    double sc = std::sqrt(N / e);
    for (int n = 0; n < 2 * N; ++n) w[(size_t)r * 2 * N + n] *= sc;
  }
  return bad;
}

// "project the thresholds to a valid ordered set", per SURVEY Q22:
// sort ascending, clamp into [lo, hi], forward sweep enforcing a minimum gap.
void oracle_project_thresholds(int rows, int n, double* rho, double lo, double hi, double gap) {
  for (int r = 0; r < rows; ++r) {
    double* p = rho + (size_t)r * n;
    std::sort(p, p + n);
    for (int i = 0; i < n; ++i) p[i] = std::min(std::max(p[i], lo), hi);
    for (int i = 1; i < n; ++i) p[i] = std::max(p[i], p[i - 1] + gap);
  }
}

}  // extern "C"
