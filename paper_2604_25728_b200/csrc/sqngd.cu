// libsqngd.so -- host side of the C-ABI (include/sqngd.h): context, validation,
// launch configuration, and the orchestration of the kernels in af_kernels.cuh /
// misc_kernels.cuh.  Every arithmetic step of the hot path runs on the GPU.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "../../include/sqngd.h"
#include "comm.h"
#include "lr_kernels.cuh"
#include "lr_tc.cuh"
#include "misc_kernels.cuh"
#include "world_peer.cuh"
#include "net.cuh"
#include "run.cuh"

using namespace sq;

static_assert(sizeof(MetricsOut) == sizeof(sqngd_metrics), "metrics layout");

namespace {

thread_local std::string g_last_error;

// Launch geometry per FFT length: E elements per thread, G groups per CTA, and the
// minimum resident CTAs per SM handed to __launch_bounds__ (caps registers at 128).
#ifndef SQNGD_E
#define SQNGD_E 16
#endif
#ifndef SQNGD_MINB256
#define SQNGD_MINB256 2
#endif
#ifndef SQNGD_MINB128
#define SQNGD_MINB128 3
#endif
#ifndef SQNGD_RHO_TB
#define SQNGD_RHO_TB 16
#endif
constexpr int kRhoTB = SQNGD_RHO_TB;  // k_grad_rho: thresholds per block (256 / TB lanes each)
constexpr int plan_E(int P) { return P <= SQNGD_E ? P : SQNGD_E; }
constexpr int plan_G(int P) { return (P / plan_E(P)) >= 128 ? 1 : 128 / (P / plan_E(P)); }
constexpr int plan_MINB(int P) {
  return (P / plan_E(P)) * plan_G(P) >= 512 ? 1 : (P / plan_E(P)) * plan_G(P) >= 256 ? SQNGD_MINB256 : SQNGD_MINB128;
}

}  // namespace

struct sqngd_ctx_s {
  // Device allocations of the workspace.  With SQNGD_GUARD=1 (read at create) every buffer gets a
  // 4 KiB guard band on each side filled with 0x5A; sqngd_check_guards verifies the bands (an
  // out-of-bounds write by any kernel into a neighbouring guard shows up as a changed byte).
  static constexpr size_t kGuard = 4096;
  bool guard = false;
  std::vector<std::pair<char*, size_t>> guarded;  // (base, user bytes)
  template <class T>
  cudaError_t dmalloc(T** p, size_t bytes) {
    if (!guard) return cudaMalloc(reinterpret_cast<void**>(p), bytes);
    char* base = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemset(base, 0x5A, bytes + 2 * kGuard)) != cudaSuccess) return e;
    guarded.push_back({base, bytes});
    *p = reinterpret_cast<T*>(base + kGuard);
    return cudaSuccess;
  }
  void dfree(void* p) {
    if (!p) return;
    for (auto& g : guarded)
      if (g.first + kGuard == p) {
        cudaFree(g.first);
        g.first = nullptr;
        return;
      }
    cudaFree(p);
  }
  sqngd_config cfg{};
  int dev = 0, rank = 0, world = 1;
  bool multi = false;  // the sharded path with its grouped collective (world > 1, or a 1-rank NCCL context)
  int P = 0, L = 0, BR = 0, sms = 0;
  uint32_t n_cells = 0, flags = 0;
  // persistent grid: resident groups per fused-kernel mode (0 fwd, 1 adj A, 2 adj B)
  int64_t slots[3] = {1, 1, 1};
  int64_t units = 0;       // R * M * K
  int* counter = nullptr;  // dynamic unit counter
  float2* spec = nullptr;  // [R][M][P] Step-A spectral sums
  std::string err;
  // device workspace
  float2* tw = nullptr;     // [K][N] e^{j 2 pi (n+1) f_k / N} (fp64-built)
  float2* H = nullptr;      // [R][M][P] filter spectra / P
  float2* Xc = nullptr;     // [R][M][K][P] X cache: FFT_P of the Doppler-modulated codes (a3)
  float2* ftw = nullptr;    // Stockham twiddle table of the plan
  float2* ftwr = nullptr;   // twiddle table of the row kernels' plan (Launch::PLR)
  float2* ftwn = nullptr;   // twiddle table of the Chebyshev node kernels' plan (Launch::PLN)
  float2* s_soft = nullptr; // [R][M][N]
  float2* s_hard = nullptr;
  float* dq = nullptr;      // [R][M][N]
  int* lut = nullptr;       // [R][BR+1]
  Part part{};              // per unit u = (r M + a) K + k: keys, shift, sum, scale; [U][P] gradient slots
  Red* red = nullptr;       // [R]
  double2* cm = nullptr;    // [R][M]
  float2* red_grad = nullptr;  // [R][M][N]
  float* dy = nullptr;         // [R][M][N]
  // Adam(rho) + projection: a 1024-thread kernel.  As the optimization proceeds the thresholds form
  // clusters that Adam reorders every step, so the projection's sort runs every step.
  float2* gw = nullptr;        // step scratch: grad_w [R][M][N]
  float* gz = nullptr;         // [R][M][N]
  float* grho = nullptr;       // [R][BR]
  MetricsOut* met = nullptr;   // [R] scratch
  int* status = nullptr;       // latched device status bits
  // Chebyshev Doppler engine (lr_kernels.cuh): Q nodes, tables, node AFs / cotangents
  bool lr = false;
  int Q = 0, QS = 0, nch = 0, kw = 1, LS = 0;
  int nch16 = 0, NT = 0, NTF = 0;
  int lsplit = 1;              // k_adj_gc CTAs per node (fills the GPU when R M Q nodes are few)
  float4* tabF = nullptr;      // [NT][32][2] k_lrt forward B fragments
  float4* tabA = nullptr;      // [NT][32][2] k_lrt adjoint B fragments
  uint4* tabF16 = nullptr;     // [NT][32] k_lrt forward B fragments (FP16 packed split)
  uint2* tabM16 = nullptr;     // [32] k_lrt middle-bin B fragment
  uint4* tabB = nullptr;       // [npc][2] k_lrf (tcgen05 forward) B images, one per 64 bin pairs
  int nc128 = 0, npc = 0;      // k_lrf: 128-lag chunks per pair, 64-pair MMA chunks
  bool use_lrf = false;        // forward-only contraction on tcgen05 (k_lrf) instead of k_lrt
  size_t lrf_smem = 0;
  int64_t units_lr = 0;        // fused-kernel units: R M^2 x (16-lag chunks for k_lrt | 128-lag tiles for k_lrt5)
  size_t lr_smem = 0;          // k_lrt dynamic shared memory
  LrRed* lred = nullptr;       // [R] running maxima of the fused kernel
  cudaStream_t side = nullptr; // graph branch for k_lr_finish (fork / join events)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double lr_err = 0.0;         // interpolation error bound of the chosen Q (host estimate)
  float2* Vt = nullptr;        // [Q][N] e^{j 2 pi (n - n_c) f*_q / N}
  float* coef = nullptr;       // [K/2 + 1][QS] alpha / beta rows
  float* wmax = nullptr;       // [L] max_k weights (weighted ROI)
  float2* Rn = nullptr;        // [R M M][Q][LS] node AFs
  float2* Gn = nullptr;        // [R M M][Q][LS] node cotangents
  float2* tslot = nullptr;     // [R M Q][N] Step-B node time-domain partials
  // multi-GPU (comm.h): this rank's shard, the grouped collective's buffers, the reference shifts
  Comm* comm = nullptr;
  PeerComm* peer_pending = nullptr;  // window exported (sqngd_peer_export), not yet attached
  int row_lo = 0, row_hi = 0;   // Chebyshev engine: (restart, transmit channel) rows [row_lo, row_hi)
  double* pay = nullptr;        // [R][1 + 2 M N] fp64 SUM payload
  unsigned long long* keyb = nullptr;  // [R][3] u64 MAX payload
  double* mref = nullptr;       // [R] reference shift (previous evaluation's global maximum)
  void* run_dev = nullptr;     // sqngd_run bookkeeping (run.cu), reused across calls
  void* run_host = nullptr;    // pinned stop-flag mirror
  size_t run_dev_bytes = 0, run_host_bytes = 0;
  long long* d_t = nullptr;    // device Adam step counters (t_a, t_b) at the start of sqngd_step
  double* snrl_w = nullptr;    // [R] max_m SNRL_m of the step's entry iterate (hard_out via Step A)
  float2* d_ct = nullptr;      // [2][cts] bias corrections of the step's inner iterations (k_set_t)
  int cts = 0;
  // generator z = f_theta(y0) (net.cu, NEXT-2)
  bool net = false;
  NetDims nd{};
  NetWs nws{};
  float* net_ws = nullptr;
  cudaStream_t side_net = nullptr;               // graph branch: generator backward beside the grad-rho pass
  cudaEvent_t ev_nf = nullptr, ev_nj = nullptr;
  // CUDA graphs of sqngd_step (one per (state buffers, block, outputs, profiling))
  struct GraphEntry {
    const void* key[16];
    int block;
    bool prof;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> marks;  // event-record nodes (profiling)
    bool replayed = false;
    cudaGraph_t graph = nullptr;   // kept for the k_set_t node below
    cudaGraphNode_t set_t = nullptr;  // the step counters' kernel node: its (t_a, t_b) are set per replay
    cudaKernelNodeParams set_p{};
  };
  std::vector<GraphEntry*> graphs;
  void drop_graphs() {
    for (auto* g : graphs) {
      if (g->exec) cudaGraphExecDestroy(g->exec);
      if (g->graph) cudaGraphDestroy(g->graph);
      for (auto& mk : g->marks) {
        cudaEventDestroy(std::get<1>(mk));
        cudaEventDestroy(std::get<2>(mk));
      }
      delete g;
    }
    graphs.clear();
  }
  GraphEntry* capturing = nullptr;
  bool use_graphs = true;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_marks;  // (class, index of start event)
  int64_t launches = 0;
  cudaEvent_t ev_get() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
};

// Brackets one fused-kernel launch with events when profiling is on.
struct ProfScope {
  sqngd_ctx_s* c;
  int cls;
  size_t idx = 0;
  cudaStream_t st;
  // (profiling runs sqngd_step eagerly: events recorded as graph nodes cannot be timed)
  ProfScope(sqngd_ctx_s* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
    if (!c->prof || c->capturing) return;
    idx = c->ev_used;
    cudaEventRecord(c->ev_get(), st);
  }
  ~ProfScope() {
    if (!c->prof || c->capturing) return;
    cudaEventRecord(c->ev_get(), st);
    c->ev_marks.push_back({cls, idx});
  }
};

// ----------------------------------------------------------------------------- helpers
#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) return fail(ctx, SQNGD_E_CUDA, #x, cudaGetErrorString(e_)); \
  } while (0)

static sqngd_status fail(sqngd_ctx ctx, sqngd_status st, const char* what, const char* why = "") {
  std::string msg = std::string(what) + (why && *why ? std::string(": ") + why : std::string());
  if (ctx) ctx->err = msg;
  g_last_error = msg;
  return st;
}

static inline cudaStream_t S(sqngd_stream st) { return reinterpret_cast<cudaStream_t>(st); }

// ----------------------------------------------------------------------------- per-P dispatch
template <int P>
struct Launch {
  static constexpr int E = plan_E(P);
  using PL = Plan<P, E>;
  static constexpr int G = plan_G(P);
  static constexpr int MINB = plan_MINB(P);
  static constexpr int THREADS = PL::T * G;
  // latency-bound row kernels (one transform per filter row, few rows): 8 elements per thread,
  // twice the threads per transform (measured: the E = 16 row kernel runs one warp per SMSP)
#ifndef SQNGD_EN
#define SQNGD_EN 16
#endif
  // Chebyshev engine node kernels (k_node, k_adj_g, node k_xhat): few hundred units per launch
  static constexpr int EN = P <= SQNGD_EN ? P : SQNGD_EN;
  using PLN = Plan<P, EN>;
  static constexpr int GN = (P / EN) >= 128 ? 1 : 128 / (P / EN);
  static constexpr int THREADS_N = PLN::T * GN;
  static constexpr int MINBN = (P / EN) * GN >= 512 ? 1 : (P / EN) * GN >= 256 ? 2 : 3;
  static size_t smem_n() { return (size_t)GN * FftSmem<PLN>::TOTAL * sizeof(float2) + 16; }
  static std::vector<float2> twiddles_n() {
    std::vector<float2> t(PLN::TWSIZE, make_float2(1.f, 0.f));
    build_twiddle_table<PLN>(t.data());
    return t;
  }
  static constexpr int ER = P <= 8 ? P : 8;
  using PLR = Plan<P, ER>;
  static constexpr int GR = (P / ER) >= 128 ? 1 : 128 / (P / ER);
  static constexpr int THREADS_R = PLR::T * GR;
  static size_t smem_r() { return (size_t)GR * FftSmem<PLR>::TOTAL * sizeof(float2) + 16; }
  static std::vector<float2> twiddles_r() {
    std::vector<float2> t(PLR::TWSIZE, make_float2(1.f, 0.f));
    build_twiddle_table<PLR>(t.data());
    return t;
  }

  template <int MODE>
  static size_t smem() {
    return (size_t)G * GroupSmem<PL, MODE>::TOTAL * sizeof(float2) + (SQNGD_AF_TWS ? PL::TWSIZE * sizeof(float2) : 0);
  }
  static size_t smem_fft() { return (size_t)G * FftSmem<PL>::TOTAL * sizeof(float2) + 16; }

  static cudaError_t prepare(int* blocks_per_sm) {
    cudaError_t e;
    e = cudaFuncSetAttribute(k_af<PL, G, MINB, MODE_FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem<MODE_FWD>());
    if (e) return e;
    e = cudaFuncSetAttribute(k_af<PL, G, MINB, MODE_ADJ_A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem<MODE_ADJ_A>());
    if (e) return e;
    e = cudaFuncSetAttribute(k_af<PL, G, MINB, MODE_ADJ_B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem<MODE_ADJ_B>());
    if (e) return e;
    e = cudaFuncSetAttribute(k_filter_fft<PL, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft());
    if (e) return e;
    e = cudaFuncSetAttribute(k_xhat<PL, G, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft());
    if (e) return e;
    e = cudaFuncSetAttribute(k_rows_ifft<PL, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft());
    if (e) return e;
    e = cudaFuncSetAttribute(k_rows_ifft_fin<PLR, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r());
    if (e) return e;
    e = cudaFuncSetAttribute(k_rows_adam_w<PLR, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r());
    if (e) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[0], k_af<PL, G, MINB, MODE_FWD>, THREADS, smem<MODE_FWD>());
    if (e) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[1], k_af<PL, G, MINB, MODE_ADJ_A>, THREADS, smem<MODE_ADJ_A>());
    if (e) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[2], k_af<PL, G, MINB, MODE_ADJ_B>, THREADS, smem<MODE_ADJ_B>());
  }
  static std::vector<float2> twiddles() {
    std::vector<float2> t(PL::TWSIZE, make_float2(1.f, 0.f));
    build_twiddle_table<PL>(t.data());
    return t;
  }
  static void filter(int RM, int N, const float2* w, const float2* ftw, float2* H, const float2* s, double2* cm,
                     cudaStream_t st) {
    const int blocks = (RM + G - 1) / G;
    k_filter_fft<PL, G><<<blocks, THREADS, smem_fft(), st>>>(RM, N, w, ftw, H, s, cm);
  }
  static void xhat(int u0, int units, int M, int N, int K, const float2* s, const float2* dtw, const float2* ftw,
                   float2* Xc, const float2* w, double2* cm, cudaStream_t st) {
    const int blocks = (units + G - 1) / G;
    k_xhat<PL, G, MINB><<<blocks, THREADS, smem_fft(), st>>>(u0, units, M, N, K, s, dtw, ftw, Xc, w, cm);
  }
  static void xhat_n(int u0, int units, int M, int N, int K, const float2* s, const float2* dtw, const float2* ftwn,
                     float2* Xc, const float2* w, double2* cm, cudaStream_t st) {
    const int blocks = (units + GN - 1) / GN;
    k_xhat<PLN, GN, MINBN><<<blocks, THREADS_N, smem_n(), st>>>(u0, units, M, N, K, s, dtw, ftwn, Xc, w, cm);
  }
  static void rows_ifft(int rows, int N, const float2* in, const float2* ftw, float2* out, cudaStream_t st) {
    const int blocks = (rows + G - 1) / G;
    k_rows_ifft<PL, G><<<blocks, THREADS, smem_fft(), st>>>(rows, N, in, ftw, out);
  }
  static void rows_adam_w(int rows, const float2* in, const float2* ftwr, const FinArgs& f, const AdamP& ap,
                          float2* w, float* mw, float* vw, float2* H, double2* cm, int* status, cudaStream_t st) {
    const int blocks = (rows + GR - 1) / GR;
    k_rows_adam_w<PLR, GR><<<blocks, THREADS_R, smem_r(), st>>>(rows, in, ftwr, f, ap, w, mw, vw, H, cm, status);
  }
  static void rows_ifft_fin(int rows, const float2* in, const float2* ftwr, const FinArgs& f, int* status,
                            cudaStream_t st) {
    const int blocks = (rows + GR - 1) / GR;
    k_rows_ifft_fin<PLR, GR><<<blocks, THREADS_R, smem_r(), st>>>(rows, in, ftwr, f, status);
  }
  static void af(int mode, const KP& kp, int64_t slots, const float2* Xc, const float2* H, const float2* tw,
                 const float2* ftw, float* af_mag, const Part& part, cudaStream_t st) {
    const int64_t units = kp.u_hi - kp.u_lo;
    if (units <= 0) return;
    const int blocks = (int)((std::min<int64_t>(units, slots) + G - 1) / G);
    if (mode == MODE_FWD)
      k_af<PL, G, MINB, MODE_FWD><<<blocks, THREADS, smem<MODE_FWD>(), st>>>(kp, Xc, H, tw, ftw, af_mag, part);
    else if (mode == MODE_ADJ_A)
      k_af<PL, G, MINB, MODE_ADJ_A><<<blocks, THREADS, smem<MODE_ADJ_A>(), st>>>(kp, Xc, H, tw, ftw, nullptr, part);
    else
      k_af<PL, G, MINB, MODE_ADJ_B><<<blocks, THREADS, smem<MODE_ADJ_B>(), st>>>(kp, Xc, H, tw, ftw, nullptr, part);
  }
  static int groups_per_block() { return G; }
  // Chebyshev engine: node AFs, node adjoint correlations, Step-B node tail
  static void node(int u0, int units, int M, int Q, int N, int LS, const float2* Xc, const float2* H,
                   const float2* ftwn, float2* Rn, int R, LrRed* lred, cudaStream_t st) {
    k_node<PLN, GN, MINBN><<<(units + GN - 1) / GN, THREADS_N, smem_n(), st>>>(u0, units, M, Q, N, LS, Xc, H, ftwn, Rn,
                                                                               R, lred);
  }
  static void adj_g(const AdjGArgs& a, const float2* ftwn, cudaStream_t st) {  // Step A node adjoints
    const int blocks = (a.units + GN - 1) / GN;
    k_adj_g<PLN, GN, MINBN><<<blocks, THREADS_N, smem_n(), st>>>(a, ftwn);
  }
  // Step-B node adjoints summed inside the CTA: NGC groups per CTA (shared memory: NGC exchange buffers)
  static constexpr int NGC = (PLN::T >= 512) ? 1 : (PLN::T >= 256 ? 2 : ((128 / PLN::T) > 4 ? 128 / PLN::T : 4));
  static size_t smem_c() { return (size_t)NGC * FftSmem<PLN>::TOTAL * sizeof(float2) + 16; }
  static void adj_gc(const AdjGArgs& a, int ctas, const float2* ftwn, cudaStream_t st) {
    if (ctas > 0) k_adj_gc<PLN, NGC><<<ctas, PLN::T * NGC, smem_c(), st>>>(a, ftwn);
  }
  static cudaError_t prepare_lr() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_node<PLN, GN, MINBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n())))
      return e;
    if ((e = cudaFuncSetAttribute(k_adj_g<PLN, GN, MINBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n())))
      return e;
    if ((e = cudaFuncSetAttribute(k_xhat<PLN, GN, MINBN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_n())))
      return e;
    return cudaFuncSetAttribute(k_adj_gc<PLN, NGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c());
  }
};

// k_lrt instantiations: Q in {4, 6, ..., 16} x loss mode x weighted ROI x gradient.
template <int Q>
struct LrLaunch {
  // tensor-core variant
  template <int LM, bool HW, int KM>
  static void go_t(const LrtArgs& a, int rows, size_t smem, cudaStream_t st) {  // grid (chunk, l, row - row0)
    if (rows > 0) k_lrt<Q, LM, HW, KM><<<dim3(a.nch, a.M, rows), 32 * a.kw, smem, st>>>(a);
  }
  template <int LM>
  static void go_lm(bool hw, int km, const LrtArgs& a, int units, size_t smem, cudaStream_t st) {
    if (km == 0) hw ? go_t<LM, true, 0>(a, units, smem, st) : go_t<LM, false, 0>(a, units, smem, st);
    else if (km == 2) hw ? go_t<LM, true, 2>(a, units, smem, st) : go_t<LM, false, 2>(a, units, smem, st);
    else if constexpr (LM != 0) hw ? go_t<LM, true, 1>(a, units, smem, st) : go_t<LM, false, 1>(a, units, smem, st);
  }
  // km: 0 forward, 1 forward + adjoint (LSE / p-norm only), 2 forward writing the |A| map
  static void launch_t(int lm, bool hw, int km, const LrtArgs& a, int units, size_t smem, cudaStream_t st) {
    if (lm == 0) go_lm<0>(hw, km, a, units, smem, st);
    else if (lm == 1) go_lm<1>(hw, km, a, units, smem, st);
    else go_lm<2>(hw, km, a, units, smem, st);
  }
  template <int LM, bool HW, int KM>
  static cudaError_t attr_t(size_t smem) {
    return cudaFuncSetAttribute(k_lrt<Q, LM, HW, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  template <int LM>
  static cudaError_t attr_lm(size_t smem) {
    cudaError_t e;
    if ((e = attr_t<LM, false, 0>(smem)) || (e = attr_t<LM, true, 0>(smem)) || (e = attr_t<LM, false, 2>(smem)) ||
        (e = attr_t<LM, true, 2>(smem)))
      return e;
    if constexpr (LM != 0)
      if ((e = attr_t<LM, false, 1>(smem)) || (e = attr_t<LM, true, 1>(smem))) return e;
    return cudaSuccess;
  }
  static cudaError_t prepare_t(size_t smem) {
    cudaError_t e;
    if ((e = attr_lm<0>(smem)) || (e = attr_lm<1>(smem)) || (e = attr_lm<2>(smem))) return e;
    return cudaSuccess;
  }
  static cudaError_t occupancy_t(int* bps, int threads, size_t smem) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k_lrt<Q, 1, false, 1>, threads, smem);
  }
};

// k_lrf (tcgen05 forward contraction) instantiations: loss mode x weighted ROI x map.
struct LrfLaunch {
  template <int LM, bool HW, bool MAP>
  static cudaError_t attr(size_t smem) {
    return cudaFuncSetAttribute(k_lrf<LM, HW, MAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  template <int LM>
  static cudaError_t attr_lm(size_t smem) {
    cudaError_t e;
    if ((e = attr<LM, false, false>(smem)) || (e = attr<LM, true, false>(smem)) || (e = attr<LM, false, true>(smem)) ||
        (e = attr<LM, true, true>(smem)))
      return e;
    return cudaSuccess;
  }
  static cudaError_t prepare(size_t smem) {
    cudaError_t e;
    if ((e = attr_lm<0>(smem)) || (e = attr_lm<1>(smem)) || (e = attr_lm<2>(smem))) return e;
    return cudaSuccess;
  }
  template <int LM, bool HW, bool MAP>
  static void go(const LrfArgs& a, int rows, size_t smem, cudaStream_t st) {
    if (rows > 0) k_lrf<LM, HW, MAP><<<dim3(a.nc, a.M, rows), kLrfThreads, smem, st>>>(a);
  }
  template <int LM>
  static void go_lm(bool hw, bool map, const LrfArgs& a, int rows, size_t smem, cudaStream_t st) {
    if (map) hw ? go<LM, true, true>(a, rows, smem, st) : go<LM, false, true>(a, rows, smem, st);
    else hw ? go<LM, true, false>(a, rows, smem, st) : go<LM, false, false>(a, rows, smem, st);
  }
  static void launch(int lm, bool hw, bool map, const LrfArgs& a, int rows, size_t smem, cudaStream_t st) {
    if (lm == 0) go_lm<0>(hw, map, a, rows, smem, st);
    else if (lm == 1) go_lm<1>(hw, map, a, rows, smem, st);
    else go_lm<2>(hw, map, a, rows, smem, st);
  }
};

template <class Fn>
static bool with_Q(int Q, Fn&& fn) {
  switch (Q) {
    case 4: fn(LrLaunch<4>{}); return true;
    case 6: fn(LrLaunch<6>{}); return true;
    case 8: fn(LrLaunch<8>{}); return true;
    case 10: fn(LrLaunch<10>{}); return true;
    case 12: fn(LrLaunch<12>{}); return true;
    case 14: fn(LrLaunch<14>{}); return true;
    case 16: fn(LrLaunch<16>{}); return true;
    default: return false;
  }
}

template <class Fn>
static bool with_P(int P, Fn&& fn) {
  switch (P) {
    case 4: fn(Launch<4>{}); return true;
    case 8: fn(Launch<8>{}); return true;
    case 16: fn(Launch<16>{}); return true;
    case 32: fn(Launch<32>{}); return true;
    case 64: fn(Launch<64>{}); return true;
    case 128: fn(Launch<128>{}); return true;
    case 256: fn(Launch<256>{}); return true;
    case 512: fn(Launch<512>{}); return true;
    case 1024: fn(Launch<1024>{}); return true;
    case 2048: fn(Launch<2048>{}); return true;
    case 4096: fn(Launch<4096>{}); return true;
    case 8192: fn(Launch<8192>{}); return true;
    default: return false;
  }
}

static KP make_kp(const sqngd_ctx_s* c, int want_S) {
  KP kp;
  const sqngd_config& g = c->cfg;
  kp.R = g.R; kp.M = g.M; kp.N = g.N; kp.K = g.K; kp.L = c->L; kp.P = c->P;
  kp.tau_lo = g.tau_lo; kp.tau_hi = g.tau_hi; kp.excl0 = g.exclude_auto_zero_delay;
  kp.loss_mode = g.loss_mode; kp.beta_or_p = (float)g.beta_or_p; kp.invN = 1.0f / (float)g.N;
  kp.weights = g.weights;
  int64_t lo, hi;
  sqngd_shard_range(c->units, c->rank, c->world, &lo, &hi);
  kp.u_lo = (int)lo; kp.u_hi = (int)hi;
  kp.want_S = want_S;
  kp.counter = c->counter;
  kp.tiew = reinterpret_cast<uint32_t*>(c->counter + 2);
  kp.track_tie = 0;
  kp.mld = g.map_ld > 0 ? g.map_ld : c->L;
  return kp;
}

// ----------------------------------------------------------------------------- Chebyshev engine tables
// Doppler bin k of the inclusive uniform grid (Q8).
static double grid_f(const sqngd_config& c, int k) {
  return c.K == 1 ? c.f_lo : c.f_lo + (c.f_hi - c.f_lo) * (double)k / (double)(c.K - 1);
}

// Q Chebyshev nodes (first kind) of [f_lo, f_hi] and the Lagrange basis l_q(f_k) (barycentric form,
// weights (-1)^q sin((2q+1) pi / 2Q)), in fp64.  Returns the interpolation error bound
//   max_{k, t} | e^{j 2 pi t f_k} - sum_q l_q(f_k) e^{j 2 pi t f*_q} |,  t = (n - n_c)/N,
// evaluated on 513 t-samples of [-(N-1)/2N, (N-1)/2N] (the error is smooth in t); by
// Cauchy-Schwarz |At_interp - At| <= err * ||s|| ||w|| for every cell.
static double lr_tables(const sqngd_config& c, int Q, std::vector<double>& fq, std::vector<double>& ell) {
  const double ctr = 0.5 * (c.f_lo + c.f_hi), hw = 0.5 * (c.f_hi - c.f_lo);
  fq.assign(Q, 0.0);
  std::vector<double> bw(Q);
  for (int q = 0; q < Q; ++q) {
    const double th = (2.0 * q + 1.0) * M_PI / (2.0 * Q);
    fq[q] = ctr + hw * std::cos(th);
    bw[q] = ((q & 1) ? -1.0 : 1.0) * std::sin(th);
  }
  ell.assign((size_t)c.K * Q, 0.0);
  for (int k = 0; k < c.K; ++k) {
    const double f = grid_f(c, k);
    int hit = -1;
    for (int q = 0; q < Q; ++q)
      if (std::fabs(f - fq[q]) <= 1e-15 * std::max(1.0, std::fabs(hw))) hit = q;
    double* lr = &ell[(size_t)k * Q];
    if (hit >= 0) {
      lr[hit] = 1.0;
      continue;
    }
    double den = 0.0;
    for (int q = 0; q < Q; ++q) den += bw[q] / (f - fq[q]);
    for (int q = 0; q < Q; ++q) lr[q] = bw[q] / (f - fq[q]) / den;
  }
  double err = 0.0;
  const int NT = 513;
  const double tmax = (c.N - 1) / (2.0 * c.N);
  for (int k = 0; k < c.K; ++k) {
    const double f = grid_f(c, k);
    for (int i = 0; i < NT; ++i) {
      const double t = -tmax + 2.0 * tmax * i / (NT - 1);
      double re = std::cos(2.0 * M_PI * t * f), im = std::sin(2.0 * M_PI * t * f);
      for (int q = 0; q < Q; ++q) {
        const double a = 2.0 * M_PI * t * fq[q], lq = ell[(size_t)k * Q + q];
        re -= lq * std::cos(a);
        im -= lq * std::sin(a);
      }
      err = std::max(err, std::hypot(re, im));
    }
  }
  return err;
}

// ----------------------------------------------------------------------------- C-ABI
extern "C" {

const char* sqngd_version(void) { return "sqngd-b200 0.1 (sm_100a)"; }

int64_t sqngd_net_num_params(const sqngd_config* cfg) {
  if (!cfg || cfg->net_width <= 0) return 0;
  NetDims d;
  const char* why = "";
  if (!net_dims(1, cfg->M * cfg->N, cfg->net_width, cfg->net_depth, &d, &why)) return 0;
  return (int64_t)d.P;
}

int64_t sqngd_num_units(const sqngd_config* cfg) {
  return cfg ? (int64_t)cfg->R * cfg->M * cfg->K : 0;
}

void sqngd_shard_range(int64_t units, int rank, int world, int64_t* lo, int64_t* hi) {
  if (world < 1) world = 1;
  const int64_t base = units / world, rem = units % world;
  const int64_t l = rank * base + std::min<int64_t>(rank, rem);
  *lo = l;
  *hi = l + base + (rank < rem ? 1 : 0);
}

const char* sqngd_last_error(sqngd_ctx ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

}  // extern "C"

// internal accessors for run.cu (C++ linkage, not part of the C-ABI)
const sqngd_config* sq_ctx_config(sqngd_ctx ctx) { return &ctx->cfg; }
int sq_ctx_device(sqngd_ctx ctx) { return ctx->dev; }
sqngd_status sq_ctx_fail(sqngd_ctx ctx, sqngd_status st, const char* what, const char* why) {
  return fail(ctx, st, what, why);
}
void* sq_ctx_run_ws(sqngd_ctx ctx, size_t dev_bytes, void** host, size_t host_bytes) {
  if (dev_bytes > ctx->run_dev_bytes) {
    if (ctx->run_dev) cudaFree(ctx->run_dev);
    ctx->run_dev = nullptr;
    ctx->run_dev_bytes = 0;
    if (ctx->dmalloc(&ctx->run_dev, dev_bytes) != cudaSuccess) return nullptr;
    ctx->run_dev_bytes = dev_bytes;
  }
  if (host_bytes > ctx->run_host_bytes) {
    if (ctx->run_host) cudaFreeHost(ctx->run_host);
    ctx->run_host = nullptr;
    ctx->run_host_bytes = 0;
    if (cudaMallocHost(&ctx->run_host, host_bytes) != cudaSuccess) return nullptr;
    ctx->run_host_bytes = host_bytes;
  }
  *host = ctx->run_host;
  return ctx->run_dev;
}

extern "C" {

}  // extern "C"

static sqngd_status create_impl(const sqngd_config* cfgp, int cuda_device, const void* nccl_unique_id, LoopGroup* group,
                                int rank, int world, sqngd_ctx* out) {
  sqngd_ctx ctx = nullptr;
  if (!cfgp || !out) return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: null argument");
  *out = nullptr;
  const sqngd_config cfg = *cfgp;
  if (cfg.R < 1 || cfg.M < 1 || cfg.N < 2 || cfg.N > 4096 || cfg.B < 2 || cfg.r_n < 1 || cfg.K < 1 ||
      !(cfg.c > 0) || cfg.loss_mode < 0 || cfg.loss_mode > 2)
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: dims (need R,M>=1, 2<=N<=4096, B>=2, r_n>=1, K>=1, c>0)");
  if (cfg.tau_lo < -(cfg.N - 1) || cfg.tau_hi > cfg.N - 1 || cfg.tau_lo > cfg.tau_hi)
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: ROI lags outside [-(N-1), N-1]");
  if (cfg.loss_mode != 0 && !(cfg.beta_or_p > 0))
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: beta_or_p must be > 0 for LSE / PNORM");
  if (cfg.B * cfg.r_n > 8192) return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: B*r_n > 8192");
  if (cfg.map_ld != 0 && cfg.map_ld < 2 * cfg.N - 1)
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: map_ld must be 0 or >= 2N-1");
  if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: rank/world");
  if (cfg.doppler_engine < 0 || cfg.doppler_engine > 2)
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: doppler_engine");
  NetDims nd{};
  if (cfg.net_width != 0) {
    const char* why = "";
    if (!net_dims(cfg.R, cfg.M * cfg.N, cfg.net_width, cfg.net_depth, &nd, &why) || !(cfg.lr_theta >= 0))
      return fail(nullptr, SQNGD_E_INVALID, "sqngd_create", cfg.lr_theta >= 0 ? why : "lr_theta");
  }
  const int L = 2 * cfg.N - 1;
  if ((double)cfg.M * cfg.M * L * cfg.K >= 4294967295.0)
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: M^2 (2N-1) K cell index exceeds 32 bits");

  ctx = new sqngd_ctx_s();
  if (const char* e = getenv("SQNGD_GUARD")) ctx->guard = e[0] == '1';
  ctx->cfg = cfg;
  ctx->dev = cuda_device;
  ctx->rank = rank;
  ctx->world = world;
  ctx->L = L;
  ctx->BR = cfg.B * cfg.r_n;
  int P = 1;
  while (P < L) P <<= 1;
  ctx->P = P;

  // ROI cell count |S| and flags (host copy of the weights, if any)
  {
    std::vector<float> wts;
    if (cfg.weights) {
      wts.resize((size_t)cfg.K * L);
      if (cudaSetDevice(cuda_device) != cudaSuccess ||
          cudaMemcpy(wts.data(), cfg.weights, wts.size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess) {
        delete ctx;
        return fail(nullptr, SQNGD_E_CUDA, "sqngd_create: reading weights");
      }
    }
    uint64_t cells = 0;
    for (int m = 0; m < cfg.M; ++m)
      for (int l = 0; l < cfg.M; ++l)
        for (int tau = cfg.tau_lo; tau <= cfg.tau_hi; ++tau) {
          if (m == l && cfg.exclude_auto_zero_delay && tau == 0) continue;
          for (int k = 0; k < cfg.K; ++k)
            if (!cfg.weights || wts[(size_t)k * L + tau + cfg.N - 1] > 0.f) ++cells;
        }
    if (cells == 0) {
      delete ctx;
      return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: empty ROI");
    }
    ctx->n_cells = (uint32_t)std::min<uint64_t>(cells, 0xFFFFFFFFu);
    if (cfg.M == 1) ctx->flags |= SQNGD_FLAG_NO_CROSS;
    if (std::max(std::fabs(cfg.f_lo), std::fabs(cfg.f_hi)) > 0.5 * cfg.N) ctx->flags |= SQNGD_FLAG_DOPPLER_ALIAS;
  }

  CK(cudaSetDevice(cuda_device));
  CK(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, cuda_device));
  int bps[3] = {1, 1, 1}, G = 1;
  cudaError_t perr = cudaSuccess;
  std::vector<float2> ftw_host, ftwr_host, ftwn_host;
  bool okP = with_P(P, [&](auto Lc) {
    using LC = decltype(Lc);
    perr = LC::prepare(bps);
    G = LC::groups_per_block();
    ftw_host = LC::twiddles();
    ftwr_host = LC::twiddles_r();
    ftwn_host = LC::twiddles_n();
  });
  if (!okP) {
    delete ctx;
    return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: unsupported FFT length");
  }
  if (perr != cudaSuccess) {
    std::string m = cudaGetErrorString(perr);
    delete ctx;
    return fail(nullptr, SQNGD_E_CUDA, "sqngd_create: kernel setup", m.c_str());
  }
  for (int md = 0; md < 3; ++md) ctx->slots[md] = (int64_t)ctx->sms * std::max(1, bps[md]) * G;
  ctx->units = (int64_t)cfg.R * cfg.M * cfg.K;

  // Doppler engine (include/sqngd.h SQNGD_ENGINE_*): node count Q for lr_tol, tables, unit split.
  std::vector<double> lr_fq, lr_ell;
  if (cfg.doppler_engine != SQNGD_ENGINE_FFT && cfg.K >= 3) {
    const double tol = cfg.lr_tol > 0 ? cfg.lr_tol : 1e-7;
    for (int Q = 4; Q <= 16; Q += 2) {
      const double err = lr_tables(cfg, Q, lr_fq, lr_ell);
      if (err <= tol) {
        ctx->Q = Q;
        ctx->lr_err = err;
        break;
      }
    }
    ctx->lr = ctx->Q > 0 && (cfg.doppler_engine == SQNGD_ENGINE_CHEBYSHEV || 3 * ctx->Q <= cfg.K);
  }
  if (cfg.doppler_engine == SQNGD_ENGINE_CHEBYSHEV && !ctx->lr) {
    delete ctx;
    return fail(nullptr, SQNGD_E_INVALID,
                "sqngd_create: CHEBYSHEV engine needs K >= 3 and <= 16 nodes for lr_tol");
  }
  if (ctx->lr) {
    ctx->QS = (ctx->Q + 3) & ~3;
    ctx->nch = (L + 31) / 32;
    ctx->LS = ctx->nch * 32;
    ctx->nch16 = (L + 15) / 16;
    const int Kp = cfg.K / 2;
    ctx->NT = (Kp + 7) / 8;
    ctx->NTF = Kp / 8;
    ctx->units_lr = (int64_t)cfg.R * cfg.M * cfg.M * ctx->nch16;
    cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
    with_Q(ctx->Q, [&](auto Qc) { e1 = decltype(Qc)::prepare_t(0); });
    ctx->kw = 1;      // measured (C3): one warp per unit is best for k_lrt (no CTA-level reduction)
    ctx->lr_smem = 0;
    with_P(P, [&](auto Lc) { e2 = decltype(Lc)::prepare_lr(); });
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      std::string m = cudaGetErrorString(e1 != cudaSuccess ? e1 : e2);
      delete ctx;
      return fail(nullptr, SQNGD_E_CUDA, "sqngd_create: Chebyshev kernel setup", m.c_str());
    }
  }

  const size_t RMN = (size_t)cfg.R * cfg.M * cfg.N;
  CK(ctx->dmalloc(&ctx->tw, sizeof(float2) * (size_t)cfg.K * cfg.N));
  CK(ctx->dmalloc(&ctx->H, sizeof(float2) * (size_t)cfg.R * cfg.M * P));
  // X cache: K bins (FFT engine) or Q nodes (Chebyshev engine; Q may exceed K when forced)
  CK(ctx->dmalloc(&ctx->Xc, sizeof(float2) * (size_t)cfg.R * cfg.M * std::max(cfg.K, ctx->Q) * P));
  CK(ctx->dmalloc(&ctx->ftw, sizeof(float2) * ftw_host.size()));
  CK(cudaMemcpy(ctx->ftw, ftw_host.data(), sizeof(float2) * ftw_host.size(), cudaMemcpyHostToDevice));
  CK(ctx->dmalloc(&ctx->ftwn, sizeof(float2) * ftwn_host.size()));
  CK(cudaMemcpy(ctx->ftwn, ftwn_host.data(), sizeof(float2) * ftwn_host.size(), cudaMemcpyHostToDevice));
  CK(ctx->dmalloc(&ctx->ftwr, sizeof(float2) * ftwr_host.size()));
  CK(cudaMemcpy(ctx->ftwr, ftwr_host.data(), sizeof(float2) * ftwr_host.size(), cudaMemcpyHostToDevice));
  const int64_t uslots = std::max(ctx->units, ctx->units_lr);
  const int64_t gslots = std::max(ctx->units, ctx->lr ? (int64_t)cfg.R * cfg.M * cfg.M * ctx->Q : (int64_t)0);
  CK(ctx->dmalloc(&ctx->part.scale, sizeof(float) * uslots));
  // [0]: the FFT engine's dynamic unit counter; [1]: unused; [2, 2 + 2R): the per-restart tie words
  // (KP::tiew), zeroed together with the counter before every FFT-engine launch
  CK(ctx->dmalloc(&ctx->counter, (2 + 2 * (size_t)cfg.R) * sizeof(int)));
  CK(ctx->dmalloc(&ctx->d_t, 2 * sizeof(long long)));
  CK(ctx->dmalloc(&ctx->snrl_w, sizeof(double) * cfg.R));
  ctx->cts = std::max(1, std::max(cfg.n_h, cfg.n_x));
  CK(ctx->dmalloc(&ctx->d_ct, 2 * sizeof(float2) * ctx->cts));
  if (const char* e = getenv("SQNGD_NO_GRAPH")) ctx->use_graphs = !(e[0] == '1');
  CK(ctx->dmalloc(&ctx->spec, sizeof(float2) * (size_t)cfg.R * cfg.M * P));
  CK(ctx->dmalloc(&ctx->s_soft, sizeof(float2) * RMN));
  CK(ctx->dmalloc(&ctx->s_hard, sizeof(float2) * RMN));
  CK(ctx->dmalloc(&ctx->dq, sizeof(float) * RMN));
  CK(ctx->dmalloc(&ctx->lut, sizeof(int) * (size_t)cfg.R * (ctx->BR + 1)));
  CK(ctx->dmalloc(&ctx->part.key, sizeof(unsigned long long) * 2 * uslots));
  CK(ctx->dmalloc(&ctx->part.m, sizeof(float) * uslots));
  CK(ctx->dmalloc(&ctx->part.S, sizeof(float) * uslots));
  CK(ctx->dmalloc(&ctx->part.g, sizeof(float2) * (size_t)gslots * P));
  CK(ctx->dmalloc(&ctx->red, sizeof(Red) * cfg.R));
  CK(ctx->dmalloc(&ctx->cm, sizeof(double2) * cfg.R * cfg.M));
  CK(ctx->dmalloc(&ctx->red_grad, sizeof(float2) * RMN));
  CK(ctx->dmalloc(&ctx->dy, sizeof(float) * RMN));
  {  // Adam(rho) + projection: 2 n2 floats of dynamic shared memory (64 KB at B r_n = 8192, above
     // the 48 KB a launch gets without opting in)
    int n2 = 1;
    while (n2 < ctx->BR) n2 <<= 1;
    CK(cudaFuncSetAttribute(k_adam_project_rho, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(2 * n2 * sizeof(float))));
  }
  CK(ctx->dmalloc(&ctx->gw, sizeof(float2) * RMN));
  CK(ctx->dmalloc(&ctx->gz, sizeof(float) * RMN));
  CK(ctx->dmalloc(&ctx->grho, sizeof(float) * (size_t)cfg.R * ctx->BR));
  CK(ctx->dmalloc(&ctx->met, sizeof(MetricsOut) * cfg.R));
  CK(ctx->dmalloc(&ctx->status, sizeof(int)));
  CK(cudaMemset(ctx->status, 0, sizeof(int)));
  if (cfg.net_width != 0) {
    ctx->net = true;
    ctx->nd = nd;
    CK(ctx->dmalloc(&ctx->net_ws, sizeof(float) * net_ws_floats(nd)));
    ctx->nws = net_ws_carve(nd, ctx->net_ws);
    CK(net_prepare(nd));
    CK(cudaStreamCreateWithFlags(&ctx->side_net, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_nf, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_nj, cudaEventDisableTiming));
  }

  // Doppler twiddles e^{j 2 pi n f_k / N}, n one-based (Eq. 33, Q2), phase reduced mod 1 in fp64.
  {
    std::vector<float2> tw((size_t)cfg.K * cfg.N);
    for (int k = 0; k < cfg.K; ++k) {
      const double f = cfg.K == 1 ? cfg.f_lo : cfg.f_lo + (cfg.f_hi - cfg.f_lo) * (double)k / (double)(cfg.K - 1);
      for (int n = 0; n < cfg.N; ++n) {
        double cyc = (double)(n + 1) * f / (double)cfg.N;
        cyc -= std::floor(cyc);
        tw[(size_t)k * cfg.N + n] = make_float2((float)std::cos(2.0 * M_PI * cyc), (float)std::sin(2.0 * M_PI * cyc));
      }
    }
    CK(cudaMemcpy(ctx->tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }

  if (ctx->lr) {  // Chebyshev engine tables (fp64-built) and node buffers
    const int Q = ctx->Q, QH = Q / 2, Kp = cfg.K / 2;
    const double nc = 0.5 * (cfg.N + 1);
    std::vector<float2> vt((size_t)Q * cfg.N);
    for (int q = 0; q < Q; ++q)
      for (int n = 0; n < cfg.N; ++n) {  // V_q(n) = e^{j 2 pi (n - n_c) f*_q / N}, n one-based (Q2)
        double cyc = ((double)(n + 1) - nc) * lr_fq[q] / (double)cfg.N;
        cyc -= std::floor(cyc);
        vt[(size_t)q * cfg.N + n] = make_float2((float)std::cos(2.0 * M_PI * cyc), (float)std::sin(2.0 * M_PI * cyc));
      }
    std::vector<float> cf((size_t)(Kp + 1) * ctx->QS, 0.f);
    for (int p = 0; p < Kp; ++p)
      for (int j = 0; j < QH; ++j) {
        const double a = lr_ell[(size_t)p * Q + j], b = lr_ell[(size_t)p * Q + Q - 1 - j];
        cf[(size_t)p * ctx->QS + j] = (float)(0.5 * (a + b));       // alpha_j
        cf[(size_t)p * ctx->QS + QH + j] = (float)(0.5 * (a - b));  // beta_j
      }
    if (cfg.K & 1)
      for (int j = 0; j < QH; ++j) cf[(size_t)Kp * ctx->QS + j] = (float)lr_ell[(size_t)Kp * Q + j];
    CK(ctx->dmalloc(&ctx->Vt, sizeof(float2) * vt.size()));
    CK(cudaMemcpy(ctx->Vt, vt.data(), sizeof(float2) * vt.size(), cudaMemcpyHostToDevice));
    CK(ctx->dmalloc(&ctx->coef, sizeof(float) * cf.size()));
    CK(cudaMemcpy(ctx->coef, cf.data(), sizeof(float) * cf.size(), cudaMemcpyHostToDevice));
    {  // k_lrt B fragments: alpha / beta per (j, pair), TF32 hi + lo, in mma.sync m16n8k8 lane order
      auto alpha = [&](int j, int p) -> double {
        if (j >= QH || p >= Kp) return 0.0;
        return 0.5 * (lr_ell[(size_t)p * Q + j] + lr_ell[(size_t)p * Q + Q - 1 - j]);
      };
      auto beta = [&](int j, int p) -> double {
        if (j >= QH || p >= Kp) return 0.0;
        return 0.5 * (lr_ell[(size_t)p * Q + j] - lr_ell[(size_t)p * Q + Q - 1 - j]);
      };
      auto tf32 = [](double x, float& hi, float& lo) {  // cvt.rna.tf32: round to nearest, ties away
        float f = (float)x;
        uint32_t u;
        std::memcpy(&u, &f, 4);
        u = (u + 0x1000u) & 0xFFFFE000u;
        std::memcpy(&hi, &u, 4);
        lo = (float)(x - (double)hi);
      };
      auto frag = [&](double b0, double b1) {
        float4 o;
        tf32(b0, o.x, o.z);
        tf32(b1, o.y, o.w);
        return o;
      };
      std::vector<float4> tf((size_t)ctx->NT * 64), ta((size_t)ctx->NT * 64);
      for (int t = 0; t < ctx->NT; ++t)
        for (int ln = 0; ln < 32; ++ln) {
          const int gg = ln >> 2, cc = ln & 3;
          const size_t o = ((size_t)t * 32 + ln) * 2;
          tf[o] = frag(alpha(cc, 8 * t + gg), alpha(cc + 4, 8 * t + gg));
          tf[o + 1] = frag(beta(cc, 8 * t + gg), beta(cc + 4, 8 * t + gg));
          ta[o] = frag(alpha(gg, 8 * t + 2 * cc), alpha(gg, 8 * t + 2 * cc + 1));
          ta[o + 1] = frag(beta(gg, 8 * t + 2 * cc), beta(gg, 8 * t + 2 * cc + 1));
        }
      {  // FP16 packed-split forward fragments (m16n8k16): K rows [hi(c) ; hi(c) ; lo(c) ; 0]
        auto f16 = [](double x) -> uint16_t { return __half_as_ushort(__float2half_rn((float)x)); };
        auto split16 = [&](double x, int part) -> uint16_t {  // part 0: hi, 1: hi (for x_lo), 2: lo
          const __half h = __float2half_rn((float)x);
          if (part < 2) return __half_as_ushort(h);
          return f16(x - (double)__half2float(h));
        };
        // K row k (k_lrt layout): lane c = (k mod 8) / 2 owns node pair j = c; rows 2c, 2c+1 hold
        // hi(c_c) (against hi(x_c), lo(x_c)), row 2c+8 lo(c_c) (against hi(x_c)), row 2c+9 the
        // pair j = 4 share: hi(c_4), hi(c_4), lo(c_4), 0 for c = 0..3.
        auto Bk = [&](int k, int p, bool is_alpha, bool mid) -> uint16_t {  // B[k][pair p]
          const int cc = (k & 7) >> 1, t = k & 1, hi_half = k >> 3;
          int j = cc, part = hi_half ? 2 : 0;
          if (hi_half && t) {
            if (cc == 3) return 0;
            j = 4;
            part = cc == 2 ? 2 : 0;
          }
          if (j >= QH) return 0;
          double c;
          if (mid) c = lr_ell[(size_t)Kp * Q + j];
          else c = is_alpha ? alpha(j, p) : beta(j, p);
          return split16(c, part);
        };
        auto pack = [](uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); };
        std::vector<uint4> t16((size_t)ctx->NT * 32);
        std::vector<uint2> m16(32);
        for (int t = 0; t < ctx->NT; ++t)
          for (int ln = 0; ln < 32; ++ln) {
            const int gg = ln >> 2, cc = ln & 3, p = 8 * t + gg;
            t16[(size_t)t * 32 + ln] = make_uint4(pack(Bk(2 * cc, p, true, false), Bk(2 * cc + 1, p, true, false)),
                                                  pack(Bk(2 * cc + 8, p, true, false), Bk(2 * cc + 9, p, true, false)),
                                                  pack(Bk(2 * cc, p, false, false), Bk(2 * cc + 1, p, false, false)),
                                                  pack(Bk(2 * cc + 8, p, false, false), Bk(2 * cc + 9, p, false, false)));
          }
        for (int ln = 0; ln < 32; ++ln) {
          const int gg = ln >> 2, cc = ln & 3;
          const bool col0 = gg == 0 && (cfg.K & 1);
          m16[ln] = make_uint2(col0 ? pack(Bk(2 * cc, 0, true, true), Bk(2 * cc + 1, 0, true, true)) : 0u,
                               col0 ? pack(Bk(2 * cc + 8, 0, true, true), Bk(2 * cc + 9, 0, true, true)) : 0u);
        }
        CK(ctx->dmalloc(&ctx->tabF16, sizeof(uint4) * t16.size()));
        CK(cudaMemcpy(ctx->tabF16, t16.data(), sizeof(uint4) * t16.size(), cudaMemcpyHostToDevice));
        CK(ctx->dmalloc(&ctx->tabM16, sizeof(uint2) * 32));
        CK(cudaMemcpy(ctx->tabM16, m16.data(), sizeof(uint2) * 32, cudaMemcpyHostToDevice));
      }
      // k_lrf (tcgen05 forward): per 32-pair chunk c, two 64 x 16 fp16 images in the canonical K-major
      // layout (lrf_off): row n = output column (n < 32: A0 of pair 32c + n, else A1 of pair 32c + n - 32),
      // K = [hi(c_j) j<5 | hi(c_j) | lo(c_j) | 0]; B_E holds alpha, B_O holds +beta (A0) / -beta (A1).
      if (QH <= 5 && Kp >= 1) {
        ctx->nc128 = (L + kLrfRows - 1) / kLrfRows;
        ctx->npc = (Kp + kLrfPairs - 1) / kLrfPairs;
        std::vector<uint8_t> img((size_t)ctx->npc * 2 * kLrfImgB, 0);
        for (int cch = 0; cch < ctx->npc; ++cch)
          for (int e = 0; e < 2; ++e)
            for (int n = 0; n < 2 * kLrfPairs; ++n) {
              const int p = cch * kLrfPairs + (n % kLrfPairs);
              if (p >= Kp) continue;
              const double sg = (e == 1 && n >= kLrfPairs) ? -1.0 : 1.0;
              for (int j = 0; j < QH; ++j) {
                const double cv = sg * (e == 0 ? alpha(j, p) : beta(j, p));
                const __half h = __float2half_rn((float)cv);
                const __half lo = __float2half_rn((float)(cv - (double)__half2float(h)));
                const uint16_t parts[3] = {__half_as_ushort(h), __half_as_ushort(h), __half_as_ushort(lo)};
                for (int t3 = 0; t3 < 3; ++t3) {
                  const uint32_t off = (uint32_t)(cch * 2 + e) * kLrfImgB + lrf_off(n, 5 * t3 + j);
                  std::memcpy(&img[off], &parts[t3], 2);
                }
              }
            }
        CK(ctx->dmalloc(&ctx->tabB, img.size()));
        CK(cudaMemcpy(ctx->tabB, img.data(), img.size(), cudaMemcpyHostToDevice));
        ctx->lrf_smem = lrf_smem_bytes(ctx->npc, QH);
        ctx->use_lrf = ctx->lrf_smem <= 200 * 1024;
        if (const char* ev = getenv("SQNGD_LRF")) ctx->use_lrf = ctx->use_lrf && ev[0] != '0';
        if (ctx->use_lrf) CK(LrfLaunch::prepare(ctx->lrf_smem));
      }
      CK(ctx->dmalloc(&ctx->tabF, sizeof(float4) * tf.size()));
      CK(cudaMemcpy(ctx->tabF, tf.data(), sizeof(float4) * tf.size(), cudaMemcpyHostToDevice));
      CK(ctx->dmalloc(&ctx->tabA, sizeof(float4) * ta.size()));
      CK(cudaMemcpy(ctx->tabA, ta.data(), sizeof(float4) * ta.size(), cudaMemcpyHostToDevice));
    }
    std::vector<float> wm((size_t)L, 1.f);
    if (cfg.weights) {
      std::vector<float> wts((size_t)cfg.K * L);
      CK(cudaMemcpy(wts.data(), cfg.weights, wts.size() * sizeof(float), cudaMemcpyDeviceToHost));
      for (int i = 0; i < L; ++i) {
        float mx = 0.f;
        for (int k = 0; k < cfg.K; ++k) mx = std::max(mx, wts[(size_t)k * L + i]);
        wm[i] = mx;
      }
    }
    CK(ctx->dmalloc(&ctx->wmax, sizeof(float) * L));
    CK(cudaMemcpy(ctx->wmax, wm.data(), sizeof(float) * L, cudaMemcpyHostToDevice));
    const size_t pairs = (size_t)cfg.R * cfg.M * cfg.M;
    CK(ctx->dmalloc(&ctx->Rn, sizeof(float2) * pairs * Q * ctx->LS));
    CK(ctx->dmalloc(&ctx->Gn, sizeof(float2) * pairs * Q * ctx->LS));
    CK(ctx->dmalloc(&ctx->lred, sizeof(LrRed) * cfg.R));
    CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    // (splitting each node's l sum over 2 CTAs to fill more SMs at C3 (80 nodes) measured no gain:
    // 10543 vs 10685 evals/s; lsplit stays 1)
    CK(ctx->dmalloc(&ctx->tslot, sizeof(float2) * (size_t)cfg.R * cfg.M * Q * ctx->lsplit * ((cfg.N + 1) & ~1)));
  }

  {  // this rank's shard of the Chebyshev engine's (restart, transmit channel) rows
    int64_t lo, hi;
    sqngd_shard_range((int64_t)cfg.R * cfg.M, rank, world, &lo, &hi);
    ctx->row_lo = (int)lo;
    ctx->row_hi = (int)hi;
  }
  // One grouped collective per evaluation (comm.h) for world > 1.  With world == 1 an ncclUniqueId
  // still selects the collective path over a 1-rank NCCL communicator: the same code (pack, grouped
  // NCCL calls captured in the step graph, unpack) runs on one GPU.
  if (world > 1 || nccl_unique_id) {
    ctx->multi = true;
    CK(ctx->dmalloc(&ctx->pay, sizeof(double) * (size_t)cfg.R * (1 + 2 * (size_t)cfg.M * cfg.N)));
    CK(ctx->dmalloc(&ctx->keyb, sizeof(unsigned long long) * 3 * cfg.R));
    CK(ctx->dmalloc(&ctx->mref, sizeof(double) * cfg.R));
    k_world_init<<<(cfg.R + 127) / 128, 128>>>(cfg.R, cfg.loss_mode, ctx->mref);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::string why;
    if (group) {
      LoopComm* lc = new LoopComm();
      lc->g = group;
      lc->rank = rank;
      lc->status = ctx->status;
      lc->cap_sum = (size_t)cfg.R * (1 + 2 * (size_t)cfg.M * cfg.N);
      lc->cap_max = (size_t)3 * cfg.R;
      ctx->comm = lc;
    } else {
      if (!nccl_unique_id) {
        sqngd_destroy(ctx);
        return fail(nullptr, SQNGD_E_INVALID, "sqngd_create: world > 1 needs an ncclUniqueId");
      }
      NcclComm* nc = new NcclComm();
      ctx->comm = nc;
      if (!nc->init(nccl_unique_id, rank, world, &why)) {
        sqngd_destroy(ctx);
        return fail(nullptr, SQNGD_E_NCCL, "sqngd_create: NCCL init", why.c_str());
      }
    }
  }
  *out = ctx;
  return SQNGD_OK;
}

extern "C" {

sqngd_status sqngd_create(const sqngd_config* cfg, int cuda_device, const void* nccl_unique_id, int rank, int world,
                          sqngd_ctx* out) {
  return create_impl(cfg, cuda_device, nccl_unique_id, nullptr, rank, world, out);
}

struct sqngd_loopback_s {
  LoopGroup g;
};

sqngd_loopback sqngd_loopback_create(int world) {
  if (world < 2 || world > kLoopMax) return nullptr;
  sqngd_loopback lb = new sqngd_loopback_s();
  if (!lb->g.init(world)) {
    delete lb;
    return nullptr;
  }
  return lb;
}

void sqngd_loopback_destroy(sqngd_loopback lb) { delete lb; }

sqngd_status sqngd_loopback_set_peer(sqngd_loopback lb, int on) {
  if (!lb) return fail(nullptr, SQNGD_E_INVALID, "sqngd_loopback_set_peer: null group");
  std::unique_lock<std::mutex> lk(lb->g.mu);
  lb->g.peer = on != 0;
  lb->g.peer_fused = on == 2 || on == 3;
  lb->g.drop_signal_rank = on == 3 ? lb->g.world - 1 : -1;
  return SQNGD_OK;
}

sqngd_status sqngd_peer_export(sqngd_ctx ctx, void* handle64) {
  if (!ctx || !handle64) return fail(ctx, SQNGD_E_INVALID, "sqngd_peer_export: null argument");
  if (!ctx->multi || !ctx->comm) return fail(ctx, SQNGD_E_INVALID, "sqngd_peer_export: not a multi-GPU context");
  CK(cudaSetDevice(ctx->dev));
  if (!ctx->peer_pending) {
    ctx->peer_pending = new PeerComm();
    const sqngd_config& c = ctx->cfg;
    cudaError_t e = ctx->peer_pending->own.alloc((size_t)c.R * (1 + 2 * (size_t)c.M * c.N), (size_t)3 * c.R);
    if (e != cudaSuccess) {
      delete ctx->peer_pending;
      ctx->peer_pending = nullptr;
      return fail(ctx, SQNGD_E_NOMEM, "sqngd_peer_export: window", cudaGetErrorString(e));
    }
    CK(cudaDeviceSynchronize());
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->peer_pending->own.base));
  memcpy(handle64, &h, sizeof(h));
  return SQNGD_OK;
}

sqngd_status sqngd_peer_attach(sqngd_ctx ctx, const void* handles) {
  if (!ctx || !handles) return fail(ctx, SQNGD_E_INVALID, "sqngd_peer_attach: null argument");
  if (!ctx->peer_pending) return fail(ctx, SQNGD_E_INVALID, "sqngd_peer_attach: call sqngd_peer_export first");
  CK(cudaSetDevice(ctx->dev));
  std::string why;
  if (!ctx->peer_pending->attach(handles, ctx->rank, ctx->world, ctx->status, &why)) {
    ctx->peer_pending->destroy();
    delete ctx->peer_pending;
    ctx->peer_pending = nullptr;
    return fail(ctx, SQNGD_E_CUDA, "sqngd_peer_attach", why.c_str());
  }
  if (const char* ev = getenv("SQNGD_PEER_FUSED")) ctx->peer_pending->use_fused = !(ev[0] == '0');
  CK(cudaDeviceSynchronize());
  // the step graphs captured so far hold the previous backend's collective: drop them
  ctx->drop_graphs();
  if (ctx->comm) {
    ctx->comm->destroy();
    delete ctx->comm;
  }
  ctx->comm = ctx->peer_pending;
  ctx->peer_pending = nullptr;
  return SQNGD_OK;
}

sqngd_status sqngd_create_loopback(const sqngd_config* cfg, int cuda_device, sqngd_loopback group, int rank,
                                   sqngd_ctx* out) {
  if (!group) return fail(nullptr, SQNGD_E_INVALID, "sqngd_create_loopback: null group");
  return create_impl(cfg, cuda_device, nullptr, &group->g, rank, group->g.world, out);
}

sqngd_status sqngd_check_guards(sqngd_ctx ctx, int64_t* corrupted) {
  if (!ctx || !corrupted) return fail(ctx, SQNGD_E_INVALID, "sqngd_check_guards: null argument");
  *corrupted = -1;
  if (!ctx->guard) return SQNGD_OK;
  CK(cudaSetDevice(ctx->dev));
  CK(cudaDeviceSynchronize());
  const size_t G = sqngd_ctx_s::kGuard;
  std::vector<unsigned char> band(G);
  int64_t bad = 0;
  for (auto& g : ctx->guarded) {
    if (!g.first) continue;
    bool ok = true;
    for (int side = 0; side < 2 && ok; ++side) {
      CK(cudaMemcpy(band.data(), g.first + (side ? G + g.second : 0), G, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < G; ++i)
        if (band[i] != 0x5A) { ok = false; break; }
    }
    bad += ok ? 0 : 1;
  }
  *corrupted = bad;
  return SQNGD_OK;
}

void sqngd_destroy(sqngd_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev);
  ctx->drop_graphs();
  if (ctx->peer_pending) {
    ctx->peer_pending->destroy();
    delete ctx->peer_pending;
    ctx->peer_pending = nullptr;
  }
  void* ptrs[] = {ctx->tabB, ctx->snrl_w, ctx->d_ct, ctx->d_t, ctx->tw, ctx->H, ctx->Xc, ctx->ftw, ctx->part.scale, ctx->counter, ctx->spec, ctx->s_soft, ctx->s_hard, ctx->dq, ctx->lut, ctx->part.key, ctx->part.m,
                  ctx->part.S, ctx->part.g, ctx->red, ctx->cm, ctx->red_grad, ctx->dy,
                  ctx->gw, ctx->gz, ctx->grho, ctx->met, ctx->status, ctx->Vt, ctx->coef, ctx->wmax, ctx->Rn,
                  ctx->Gn, ctx->tslot, ctx->lred, ctx->pay, ctx->keyb, ctx->mref, ctx->tabF, ctx->tabA, ctx->ftwr, ctx->ftwn, ctx->tabF16, ctx->tabM16, ctx->net_ws};
  for (void* p : ptrs) ctx->dfree(p);
  if (ctx->run_dev) ctx->dfree(ctx->run_dev);
  if (ctx->run_host) cudaFreeHost(ctx->run_host);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_nf) cudaEventDestroy(ctx->ev_nf);
  if (ctx->ev_nj) cudaEventDestroy(ctx->ev_nj);
  if (ctx->side_net) cudaStreamDestroy(ctx->side_net);
  if (ctx->comm) {
    ctx->comm->destroy();
    delete ctx->comm;
  }
  delete ctx;
}

sqngd_status sqngd_engine_info(sqngd_ctx ctx, int32_t* engine, int32_t* q_nodes, double* err_bound) {
  if (!ctx) return fail(nullptr, SQNGD_E_INVALID, "sqngd_engine_info: null ctx");
  if (engine) *engine = ctx->lr ? SQNGD_ENGINE_CHEBYSHEV : SQNGD_ENGINE_FFT;
  if (q_nodes) *q_nodes = ctx->lr ? ctx->Q : 0;
  if (err_bound) *err_bound = ctx->lr ? ctx->lr_err : 0.0;
  return SQNGD_OK;
}

sqngd_status sqngd_profile_enable(sqngd_ctx ctx, int on) {
  if (!ctx) return fail(nullptr, SQNGD_E_INVALID, "sqngd_profile_enable: null ctx");
  ctx->prof = on != 0;
  return SQNGD_OK;
}

sqngd_status sqngd_profile_read(sqngd_ctx ctx, double* ms, int64_t* count, int64_t* launches, int reset) {
  if (!ctx) return fail(nullptr, SQNGD_E_INVALID, "sqngd_profile_read: null ctx");
  CK(cudaSetDevice(ctx->dev));
  CK(cudaDeviceSynchronize());
  double acc[4] = {0, 0, 0, 0};
  int64_t cnt[4] = {0, 0, 0, 0};
  for (auto& mk : ctx->ev_marks) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ctx->ev_pool[mk.second], ctx->ev_pool[mk.second + 1]));
    acc[mk.first] += t;
    cnt[mk.first] += 1;
  }
  for (auto* g : ctx->graphs) {  // graphs replayed since the last reset: their latest replay
    if (!g->replayed) continue;
    for (auto& mk : g->marks) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, std::get<1>(mk), std::get<2>(mk)));
      acc[std::get<0>(mk)] += t;
      cnt[std::get<0>(mk)] += 1;
    }
  }
  for (int i = 0; i < 4; ++i) {
    if (ms) ms[i] = acc[i];
    if (count) count[i] = cnt[i];
  }
  if (launches) *launches = ctx->launches;
  if (reset) {
    ctx->ev_marks.clear();
    ctx->ev_used = 0;
    ctx->launches = 0;
    for (auto* g : ctx->graphs) g->replayed = false;
  }
  return SQNGD_OK;
}

sqngd_status sqngd_sync(sqngd_ctx ctx, sqngd_stream stream) {
  if (!ctx) return fail(nullptr, SQNGD_E_INVALID, "sqngd_sync: null ctx");
  CK(cudaSetDevice(ctx->dev));
  CK(cudaStreamSynchronize(S(stream)));
  int st = 0;
  CK(cudaMemcpy(&st, ctx->status, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemset(ctx->status, 0, sizeof(int)));
  // (first: without the combine everything downstream is a symptom)
  if (st & kPeerTimeoutBit) return fail(ctx, SQNGD_E_NCCL, "peer all-reduce: a rank did not signal in time");
  if (st & ST_NONFINITE) return fail(ctx, SQNGD_E_NONFINITE, "non-finite loss or gradient");
  if (st & ST_DEGENERATE) return fail(ctx, SQNGD_E_DEGENERATE, "degenerate mainlobe or zero-energy filter");
  if (st & ST_INVALID) return fail(ctx, SQNGD_E_INVALID, "thresholds rho not ascending");
  return SQNGD_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------- internal pipeline
static sqngd_status launch_check(sqngd_ctx ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, SQNGD_E_CUDA, what, cudaGetErrorString(e));
  return SQNGD_OK;
}

static sqngd_status run_quantize(sqngd_ctx ctx, const float* z, const float* rho, float2* s_soft, float2* s_hard,
                                 uint8_t* b_hard, float* dq, cudaStream_t st) {
  const sqngd_config& c = ctx->cfg;
  if (s_hard || b_hard) {
    k_hard_lut<<<dim3((ctx->BR + 1 + 7) / 8, c.R), 256, ctx->BR * sizeof(float), st>>>(c.B, ctx->BR, c.c, rho, ctx->lut,
                                                                                        ctx->status);
    ctx->launches += 1;
  }
  ctx->launches += 1;
  const int MN = c.M * c.N;
  k_quantize<<<dim3((MN + 31) / 32, c.R), 256, ctx->BR * sizeof(float), st>>>(MN, c.B, ctx->BR, (float)c.c, z, rho,
                                                                                ctx->lut, s_soft, s_hard, b_hard, dq);
  return launch_check(ctx, "quantize");
}

// a2 (+ a6 when s is given): H = FFT(w)/P and c_m = sum_n s_m conj(w_m).
static sqngd_status run_filter_fft(sqngd_ctx ctx, const float2* w, cudaStream_t st, const float2* s = nullptr) {
  const sqngd_config& c = ctx->cfg;
  with_P(ctx->P, [&](auto Lc) { decltype(Lc)::filter(c.R * c.M, c.N, w, ctx->ftw, ctx->H, s, ctx->cm, st); });
  ctx->launches += 1;
  return launch_check(ctx, "filter fft");
}

// a3 (+ a6 when w is given): X cache of the waveform s over this rank's units (Chebyshev engine: the
// Q node modulations V_q of its rows instead of the K bins).
// full: the FFT engine's Step-A units (r, l, k) read X_{m,k} of every channel m, so with world > 1 its
// Step-A X cache is computed for all units (replicated a3 work, 1/(M+1) of its transforms); the
// forward and Step B read only their own units (r, m, k), the Chebyshev engine only its own rows.
static sqngd_status run_xhat(sqngd_ctx ctx, const float2* s, cudaStream_t st, const float2* w = nullptr,
                             bool full = false) {
  const sqngd_config& c = ctx->cfg;
  int u0, units;
  if (ctx->lr) {
    u0 = ctx->row_lo * ctx->Q;
    units = (ctx->row_hi - ctx->row_lo) * ctx->Q;
  } else if (full) {
    u0 = 0;
    units = c.R * c.M * c.K;
  } else {
    KP kp = make_kp(ctx, 0);
    u0 = kp.u_lo;
    units = kp.u_hi - kp.u_lo;
  }
  if (units <= 0) return SQNGD_OK;
  with_P(ctx->P, [&](auto Lc) {
    if (ctx->lr) decltype(Lc)::xhat_n(u0, units, c.M, c.N, ctx->Q, s, ctx->Vt, ctx->ftwn, ctx->Xc, w, ctx->cm, st);
    else decltype(Lc)::xhat(u0, units, c.M, c.N, c.K, s, ctx->tw, ctx->ftw, ctx->Xc, w, ctx->cm, st);
  });
  ctx->launches += 1;
  return launch_check(ctx, "xhat");
}

// ---------------------------------------------------------------- multi-GPU (world > 1, comm.h)
// c_m of every row (the shard's transforms computed only its own rows' c_m).
static sqngd_status run_cm_rows(sqngd_ctx ctx, const float2* s, const float2* w, cudaStream_t st) {
  const sqngd_config& c = ctx->cfg;
  const int RM = c.R * c.M;
  k_cm_rows<<<(RM + 7) / 8, 256, 0, st>>>(RM, c.N, s, w, ctx->cm);
  ctx->launches += 1;
  return launch_check(ctx, "cm rows");
}

// The one grouped collective of an evaluation: local (m_r, S_r, keys) in ctx->red and, with a gradient,
// the locally normalised partial in ctx->red_grad -> global red and red_grad on every rank.
static sqngd_status world_combine(sqngd_ctx ctx, bool with_grad, cudaStream_t st) {
  const sqngd_config& c = ctx->cfg;
  WorldArgs wa{};
  wa.R = c.R; wa.M = c.M; wa.N = c.N; wa.mode = c.loss_mode; wa.with_grad = with_grad ? 1 : 0;
  wa.bp = c.beta_or_p; wa.red = ctx->red; wa.mref = ctx->mref; wa.grad = ctx->red_grad; wa.pay = ctx->pay;
  wa.key = ctx->keyb;
  const size_t n = with_grad ? (size_t)2 * c.M * c.N : 0;
  if (ctx->comm->has_fused()) {  // pack + all-reduce over peer memory + unpack in one kernel (world_peer.cuh)
    std::string why;
    if (!ctx->comm->fused(&wa, st, &why)) return fail(ctx, SQNGD_E_NCCL, "fused peer combine", why.c_str());
    ctx->launches += 1;
    return launch_check(ctx, "world peer");
  }
  const dim3 grid((unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 256)), c.R);
  k_world_pack<<<grid, 256, 0, st>>>(wa);
  sqngd_status rc = launch_check(ctx, "world pack");
  if (rc) return rc;
  std::string why;
  if (!ctx->comm->allreduce(ctx->pay, (size_t)c.R * (1 + n), ctx->keyb, (size_t)3 * c.R, st, &why))
    return fail(ctx, SQNGD_E_NCCL, "grouped all-reduce", why.c_str());
  // (the payload stride is 1 + n per restart: pack and unpack agree on it)
  k_world_unpack<<<grid, 256, 0, st>>>(wa, ctx->status);
  ctx->launches += 2;
  return launch_check(ctx, "world unpack");
}

// Chebyshev engine, forward part: node AFs (k_node) and the fused contraction / epilogue (k_lrt), then
// the per-restart reduction (keys, shift, S, metrics) -- over this rank's rows.
static sqngd_status run_lr(sqngd_ctx ctx, bool grad, int cls, float* af_mag, const MetricsArgs& ma, cudaStream_t st,
                           bool fork) {
  const sqngd_config& c = ctx->cfg;
  const int rows = ctx->row_hi - ctx->row_lo;
  with_P(ctx->P, [&](auto Lc) {
    decltype(Lc)::node(ctx->row_lo * c.M * ctx->Q, std::max(1, rows * c.M * ctx->Q), c.M, ctx->Q, c.N, ctx->LS,
                       ctx->Xc, ctx->H, ctx->ftwn, ctx->Rn, c.R, ctx->lred, st);
  });
  LrtArgs t{};
  t.R = c.R; t.M = c.M; t.N = c.N; t.L = ctx->L; t.K = c.K; t.nch = ctx->nch16; t.kw = ctx->kw; t.LS = ctx->LS;
  t.NT = ctx->NT; t.NTF = ctx->NTF; t.coefm = ctx->coef + (size_t)(c.K / 2) * ctx->QS;
  t.tabF16 = ctx->tabF16; t.tabM16 = ctx->tabM16; t.row0 = ctx->row_lo;
  t.tau_lo = c.tau_lo; t.tau_hi = c.tau_hi; t.excl0 = c.exclude_auto_zero_delay;
  t.bp = (float)c.beta_or_p; t.invN = 1.0f / (float)c.N;
  t.weights = c.weights; t.wmax = ctx->wmax; t.tabF = ctx->tabF; t.tabA = ctx->tabA; t.Rn = ctx->Rn; t.Gn = ctx->Gn;
  t.af_mag = grad ? nullptr : af_mag; t.part = ctx->part; t.lred = ctx->lred;
  t.mld = c.map_ld > 0 ? c.map_ld : ctx->L;
  // the tcgen05 forward (lr_tc.cuh) where it measured faster: writing the dense |A| map (C3: 65 vs 75 us;
  // its map stores are 32 consecutive lags of one bin per warp).  Without a map, or with a pitched map,
  // the mma.sync kernel is faster (35 vs 42 us; 49 vs 65 us): DESIGN.md §6 "tcgen05 forward".
  const bool tc = !grad && ctx->use_lrf && af_mag != nullptr && c.map_ld == 0;
  {
    ProfScope ps(ctx, cls, st);
    if (tc) {
      LrfArgs f{};
      f.M = c.M; f.N = c.N; f.L = ctx->L; f.K = c.K; f.Kp = c.K / 2; f.Q = ctx->Q; f.nc = ctx->nc128;
      f.npc = ctx->npc; f.row0 = ctx->row_lo; f.tau_lo = c.tau_lo; f.tau_hi = c.tau_hi;
      f.excl0 = c.exclude_auto_zero_delay; f.LS = ctx->LS; f.mld = t.mld; f.bp = t.bp; f.invN = t.invN;
      f.weights = c.weights; f.wmax = ctx->wmax; f.coefm = t.coefm; f.tabB = ctx->tabB; f.Rn = ctx->Rn;
      f.af_mag = af_mag; f.part = ctx->part; f.lred = ctx->lred;
      LrfLaunch::launch(c.loss_mode, c.weights != nullptr, af_mag != nullptr, f, rows, ctx->lrf_smem, st);
    } else {
      with_Q(ctx->Q, [&](auto Qc) {
        decltype(Qc)::launch_t(c.loss_mode, c.weights != nullptr, grad ? 1 : (af_mag ? 2 : 0), t, rows, ctx->lr_smem,
                               st);
      });
    }
  }
  const int nchu = tc ? ctx->nc128 : ctx->nch16;  // unit chunks per pair of the launched kernel
  const int GPR = c.M * c.M * nchu;
  const int g_lo = ctx->row_lo * c.M * nchu, g_hi = ctx->row_hi * c.M * nchu;
  cudaStream_t fs = st;
  if (fork) {  // k_lr_finish runs beside the adjoint kernels; run_loss_grad joins before the combine
    CK(cudaEventRecord(ctx->ev_fork, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    fs = ctx->side;
  }
  MetricsArgs mloc = ma;  // multi-GPU: the metrics follow the collective
  if (ctx->multi) { mloc.out = nullptr; mloc.p_out = nullptr; mloc.loss_hist = nullptr; }
  k_lr_finish<<<c.R, 1024, 0, fs>>>(GPR, g_lo, g_hi, c.loss_mode, c.beta_or_p, ctx->part, ctx->lred, ctx->red, mloc,
                                    ctx->status);
  if (fork) CK(cudaEventRecord(ctx->ev_join, ctx->side));
  ctx->launches += 3;
  return launch_check(ctx, "chebyshev forward");
}

// Forward AF + metrics of (s, w).  Assumes H = FFT(w) is current.
static sqngd_status run_forward(sqngd_ctx ctx, const float2* s, const float2* w, float* af_mag, MetricsOut* met,
                                double* p_out, double* hist, int hist_col, cudaStream_t st, bool xhat_ready = false,
                                const double* snrl_in = nullptr) {
  const sqngd_config& c = ctx->cfg;
  sqngd_status rc;
  if (!xhat_ready && (rc = run_xhat(ctx, s, st, w))) return rc;
  KP kp = make_kp(ctx, c.loss_mode != 0);
  const double ptar = std::pow(10.0, -c.mu_db / 20.0);
  MetricsArgs ma{c.M, c.N, c.K, ctx->L, c.loss_mode, c.beta_or_p, c.eps_w, ptar, ctx->n_cells, ctx->flags,
                 ctx->red, ctx->cm, met, p_out, hist, c.n_h + c.n_x, hist_col, snrl_in};
  ma.tie_scan = met != nullptr && met != ctx->met;  // a record the caller reads: SQNGD_FLAG_TIE
  kp.track_tie = ma.tie_scan;
  MetricsArgs none = ma;
  none.out = nullptr; none.p_out = nullptr; none.loss_hist = nullptr;
  if (ctx->lr) {
    if ((rc = run_lr(ctx, false, MODE_FWD, af_mag, ma, st, false))) return rc;
  } else {
    cudaMemsetAsync(ctx->counter, 0, (2 + 2 * (size_t)c.R) * sizeof(int), st);
    {
      ProfScope ps(ctx, MODE_FWD, st);
      with_P(ctx->P, [&](auto Lc) {
        decltype(Lc)::af(MODE_FWD, kp, ctx->slots[MODE_FWD], ctx->Xc, ctx->H, ctx->tw, ctx->ftw, af_mag, ctx->part, st);
      });
    }
    ctx->launches += 2;
    if ((rc = launch_check(ctx, "af forward"))) return rc;
    k_reduce_groups<<<c.R, 1024, 0, st>>>(c.M * c.K, kp.u_lo, kp.u_hi, c.loss_mode, c.beta_or_p, ctx->part,
                                          ctx->red, ctx->multi ? none : ma, ctx->status,
                                          kp.tiew);
    if ((rc = launch_check(ctx, "metrics"))) return rc;
  }
  if (!ctx->multi) return SQNGD_OK;
  // multi-GPU: c_m of every row, the grouped collective, then the metrics
  if ((rc = run_cm_rows(ctx, s, w, st))) return rc;
  if ((rc = world_combine(ctx, false, st))) return rc;
  k_metrics<<<c.R, 32, 0, st>>>(ma, ctx->status);
  ctx->launches += 1;
  return launch_check(ctx, "metrics");
}

// k_combine_rows with 16 k-lanes (512 threads) for the long slot lists (>= 64 slots per row: the FFT
// engine's K bins, the Chebyshev Step-A M Q spectral slots), 8 otherwise; SQNGD_COMB_KL=8 forces 8.
static void launch_combine(sqngd_ctx ctx, const CombineArgs& ca, dim3 grid, cudaStream_t st) {
  static const int force8 = [] { const char* e = getenv("SQNGD_COMB_KL"); return e && e[0] == '8'; }();
  if (ca.K >= 64 && !force8) k_combine_rows<16><<<grid, 512, 0, st>>>(ca, ctx->status);
  else k_combine_rows<8><<<grid, 256, 0, st>>>(ca, ctx->status);
}

// Loss + gradient of an explicit waveform s.  Assumes H = FFT(w) is current.
// wrt 1: writes grad_w (2 dL/dw^*); wrt 2: grad_s (dL/ds^*), dy and grad_z if dq/grad_z given.
// Step-A optimizer tail fused into the gradient's last kernel (sqngd_step, single GPU).
struct StepATail {
  AdamP ap;
  float2* w;
  float* mw;
  float* vw;
};

static sqngd_status run_loss_grad(sqngd_ctx ctx, const float2* s, const float2* w, int wrt, MetricsOut* met,
                                  float2* grad_w, float2* grad_s, const float* dq, float* grad_z, double* hist,
                                  int hist_col, cudaStream_t st, bool xhat_ready = false,
                                  const StepATail* tail = nullptr, const double* snrl_in = nullptr) {
  const sqngd_config& c = ctx->cfg;
  sqngd_status rc;
  const double ptar = std::pow(10.0, -c.mu_db / 20.0);
  if (!xhat_ready && (rc = run_xhat(ctx, s, st, w, wrt == SQNGD_WRT_FILTERS))) return rc;
  FinArgs fa{c.R, c.M, c.N, wrt, c.eps_w, ptar, ctx->cm, s, w, dq, grad_w, grad_s, ctx->dy, grad_z};
  MetricsArgs ma{c.M, c.N, c.K, ctx->L, c.loss_mode, c.beta_or_p, c.eps_w, ptar, ctx->n_cells, ctx->flags,
                 ctx->red, ctx->cm, met, nullptr, hist, c.n_h + c.n_x, hist_col, snrl_in};
  ma.tie_scan = met != nullptr && met != ctx->met;  // a record the caller reads: SQNGD_FLAG_TIE
  MetricsArgs none = ma;
  none.out = nullptr; none.loss_hist = nullptr;
  const size_t n = (size_t)c.R * c.M * c.N;
  const bool multi = ctx->multi;
  if (c.loss_mode == SQNGD_LOSS_MAX) {  // Eq. 37: the exact maximum, its O(N) subgradient on every rank
    if ((rc = run_forward(ctx, s, w, nullptr, met, nullptr, hist, hist_col, st, true, snrl_in))) return rc;
    k_sparse_adj<<<c.R, 256, 0, st>>>(c.M, c.N, c.K, ctx->L, wrt, c.eps_w, c.weights, s, w, ctx->tw, ctx->red,
                                      ctx->red_grad);
    k_finalize_grad<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(fa, ctx->red_grad, ctx->status, none);
    ctx->launches += 2;
    return launch_check(ctx, "sparse adjoint");
  }
  CombineArgs ca{};
  ca.M = c.M; ca.N = c.N; ca.mode = c.loss_mode; ca.bp = c.beta_or_p; ca.eps = c.eps_w; ca.red = ctx->red;
  ca.f = fa;
  ca.part = ctx->part;
  if (ctx->lr) {  // Chebyshev engine: this rank's rows
    if ((rc = run_lr(ctx, true, wrt == SQNGD_WRT_FILTERS ? MODE_ADJ_A : MODE_ADJ_B, nullptr, ma, st, true))) return rc;
    AdjGArgs ag{};
    ag.M = c.M; ag.N = c.N; ag.Q = ctx->Q; ag.LS = ctx->LS;
    ag.nch = ctx->nch16; ag.csh = 4;
    ag.units = c.R * c.M * c.M * ctx->Q; ag.mode = c.loss_mode; ag.bp = (float)c.beta_or_p;
    ag.row_lo = ctx->row_lo; ag.row_hi = ctx->row_hi; ag.lsplit = ctx->lsplit;
    ag.u0 = ctx->row_lo * ctx->Q * ctx->lsplit;
    ag.Gn = ctx->Gn; ag.um = ctx->part.m; ag.lred = ctx->lred; ag.Xc = ctx->Xc; ag.H = ctx->H; ag.out = ctx->part.g;
    ag.Vt = ctx->Vt; ag.tslot = ctx->tslot; ag.NS = (c.N + 1) & ~1;
    with_P(ctx->P, [&](auto Lc) {
      if (wrt == SQNGD_WRT_TRANSMIT)
        decltype(Lc)::adj_gc(ag, (ctx->row_hi - ctx->row_lo) * ctx->Q * ctx->lsplit, ctx->ftwn, st);
      else decltype(Lc)::adj_g(ag, ctx->ftwn, st);
    });
    ca.part.scale = nullptr;  // node cotangents were rescaled in the adjoint kernels
    CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));  // S and the metrics from k_lr_finish
    if (wrt == SQNGD_WRT_TRANSMIT) {  // node time-domain partials of this rank's rows
      const int QS_ = ctx->Q * ctx->lsplit;  // (node, half) slots per row
      ca.K = QS_; ca.slot_stride = (c.N + 1) & ~1; ca.u_lo = ctx->row_lo * QS_; ca.u_hi = ctx->row_hi * QS_;
      ca.part.g = ctx->tslot; ca.len = c.N; ca.extra = 1.0;
      ca.fin = multi ? 0 : 1;
      ca.out = multi ? ctx->red_grad : nullptr;
      launch_combine(ctx, ca, dim3((c.N + 63) / 64, c.R * c.M), st);
      ctx->launches += 3;
      if ((rc = launch_check(ctx, "chebyshev adjoint (transmit)"))) return rc;
    } else {
      const int nsl = c.M * ctx->Q;  // spectral slots per filter row (zeros for other ranks' rows)
      ca.K = nsl; ca.slot_stride = ctx->P; ca.u_lo = 0; ca.u_hi = c.R * c.M * nsl;
      ca.len = ctx->P; ca.extra = 1.0 / ctx->P; ca.fin = 0; ca.out = ctx->spec;
      launch_combine(ctx, ca, dim3((ctx->P + 63) / 64, c.R * c.M), st);
      ctx->launches += 3;
      if (!multi) {
        if (tail) {
          with_P(ctx->P, [&](auto Lc) {
            decltype(Lc)::rows_adam_w(c.R * c.M, ctx->spec, ctx->ftwr, fa, tail->ap, tail->w, tail->mw, tail->vw,
                                      ctx->H, ctx->cm, ctx->status, st);
          });
        } else {
          with_P(ctx->P, [&](auto Lc) { decltype(Lc)::rows_ifft_fin(c.R * c.M, ctx->spec, ctx->ftwr, fa, ctx->status, st); });
        }
        return launch_check(ctx, "chebyshev adjoint (filters)");
      }
      with_P(ctx->P, [&](auto Lc) { decltype(Lc)::rows_ifft(c.R * c.M, c.N, ctx->spec, ctx->ftw, ctx->red_grad, st); });
      ctx->launches += 1;
    }
    if (!multi) return SQNGD_OK;
  } else {  // per-bin FFT engine: this rank's units
    const int mode = wrt == SQNGD_WRT_FILTERS ? MODE_ADJ_A : MODE_ADJ_B;
    KP kp = make_kp(ctx, 1);
    kp.track_tie = ma.tie_scan;
    cudaMemsetAsync(ctx->counter, 0, (2 + 2 * (size_t)c.R) * sizeof(int), st);
    {
      ProfScope ps(ctx, mode, st);
      with_P(ctx->P, [&](auto Lc) {
        decltype(Lc)::af(mode, kp, ctx->slots[mode], ctx->Xc, ctx->H, ctx->tw, ctx->ftw, nullptr, ctx->part, st);
      });
    }
    ctx->launches += 1;
    if ((rc = launch_check(ctx, "af adjoint"))) return rc;
    ca.K = c.K; ca.slot_stride = ctx->P; ca.u_lo = kp.u_lo; ca.u_hi = kp.u_hi;
    k_reduce_groups<<<c.R, 1024, 0, st>>>(c.M * c.K, kp.u_lo, kp.u_hi, c.loss_mode, c.beta_or_p, ctx->part, ctx->red,
                                          multi ? none : ma, ctx->status, kp.tiew);
    ctx->launches += 1;
    if (mode == MODE_ADJ_B) {  // single GPU: finalize inside the combine
      ca.len = c.N; ca.extra = 1.0; ca.fin = multi ? 0 : 1; ca.out = multi ? ctx->red_grad : nullptr;
      launch_combine(ctx, ca, dim3((c.N + 63) / 64, c.R * c.M), st);
      ctx->launches += 1;
    } else {
      ca.len = ctx->P; ca.extra = 1.0 / ctx->P; ca.fin = 0; ca.out = ctx->spec;
      launch_combine(ctx, ca, dim3((ctx->P + 63) / 64, c.R * c.M), st);
      ctx->launches += 2;
      if (!multi) {  // single GPU: finalize inside the row IFFT (+ Adam(w), Pi_H, next H and c_m in the step)
        if (tail) {
          with_P(ctx->P, [&](auto Lc) {
            decltype(Lc)::rows_adam_w(c.R * c.M, ctx->spec, ctx->ftwr, fa, tail->ap, tail->w, tail->mw, tail->vw,
                                      ctx->H, ctx->cm, ctx->status, st);
          });
        } else {
          with_P(ctx->P, [&](auto Lc) { decltype(Lc)::rows_ifft_fin(c.R * c.M, ctx->spec, ctx->ftwr, fa, ctx->status, st); });
        }
      } else {
        with_P(ctx->P, [&](auto Lc) { decltype(Lc)::rows_ifft(c.R * c.M, c.N, ctx->spec, ctx->ftw, ctx->red_grad, st); });
      }
    }
    if ((rc = launch_check(ctx, "combine"))) return rc;
    if (!multi) return SQNGD_OK;
  }
  // multi-GPU: every row's c_m, the grouped collective, then the finalize (+ metrics) on every rank
  if ((rc = run_cm_rows(ctx, s, w, st))) return rc;
  if ((rc = world_combine(ctx, true, st))) return rc;
  // (at least R blocks: block r < R also writes restart r's metrics)
  k_finalize_grad<<<(unsigned)std::max<size_t>((n + 255) / 256, (size_t)c.R), 256, 0, st>>>(fa, ctx->red_grad,
                                                                                             ctx->status, ma);
  ctx->launches += 1;
  return launch_check(ctx, "finalize grad");
}

// a6 reporting (Eq. 10): SNRL_m and the restart's worst SNRL into the metrics, after the forward.
static sqngd_status run_snrl(sqngd_ctx ctx, const float2* s, const float2* w, double* out, MetricsOut* met,
                             cudaStream_t st, double* worst_out = nullptr) {
  const sqngd_config& c = ctx->cfg;
  k_snrl<<<c.R, 32 * std::min(c.M, 32), 0, st>>>(c.M, c.N, s, w, out, met, ctx->status, worst_out);
  ctx->launches += 1;
  return launch_check(ctx, "snrl");
}

static sqngd_status run_grad_rho(sqngd_ctx ctx, const float* z, const float* rho, float* grad_rho, cudaStream_t st) {
  const sqngd_config& c = ctx->cfg;
  const int MN = c.M * c.N;
  k_grad_rho<kRhoTB><<<dim3((ctx->BR + kRhoTB - 1) / kRhoTB, c.R), 256, 0, st>>>(
      MN, ctx->BR, (float)c.c, (float)(-(1.0 / (2.0 * c.B)) * c.c), z, rho, ctx->dy, grad_rho);
  ctx->launches += 1;
  return launch_check(ctx, "grad rho");
}

// ----------------------------------------------------------------------------- C-ABI compute entry points
extern "C" {

sqngd_status sqngd_quantize(sqngd_ctx ctx, const float* z, const float* rho, float* s_soft, float* s_hard,
                            uint8_t* b_hard, float* dq, sqngd_stream stream) {
  if (!ctx || !z || !rho) return fail(ctx, SQNGD_E_INVALID, "sqngd_quantize: null argument");
  CK(cudaSetDevice(ctx->dev));
  return run_quantize(ctx, z, rho, reinterpret_cast<float2*>(s_soft), reinterpret_cast<float2*>(s_hard), b_hard,
                      dq, S(stream));
}

sqngd_status sqngd_af_forward(sqngd_ctx ctx, const float* s, const float* w, float* af_mag,
                              sqngd_metrics* metrics, double* p_out, double* snrl_db_out, sqngd_stream stream) {
  if (!ctx || !s || !w) return fail(ctx, SQNGD_E_INVALID, "sqngd_af_forward: null argument");
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = S(stream);
  sqngd_status rc = run_filter_fft(ctx, reinterpret_cast<const float2*>(w), st);
  if (rc) return rc;
  MetricsOut* met = metrics ? reinterpret_cast<MetricsOut*>(metrics) : ctx->met;
  if ((rc = run_forward(ctx, reinterpret_cast<const float2*>(s), reinterpret_cast<const float2*>(w), af_mag, met,
                        p_out, nullptr, 0, st)))
    return rc;
  return run_snrl(ctx, reinterpret_cast<const float2*>(s), reinterpret_cast<const float2*>(w), snrl_db_out, met, st);
}

sqngd_status sqngd_loss_grad_s(sqngd_ctx ctx, const float* s, const float* w, int wrt, sqngd_metrics* metrics,
                               float* grad_w, float* grad_s, sqngd_stream stream) {
  if (!ctx || !s || !w || (wrt != SQNGD_WRT_FILTERS && wrt != SQNGD_WRT_TRANSMIT))
    return fail(ctx, SQNGD_E_INVALID, "sqngd_loss_grad_s: bad argument");
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = S(stream);
  sqngd_status rc = run_filter_fft(ctx, reinterpret_cast<const float2*>(w), st);
  if (rc) return rc;
  MetricsOut* met = metrics ? reinterpret_cast<MetricsOut*>(metrics) : ctx->met;
  return run_loss_grad(ctx, reinterpret_cast<const float2*>(s), reinterpret_cast<const float2*>(w), wrt, met,
                       reinterpret_cast<float2*>(grad_w), reinterpret_cast<float2*>(grad_s), nullptr, nullptr,
                       nullptr, 0, st);
}

sqngd_status sqngd_af_loss_grad(sqngd_ctx ctx, const float* z, const float* rho, const float* w, int wrt,
                                sqngd_metrics* metrics, float* grad_w, float* grad_z, float* grad_rho,
                                sqngd_stream stream) {
  if (!ctx || !z || !rho || !w || (wrt != SQNGD_WRT_FILTERS && wrt != SQNGD_WRT_TRANSMIT))
    return fail(ctx, SQNGD_E_INVALID, "sqngd_af_loss_grad: bad argument");
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = S(stream);
  const float2* w2 = reinterpret_cast<const float2*>(w);
  MetricsOut* met = metrics ? reinterpret_cast<MetricsOut*>(metrics) : ctx->met;
  sqngd_status rc;
  if (wrt == SQNGD_WRT_FILTERS) {
    if ((rc = run_quantize(ctx, z, rho, nullptr, ctx->s_hard, nullptr, nullptr, st))) return rc;
    if ((rc = run_filter_fft(ctx, w2, st))) return rc;
    return run_loss_grad(ctx, ctx->s_hard, w2, wrt, met, reinterpret_cast<float2*>(grad_w), nullptr, nullptr,
                         nullptr, nullptr, 0, st);
  }
  if ((rc = run_quantize(ctx, z, rho, ctx->s_soft, nullptr, nullptr, ctx->dq, st))) return rc;
  if ((rc = run_filter_fft(ctx, w2, st))) return rc;
  if ((rc = run_loss_grad(ctx, ctx->s_soft, w2, wrt, met, nullptr, nullptr, ctx->dq, grad_z, nullptr, 0, st)))
    return rc;
  if (grad_rho) return run_grad_rho(ctx, z, rho, grad_rho, st);
  return SQNGD_OK;
}

sqngd_status sqngd_net_forward(sqngd_ctx ctx, const float* theta, const float* y0, float* z, sqngd_stream stream) {
  if (!ctx || !theta || !y0 || !z) return fail(ctx, SQNGD_E_INVALID, "sqngd_net_forward: null argument");
  if (!ctx->net) return fail(ctx, SQNGD_E_INVALID, "sqngd_net_forward: context has no generator (net_width == 0)");
  CK(cudaSetDevice(ctx->dev));
  CK(net_forward(ctx->nd, ctx->nws, theta, y0, z, true, S(stream), &ctx->launches));
  return SQNGD_OK;
}

sqngd_status sqngd_net_backward(sqngd_ctx ctx, const float* theta, const float* y0, const float* z,
                                const float* grad_z, float* grad_theta, sqngd_stream stream) {
  if (!ctx || !theta || !y0 || !z || !grad_z || !grad_theta)
    return fail(ctx, SQNGD_E_INVALID, "sqngd_net_backward: null argument");
  if (!ctx->net) return fail(ctx, SQNGD_E_INVALID, "sqngd_net_backward: context has no generator (net_width == 0)");
  CK(cudaSetDevice(ctx->dev));
  CK(net_backward(ctx->nd, ctx->nws, const_cast<float*>(theta), y0, z, grad_z, grad_theta, nullptr, nullptr, AdamP{},
                  ctx->status, S(stream), &ctx->launches));
  return SQNGD_OK;
}

}  // extern "C"

// The body of one sqngd_step: every launch goes to `st` (capturable).  Adam reads the
// step counters from ctx->d_t (set before the body), so the same graph serves every call.
static sqngd_status step_body(sqngd_ctx ctx, const sqngd_state* stt, int block, double* loss_hist,
                              sqngd_metrics* hard_out, cudaStream_t st) {
  const sqngd_config& c = ctx->cfg;
  float2* w2 = reinterpret_cast<float2*>(stt->w);
  sqngd_status rc;
  auto ap = [&](double lr, int which, int off) {
    return AdamP{(float)lr, (float)c.adam_b1, (float)c.adam_b2, (float)c.adam_eps, ctx->d_t, which, off, ctx->d_ct,
                 ctx->cts};
  };
  if (ctx->net) {  // waveform generation z = f_theta(y0) (Alg. 1)
    CK(net_forward(ctx->nd, ctx->nws, stt->theta, stt->y0, stt->z, true, st, &ctx->launches));
  }
  // hard_out: the metrics of the hard-quantized iterate the step starts from.  With Step A they come from
  // its first evaluation, which evaluates exactly that pair (X_hard, H) -- no extra AF pass; SNRL (Eq. 10)
  // from k_snrl on the same pair.  Without Step A: an explicit forward first.
  bool h_ready = false;  // H = FFT(w)/P of the current w is in ctx->H
  if (hard_out && !(block & SQNGD_BLOCK_A)) {
    if ((rc = run_quantize(ctx, stt->z, stt->rho, nullptr, ctx->s_hard, nullptr, nullptr, st))) return rc;
    if ((rc = run_filter_fft(ctx, w2, st))) return rc;
    if ((rc = run_forward(ctx, ctx->s_hard, w2, nullptr, reinterpret_cast<MetricsOut*>(hard_out), nullptr, nullptr, 0,
                          st)))
      return rc;
    if ((rc = run_snrl(ctx, ctx->s_hard, w2, nullptr, reinterpret_cast<MetricsOut*>(hard_out), st))) return rc;
    h_ready = true;
  }
  if (block & SQNGD_BLOCK_A) {  // Step A: filters with X_hard fixed
    if ((rc = run_quantize(ctx, stt->z, stt->rho, nullptr, ctx->s_hard, nullptr, nullptr, st))) return rc;
    if ((rc = run_xhat(ctx, ctx->s_hard, st, nullptr, true))) return rc;  // X_hard fixed for the block
    if (hard_out) {  // SNRL of the entry pair; on the Chebyshev engine beside the first evaluation (its
                     // k_lr_finish, which reads it, runs later on the same side stream and is joined)
      const bool side = ctx->lr && !ctx->multi && c.loss_mode != SQNGD_LOSS_MAX;
      cudaStream_t ss = st;
      if (side) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        ss = ctx->side;
      }
      if ((rc = run_snrl(ctx, ctx->s_hard, w2, nullptr, nullptr, ss, ctx->snrl_w))) return rc;
    }
    const bool fused = !ctx->multi && c.loss_mode != SQNGD_LOSS_MAX;
    h_ready = fused && c.n_h > 0;  // the fused row kernel leaves H = FFT(w)/P of the updated w
    for (int i = 0; i < c.n_h; ++i) {
      MetricsOut* met = (i == 0 && hard_out) ? reinterpret_cast<MetricsOut*>(hard_out) : ctx->met;
      const double* snrl_in = (i == 0 && hard_out) ? ctx->snrl_w : nullptr;
      if ((!fused || i == 0) && (rc = run_filter_fft(ctx, w2, st, ctx->s_hard))) return rc;
      if (fused) {  // the row kernel also updates w and prepares H, c_m for the next inner step
        const StepATail tail{ap(c.lr_w, 0, i), w2, stt->m_w, stt->v_w};
        if ((rc = run_loss_grad(ctx, ctx->s_hard, w2, SQNGD_WRT_FILTERS, met, nullptr, nullptr, nullptr, nullptr,
                                loss_hist, i, st, true, &tail, snrl_in)))
          return rc;
      } else {
        if ((rc = run_loss_grad(ctx, ctx->s_hard, w2, SQNGD_WRT_FILTERS, met, ctx->gw, nullptr, nullptr,
                                nullptr, loss_hist, i, st, true, nullptr, snrl_in)))
          return rc;
        k_adam_project_w<<<c.R * c.M, 1024, 0, st>>>(c.N, stt->w, stt->m_w, stt->v_w,
                                                     reinterpret_cast<const float*>(ctx->gw), ap(c.lr_w, 0, i),
                                                     ctx->status);
        ctx->launches += 1;
      }
      if ((rc = launch_check(ctx, "step A update"))) return rc;
    }
  }
  if (block & SQNGD_BLOCK_B) {  // Step B: transmit parameters with H fixed
    if (!h_ready && (rc = run_filter_fft(ctx, w2, st))) return rc;
    const int col0 = (block & SQNGD_BLOCK_A) ? c.n_h : 0;
    int n2 = 1;
    while (n2 < ctx->BR) n2 <<= 1;
    for (int i = 0; i < c.n_x; ++i) {
      if ((rc = run_quantize(ctx, stt->z, stt->rho, ctx->s_soft, nullptr, nullptr, ctx->dq, st))) return rc;
      if ((rc = run_loss_grad(ctx, ctx->s_soft, w2, SQNGD_WRT_TRANSMIT, ctx->met, nullptr, nullptr, ctx->dq, ctx->gz,
                              loss_hist, col0 + i, st)))
        return rc;
      // Generator mode: dL/dtheta + Adam(theta) only need dL/dz (and the tape), not the thresholds, so
      // the generator backward runs on a forked branch beside the grad-rho pass (profiling: inline).
      const bool fork_net = ctx->net && !ctx->prof;
      if (fork_net) {
        CK(cudaEventRecord(ctx->ev_nf, st));
        CK(cudaStreamWaitEvent(ctx->side_net, ctx->ev_nf, 0));
        CK(net_backward(ctx->nd, ctx->nws, stt->theta, stt->y0, stt->z, ctx->gz, nullptr, stt->m_theta, stt->v_theta,
                        ap(c.lr_theta, 1, i), ctx->status, ctx->side_net, &ctx->launches));
        CK(cudaEventRecord(ctx->ev_nj, ctx->side_net));
      }
      {  // one-pass dL/drho (k_grad_rho), then Adam(z) (blocks 1..) and Adam(rho) + projection (block 0)
        ZAdam za{};
        if (!ctx->net) {
          za.z = stt->z; za.mz = stt->m_z; za.vz = stt->v_z; za.gz = ctx->gz; za.MN = c.M * c.N; za.ap = ap(c.lr_z, 1, i);
        }
        k_grad_rho<kRhoTB><<<dim3((ctx->BR + kRhoTB - 1) / kRhoTB, c.R), 256, 0, st>>>(
            c.M * c.N, ctx->BR, (float)c.c, (float)(-(1.0 / (2.0 * c.B)) * c.c), stt->z, stt->rho, ctx->dy, ctx->grho);
        const int zch = za.z ? (c.M * c.N + 4095) / 4096 : 0;
        k_adam_project_rho<<<dim3(1 + zch, c.R), 1024, 2 * n2 * sizeof(float), st>>>(ctx->BR, stt->rho, stt->m_rho, stt->v_rho,
                                                                      ctx->grho, ap(c.lr_z, 1, i), 1e-4f,
                                                                      1.0f - 1e-4f, 1e-6f, ctx->status, za);
        ctx->launches += 2;
      }
      if (ctx->net) {  // Adam on theta through the generator's adjoint, then z = f_theta(y0) again
        ProfScope ps(ctx, 3, st);
        if (fork_net) {
          CK(cudaStreamWaitEvent(st, ctx->ev_nj, 0));
        } else {
          CK(net_backward(ctx->nd, ctx->nws, stt->theta, stt->y0, stt->z, ctx->gz, nullptr, stt->m_theta, stt->v_theta,
                          ap(c.lr_theta, 1, i), ctx->status, st, &ctx->launches));
        }
        CK(net_forward(ctx->nd, ctx->nws, stt->theta, stt->y0, stt->z, false, st, &ctx->launches));
      }
      if ((rc = launch_check(ctx, "step B update"))) return rc;
    }
  }
  return SQNGD_OK;
}

// The hard-waveform metrics of a state (quantize, H, forward, SNRL): sqngd_run's last iterate.
sqngd_status sq_ctx_hard_metrics(sqngd_ctx ctx, const sqngd_state* stt, sqngd_metrics* out, sqngd_stream stream) {
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = S(stream);
  float2* w2 = reinterpret_cast<float2*>(stt->w);
  MetricsOut* met = reinterpret_cast<MetricsOut*>(out);
  sqngd_status rc;
  if ((rc = run_quantize(ctx, stt->z, stt->rho, nullptr, ctx->s_hard, nullptr, nullptr, st))) return rc;
  if ((rc = run_filter_fft(ctx, w2, st))) return rc;
  if ((rc = run_forward(ctx, ctx->s_hard, w2, nullptr, met, nullptr, nullptr, 0, st))) return rc;
  return run_snrl(ctx, ctx->s_hard, w2, nullptr, met, st);
}

extern "C" {

sqngd_status sqngd_step(sqngd_ctx ctx, sqngd_state* stt, int block, double* loss_hist, sqngd_metrics* hard_out,
                        sqngd_stream stream) {
  if (!ctx || !stt || !stt->z || !stt->rho || !stt->w || (block & ~3) || !block)
    return fail(ctx, SQNGD_E_INVALID, "sqngd_step: bad argument");
  if (ctx->net && (!stt->theta || !stt->m_theta || !stt->v_theta || !stt->y0))
    return fail(ctx, SQNGD_E_INVALID, "sqngd_step: generator mode needs theta, m_theta, v_theta and y0");
  CK(cudaSetDevice(ctx->dev));
  const sqngd_config& c = ctx->cfg;
  const cudaStream_t st = S(stream);
  sqngd_status rc;
  // Adam step counters (k_set_t): launched ahead of the body, inside the graph when there is one (its
  // (t_a, t_b) arguments are rewritten on the instantiated graph before every replay, so a step is one
  // graph launch with no eager kernel in front of it).
  long long ta = stt->t_a, tb = stt->t_b;
  int cts = ctx->cts, nh = c.n_h, nx = c.n_x;
  double b1 = c.adam_b1, b2 = c.adam_b2;
  void* set_args[] = {&ctx->d_t, &ta, &tb, &ctx->d_ct, &cts, &nh, &nx, &b1, &b2};
  auto launch_set_t = [&]() {
    k_set_t<<<1, 64, 0, st>>>(ctx->d_t, ta, tb, ctx->d_ct, cts, nh, nx, b1, b2);
    ctx->launches += 1;
  };
  // Graph path: one GPU or NCCL (the collective is captured with the step), a capturable (non-legacy) stream.
  const bool graph_ok = ctx->use_graphs && !ctx->prof && (!ctx->multi || ctx->comm->capturable()) && st != nullptr &&
                        st != cudaStreamLegacy && st != cudaStreamPerThread;
  if (!graph_ok) {
    launch_set_t();
    if ((rc = step_body(ctx, stt, block, loss_hist, hard_out, st))) return rc;
  } else {
    const void* key[16] = {stt->z, stt->rho, stt->w, stt->m_z, stt->v_z, stt->m_rho, stt->v_rho, stt->m_w, stt->v_w,
                           loss_hist, hard_out, st, stt->theta, stt->m_theta, stt->v_theta, stt->y0};
    sqngd_ctx_s::GraphEntry* ge = nullptr;
    for (auto* g : ctx->graphs)
      if (g->block == block && g->prof == ctx->prof && std::memcmp(g->key, key, sizeof(key)) == 0) ge = g;
    if (!ge) {
      ge = new sqngd_ctx_s::GraphEntry();
      std::memcpy(ge->key, key, sizeof(key));
      ge->block = block;
      ge->prof = ctx->prof;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      ctx->capturing = ge;
      const int64_t l0 = ctx->launches;
      launch_set_t();
      rc = step_body(ctx, stt, block, loss_hist, hard_out, st);
      ctx->capturing = nullptr;
      ge->launches = ctx->launches - l0;
      ctx->launches = l0;
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(st, &graph);
      if (rc != SQNGD_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        delete ge;
        if (rc) return rc;
        return fail(ctx, SQNGD_E_CUDA, "sqngd_step: graph capture", cudaGetErrorString(e));
      }
      // the k_set_t node: the graph's root kernel node running k_set_t
      size_t nroot = 0;
      CK(cudaGraphGetRootNodes(graph, nullptr, &nroot));
      std::vector<cudaGraphNode_t> roots(nroot);
      if (nroot) CK(cudaGraphGetRootNodes(graph, roots.data(), &nroot));
      for (cudaGraphNode_t n : roots) {
        cudaGraphNodeType ty;
        CK(cudaGraphNodeGetType(n, &ty));
        if (ty != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp{};
        CK(cudaGraphKernelNodeGetParams(n, &kp));
        if (kp.func == reinterpret_cast<void*>(&k_set_t)) { ge->set_t = n; ge->set_p = kp; }
      }
      e = ge->set_t ? cudaGraphInstantiate(&ge->exec, graph, 0) : cudaErrorInvalidValue;
      ge->graph = graph;
      if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        delete ge;
        return fail(ctx, SQNGD_E_CUDA, "sqngd_step: graph instantiate", cudaGetErrorString(e));
      }
      ctx->graphs.push_back(ge);
    } else {
      cudaKernelNodeParams kp = ge->set_p;
      kp.kernelParams = set_args;
      kp.extra = nullptr;
      CK(cudaGraphExecKernelNodeSetParams(ge->exec, ge->set_t, &kp));
    }
    CK(cudaGraphLaunch(ge->exec, st));
    ge->replayed = true;
    ctx->launches += ge->launches;
  }
  if (block & SQNGD_BLOCK_A) stt->t_a += c.n_h;
  if (block & SQNGD_BLOCK_B) stt->t_b += c.n_x;
  return SQNGD_OK;
}

}  // extern "C"
