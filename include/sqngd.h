/* sqngd.h -- C-ABI of the B200 (sm_100a) SQNGD AF/CAF loss+gradient hot path.
 *
 * Method: arXiv 2604.25728 ("SQNGD", joint transmit-receive design of unimodular
 * discrete-phase waveforms and mismatched filters).  Citations are to
 * /root/reference/PAPER.md lines (P:Lx) and equation numbers; readings of the
 * paper (Q1..Q25) are listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 *   - Array pointers are CUDA DEVICE pointers unless stated otherwise, owned by
 *     the caller (e.g. torch tensors); the library never frees them.
 *   - Complex arrays are interleaved fp32 pairs (re, im): "float*" of 2x length.
 *   - Layouts are row-major: s, w, z = [R][M][N] (the paper's X[:, m] = s[m][:],
 *     P:L91-94; vec() column stacking = this flattening);
 *     rho = [R][B*r_n]; the optional AF magnitude map = [R][M][M][K][ld] (ld = map_ld, or 2N-1) with
 *     lag tau stored at index tau + N - 1 (Eq. 6 labels, Q1).
 *   - Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy default
 *     stream).  The return status reports launch-time errors; device-side
 *     conditions (non-finite values, degenerate mainlobe, unsorted thresholds)
 *     are latched in the context and returned by the next call or sqngd_sync().
 *   - One context per (device, stream owner); no internal threads.
 *   - Multi-GPU (world > 1): every rank creates its context with the same config
 *     and a shared ncclUniqueId; each rank evaluates a contiguous slice of the
 *     (restart, channel, Doppler) units and one NCCL all-reduce per evaluation
 *     combines the partials, so every rank returns the full reduced outputs.
 */
#ifndef SQNGD_H
#define SQNGD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sqngd_ctx_s* sqngd_ctx;
typedef void* sqngd_stream; /* cudaStream_t */

typedef enum {
  SQNGD_OK = 0,
  SQNGD_E_INVALID = 1,    /* bad dims, B<2, ROI outside [-N+1, N-1], K<1, empty ROI, rho unsorted */
  SQNGD_E_DEGENERATE = 2, /* |w_m^H s_m| == 0 or a zero-energy filter row (Eq. 32 undefined) */
  SQNGD_E_NONFINITE = 3,  /* NaN/Inf in a loss or gradient; sqngd_step leaves the state unchanged */
  SQNGD_E_CUDA = 4,
  SQNGD_E_NCCL = 5,
  SQNGD_E_NOMEM = 6
} sqngd_status;

typedef enum {
  SQNGD_LOSS_MAX = 0,   /* Eq. 37 max(WAPSL, WCPSL); subgradient to the unique argmax (Q17)   */
  SQNGD_LOSS_LSE = 1,   /* (1/beta) ln sum_S e^{beta v}, v = w|A|/N (north-star surrogate)    */
  SQNGD_LOSS_PNORM = 2  /* (sum_S v^p)^{1/p}                                                  */
} sqngd_loss_mode;

enum { SQNGD_WRT_FILTERS = 1, /* Step A: waveform fixed, gradient to the filters w */
       SQNGD_WRT_TRANSMIT = 2 /* Step B: filters fixed, gradient to z and rho      */ };
enum { SQNGD_BLOCK_A = 1, SQNGD_BLOCK_B = 2, SQNGD_BLOCK_AB = 3 };
enum { SQNGD_FLAG_NO_CROSS = 1,     /* M == 1: WCPSL := 0 (no cross terms, Eq. 9)              */
       SQNGD_FLAG_TIE = 2,          /* the WAPSL or WCPSL maximum (or WAPSL == WCPSL) is attained by more
                                       than one cell in the engine's fp32 arithmetic; the reported argmax is
                                       the lowest (m, l, tau, k) (Eqs. 7-9).  Exact
                                       between cells of different evaluation units; within a Chebyshev
                                       unit, two bins of one lag on the same side of the grid centre are
                                       not compared.  Single-context only (world == 1).  */
       SQNGD_FLAG_DOPPLER_ALIAS = 4 /* grid reaches beyond [-N/2, N/2]; |A| is N-periodic in f */ };

/* Problem definition (copied into the context at create). */
typedef struct {
  int32_t R;         /* independent restarts batched in one call                           */
  int32_t M;         /* channels: M transmit waveforms and M receive filters */
  int32_t N;         /* code length, 2 <= N <= 4096                                          */
  int32_t B;         /* phase alphabet size (Eq. 5), >= 2                                    */
  int32_t r_n;       /* quantizer copies (Eq. 24); thresholds per restart = B * r_n          */
  double c;          /* quantizer steepness (Eq. 21)                                         */
  int32_t K;         /* Doppler bins: inclusive uniform grid f_k = f_lo + k (f_hi-f_lo)/(K-1) */
  double f_lo, f_hi; /* paper units: f = f_d T, exponent e^{j 2 pi n f / N} (Q8) */
  int32_t tau_lo, tau_hi;          /* ROI delays, inside [-(N-1), N-1]                    */
  int32_t exclude_auto_zero_delay; /* 1: Eq. 8 "tau != 0" drops the whole tau=0 column (Q6) */
  int32_t loss_mode;               /* sqngd_loss_mode                                     */
  double beta_or_p;                /* LSE beta or p-norm p                                */
  double eps_w;                    /* Eq. 42 epsilon                                      */
  double mu_db;                    /* SNRL target (dB), p_tar = 10^{-mu/20} (Eq. 39)      */
  double lr_w, lr_z;               /* Adam rates: filters (eta_h), z and rho (Q14) */
  double adam_b1, adam_b2, adam_eps; /* Q15                                               */
  int32_t n_h, n_x;                /* inner steps per block (Alg. 1)      */
  const float* weights;            /* device [K][2N-1] w(tau,f) >= 0 (Eqs. 8-9), NULL => 1;
                                      must stay valid for the context's lifetime          */
  int32_t doppler_engine;          /* SQNGD_ENGINE_*: how the K Doppler bins are evaluated */
  double lr_tol;                   /* CHEBYSHEV: bound on |A_interp - A| / (||s|| ||w||)
                                      (0 => 1e-7); picks the node count Q at create       */
  int32_t net_depth;               /* generator residual blocks D (paper: 5)       */
  int32_t net_width;               /* generator hidden width W (paper: 128); 0 = no generator,
                                      z is the direct parameter (Q13); else W % 8 == 0, <= 128 */
  double lr_theta;                 /* Adam rate of theta (eta_x = 1e-5)             */
  int32_t map_ld;                  /* row pitch (floats) of the optional |A| map of
                                      sqngd_af_forward: 0 => 2N-1 (dense); else >= 2N-1, e.g.
                                      2N rounded up to 32 so every bin row starts on a 128-byte
                                      boundary (whole-sector stores; the pad is not written)   */
} sqngd_config;

/* Doppler engine (sqngd_config.doppler_engine).
   FFT:       one modulated FFT correlation per Doppler bin (Eqs. 33-36):
              O(M^2 K) transforms, exact up to fp32 rounding.
   CHEBYSHEV: SURVEY.md §8(f) NEXT-1 -- exact FFT correlations (Eq. 36) at Q Chebyshev
              Doppler nodes of [f_lo, f_hi], then the K-bin AF by the dense (K x Q)
              Lagrange contraction fused with the cell epilogue, and its adjoint;
              O(M^2 Q) transforms.  |A| is reproduced to lr_tol * ||s|| ||w|| (DESIGN.md
              §3 "Chebyshev engine").
   AUTO:      CHEBYSHEV when the node count Q for lr_tol is <= 16 and <= K/3 (narrow grids such
              as the paper's [-0.5, 0.5]); FFT otherwise. */
enum { SQNGD_ENGINE_AUTO = 0, SQNGD_ENGINE_FFT = 1, SQNGD_ENGINE_CHEBYSHEV = 2 };

/* One per restart, written by the library into caller-owned DEVICE memory. */
typedef struct {
  double loss;       /* Eq. 42: eps * loss_wpsl + (1 - eps) * loss_snrl                  */
  double loss_wpsl;  /* Eq. 37 (MAX) or the LSE / p-norm surrogate                      */
  double loss_snrl;  /* Eq. 41                                                          */
  double wapsl;      /* Eq. 8 / N: exact max over auto maps of w|A|/N                   */
  double wcpsl;      /* Eq. 9 / N: exact max over cross maps                            */
  double wpsl;       /* Eq. 7                                                           */
  int32_t argmax_auto[4];  /* (m, l, tau, k) of WAPSL, ties -> lowest lexicographic     */
  int32_t argmax_cross[4]; /* (m, l, tau, k) of WCPSL ((-1,...) when M == 1)            */
  uint32_t flags;          /* SQNGD_FLAG_*                                              */
  uint32_t n_cells;        /* |S|: sidelobe cells in the ROI                            */
  double apslr_db;         /* Eq. 48: 20 log10(WAPSL) (-inf when 0)        */
  double cpslr_db;         /* Eq. 48 of WCPSL (-inf when M == 1)                        */
  double pslr_db;          /* Eq. 48 of WPSL                                            */
  double snrl_db_max;      /* max_m SNRL_m, Eq. 10, from the literal norms;
                              written by sqngd_af_forward and sqngd_step's hard_out,
                              NaN in the loss+gradient calls                            */
} sqngd_metrics;

/* Optimizer state: caller-owned DEVICE buffers, mutated in place by sqngd_step.
   t_a / t_b (host integers) are the Adam step counts of the two blocks. */
typedef struct {
  float* z;     /* [R][M][N] phase parameters z = phi / 2pi (Q13)                       */
  float* rho;   /* [R][B*r_n] ascending thresholds (Eq. 24)                             */
  float* w;     /* [R][M][N] complex filters (H_Re + j H_Im, Eqs. 26-28)                */
  float *m_z, *v_z, *m_rho, *v_rho; /* Adam moments, same shapes as z / rho               */
  float *m_w, *v_w;                 /* Adam moments of (Re w, Im w): [R][M][N][2]         */
  int64_t t_a, t_b;
  /* Generator mode (cfg.net_width > 0): z = f_theta(y0) is written by sqngd_step (m_z, v_z unused)
     and Step B's Adam acts on theta instead of z.  NULL when cfg.net_width == 0. */
  float *theta, *m_theta, *v_theta; /* [R][sqngd_net_num_params] (layout: sqngd_net_forward)  */
  const float* y0;                  /* [R][M N] fixed generator input (Alg. 1)       */
} sqngd_state;

/* Build the context: validates the config (SQNGD_E_INVALID), builds the fp64
   Doppler twiddle table and the workspace on `cuda_device`.  nccl_unique_id:
   NULL for one GPU, else 128 bytes of an ncclUniqueId shared by all ranks (with world == 1 an id
   selects the same collective path over a 1-rank NCCL communicator: the NCCL backend on one GPU).
   Multi-GPU (world > 1): each rank evaluates a shard -- the FFT engine
   a contiguous slice of the R M K (restart, channel, bin) units, the Chebyshev engine a contiguous slice
   of the R M (restart, transmit channel) rows -- and every loss / gradient evaluation ends with ONE
   grouped NCCL call (SUM of the fp64 [weighted S | weighted gradient] payload, MAX of the u64 keys,
   against a reference shift all ranks share), after which every rank holds the full outputs and
   applies the identical optimizer step.  sqngd_step captures the NCCL call into its CUDA graph. */
sqngd_status sqngd_create(const sqngd_config* cfg, int cuda_device, const void* nccl_unique_id,
                          int rank, int world, sqngd_ctx* out);

/* Single-device stand-in for NCCL (tests): a group of `world` (2..8) contexts in ONE process on the same
   device, each driven by its own host thread; the grouped collective is a host barrier plus one
   reduction kernel on the last-arriving rank's stream, ordered by CUDA events (no kernel waits on
   another rank's kernel).  The contexts run the exact sharded path of world > 1; sqngd_step does not
   capture a graph for them.  Destroy the group after its contexts. */
typedef struct sqngd_loopback_s* sqngd_loopback;
sqngd_loopback sqngd_loopback_create(int world); /* NULL if world is outside 2..8 */
void sqngd_loopback_destroy(sqngd_loopback group);
sqngd_status sqngd_create_loopback(const sqngd_config* cfg, int cuda_device, sqngd_loopback group, int rank,
                                   sqngd_ctx* out);
/* The loopback group's reduction kernel.  on = 0 (default): one plain reduction kernel.  on = 1: the
   peer-memory all-reduce kernel below (k_peer_allreduce) over windows of the group's contexts, its
   signal phase launched for every rank and then its wait + reduce phase for every rank on one stream
   (every wait already satisfied), so the kernel that runs between GPUs is validated on one device. */
/* on = 2: the fused form (k_world_peer: pack + all-reduce + unpack in one kernel, the default of the
   peer backend below), again phase by phase.  on = 3 (tests of the watchdog): as 2, but the last rank's
   signal phase is never launched, so every rank's wait gives up after 2 s and latches SQNGD_E_NCCL. */
sqngd_status sqngd_loopback_set_peer(sqngd_loopback group, int on);

/* In-kernel all-reduce over NVLink peer memory instead of NCCL (DESIGN.md §7
   "In-kernel all-reduce"; no passage of the paper, which is single-GPU).  For a context created
   with world >= 1 and an ncclUniqueId:
     sqngd_peer_export  allocates this rank's window (epochs, flags, a double-buffered stage of the
                        grouped payload) and writes its 64-byte CUDA IPC handle to handle64 (host);
     sqngd_peer_attach  handles = world x 64 bytes (host), rank-major, every rank's exported handle
                        (exchanged by the caller, e.g. torch.distributed.all_gather_object); maps the
                        peers' windows, drops the step graphs captured so far and replaces the NCCL
                        backend: from then on every evaluation's grouped collective is ONE kernel of
                        this library (k_world_peer: the weighted payload computed straight into the
                        stage, flag signal over NVLink, wait, rank-ordered sum / max read from the
                        peers' stages, normalised global gradient and record written; identical bits on
                        every rank), captured in the step graph.  Environment SQNGD_PEER_FUSED=0 at
                        attach selects the 3-launch form (pack, k_peer_allreduce, unpack).
   Ranks must be separate processes on P2P-capable devices of one node (CUDA IPC); every rank calls
   both functions before its next evaluation.  A rank that never signals makes the waiting kernels
   give up after 30 s: SQNGD_E_NCCL from sqngd_sync, the context is unusable afterwards.
   SQNGD_E_INVALID: not a multi-GPU context / attach before export; SQNGD_E_CUDA: IPC mapping failed
   (the NCCL backend stays in place). */
sqngd_status sqngd_peer_export(sqngd_ctx ctx, void* handle64);
sqngd_status sqngd_peer_attach(sqngd_ctx ctx, const void* handles);
void sqngd_destroy(sqngd_ctx ctx);
/* Message for the last non-OK status (ctx may be NULL: last create error). */
const char* sqngd_last_error(sqngd_ctx ctx);
/* The Doppler engine the context selected (SQNGD_ENGINE_FFT or _CHEBYSHEV), its node count Q
   (0 for FFT) and the host-computed interpolation error bound (relative to ||s|| ||w||). */
sqngd_status sqngd_engine_info(sqngd_ctx ctx, int32_t* engine, int32_t* q_nodes, double* err_bound);
/* Synchronize `stream` and return (and clear) the latched device-side status. */
sqngd_status sqngd_sync(sqngd_ctx ctx, sqngd_stream stream);

/* a1: soft/hard quantizer + phase map (Eqs. 21-24, 43, 23).
   z [R][M][N], rho [R][B r_n] (ascending) -> s_soft, s_hard (complex [R][M][N]),
   b_hard [R][M][N] phase index in [0,B) (u8), dq = Q_A'(z) [R][M][N].  Any output may be NULL. */
sqngd_status sqngd_quantize(sqngd_ctx ctx, const float* z, const float* rho, float* s_soft,
                            float* s_hard, uint8_t* b_hard, float* dq, sqngd_stream stream);

/* a2-a6: all M^2 AF/CAF maps over (2N-1) lags x K Doppler bins by Doppler-modulated,
   zero-padded FFT correlation (Eqs. 33-36), fused with the ROI reduction (Eqs. 7-9,
   37-42).  s, w: complex [R][M][N].  af_mag: NULL or [R][M][M][K][ld] |A| (fp32), ld = cfg.map_ld
   or 2N-1 (lag tau at column tau + N - 1; columns >= 2N-1 of a pitched row are not written).
   metrics: [R] sqngd_metrics.  p_out: NULL or [R][M] doubles p_m (Eq. 38).
   snrl_db_out: NULL or [R][M] doubles SNRL_m = 10 log10(||s_m||^2 ||w_m||^2 / |s_m^H w_m|^2)
   (Eq. 10; +inf when s_m^H w_m = 0, which also latches SQNGD_E_DEGENERATE). */
sqngd_status sqngd_af_forward(sqngd_ctx ctx, const float* s, const float* w, float* af_mag,
                              sqngd_metrics* metrics, double* p_out, double* snrl_db_out, sqngd_stream stream);

/* a7-a8 for an explicit waveform s: loss and gradient by adjoint correlations.
   wrt = SQNGD_WRT_FILTERS: grad_w = dL/dRe w + j dL/dIm w = 2 dL/dw^* (Q16) [R][M][N] complex.
   wrt = SQNGD_WRT_TRANSMIT: grad_s = dL/ds^* (Wirtinger) [R][M][N] complex.
   Either gradient pointer may be NULL when not requested. */
sqngd_status sqngd_loss_grad_s(sqngd_ctx ctx, const float* s, const float* w, int wrt,
                               sqngd_metrics* metrics, float* grad_w, float* grad_s,
                               sqngd_stream stream);

/* a1-a8: quantize (z, rho) then loss + gradient.  wrt = SQNGD_WRT_FILTERS uses s_hard
   (Alg. 1 Step A) and writes grad_w; wrt = SQNGD_WRT_TRANSMIT uses s_soft (Step B) and
   writes grad_z [R][M][N] and grad_rho [R][B r_n] through Q_A (Eqs. 23-24). */
sqngd_status sqngd_af_loss_grad(sqngd_ctx ctx, const float* z, const float* rho, const float* w,
                                int wrt, sqngd_metrics* metrics, float* grad_w, float* grad_z,
                                float* grad_rho, sqngd_stream stream);

/* a9: one Alg. 1 outer iteration restricted to `block`:
   A: n_h x [loss_grad(s_hard) -> Adam(Re w, Im w) -> Pi_H (Eq. 32)];
   B: n_x x [loss_grad(s_soft) -> Adam(z), Adam(rho) -> threshold projection (Q22)].
   Generator mode: z = f_theta(y0) at the start and after every Step-B update; Step B's Adam
   acts on theta (rate lr_theta) through sqngd_net_backward's adjoint instead of on z.
   loss_hist: NULL or DEVICE [R][n_h + n_x] doubles (loss of each inner step, in order,
   A first).  hard_out: NULL or DEVICE [R] metrics of the hard-quantized iterate the step STARTS from
   (X_hard of (z, rho) and w on entry, snrl_db_max included): with Step A they are its first
   evaluation's (that evaluation is exactly this pair), without Step A an explicit forward runs
   first.  The iterate a step returns is scored by the next step (or sqngd_af_forward).
   On a latched non-finite value the remaining updates are skipped (state unchanged). */
sqngd_status sqngd_step(sqngd_ctx ctx, sqngd_state* state, int block, double* loss_hist,
                        sqngd_metrics* hard_out, sqngd_stream stream);

/* Generator: z = f_theta(y0), the transmit-side ResNet of PAPER.md Eq. 20
    with "5 residual blocks and a hidden width of 128 ... tanh ... sigmoid at the output"
   (P:L583).  With Din = M N, W = cfg.net_width, D = cfg.net_depth (DESIGN.md §3 "Generator"):
     h_0 = tanh(W_in y0 + b_in);  u_d = tanh(W1_d h_d + b1_d);  h_{d+1} = h_d + W2_d u_d + b2_d;
     z = sigmoid(W_out h_D + b_out)
   theta per restart, row-major, in this order:
     W_in [W][Din] | b_in [W] | D x (W1 [W][W] | b1 [W] | W2 [W][W] | b2 [W]) | W_out [Din][W] | b_out [Din] | pad
   where pad (< 4 floats, only when Din % 4 != 0) makes the per-restart stride P a multiple of 4;
   the forward ignores it, Adam leaves it alone and the backward writes 0 there.
   theta, y0 [R][Din], z [R][M][N] (= [R][Din]) are device pointers owned by the caller.
   sqngd_net_forward keeps the activations (tape) in the context; sqngd_net_backward needs the tape
   of the preceding forward with the same theta and y0, z its output, grad_z = dL/dz, and writes
   every entry of grad_theta [R][P].  SQNGD_E_INVALID when the context has no generator. */
int64_t sqngd_net_num_params(const sqngd_config* cfg); /* stride P per restart (parameters + pad);
                                                         0 when net_width == 0 or invalid    */
sqngd_status sqngd_net_forward(sqngd_ctx ctx, const float* theta, const float* y0, float* z, sqngd_stream stream);
sqngd_status sqngd_net_backward(sqngd_ctx ctx, const float* theta, const float* y0, const float* z,
                                const float* grad_z, float* grad_theta, sqngd_stream stream);

/* Alg. 1 driver.  Up to opts->T outer iterations of
   sqngd_step(SQNGD_BLOCK_AB) on `state`, each followed by the hard-waveform metrics (Eq. 43 then
   Eq. 7).  Per restart r the state with the lowest hard WPSL so far is copied into `best`
   (DEVICE buffers z, rho, w, and theta in generator mode; the other members are ignored): the
   output (X_hard, H) of Alg. 1 is quantize(best.z, best.rho) and best.w.  Stopping criterion
   ("further reduction of L does not lead to improvement in the WPSL"; DESIGN.md §3
   "Stopping rule"): an outer iteration improves restart r when its hard WPSL is below the best so far
   by more than opts->tol (1e-6); training stops after the outer iteration at which EVERY
   restart has gone opts->patience consecutive iterations without an improvement and, when
   opts->require_loss_decrease, has a hard loss L below the L of its last improvement (L kept
   decreasing over the window).  patience <= 0: run all T.
   best_wpsl [R] doubles, best_iter [R] int32 (1-based outer iteration of the snapshot), wpsl_hist and
   loss_hist (NULL or [T][R] doubles: hard WPSL / hard loss per iteration until the stop) are DEVICE
   pointers.  Iterate t is scored by the hard_out of step t + 1 (its first Step-A evaluation, from a
   copy of the state taken before that step) and the last iterate by one forward after the loop
   (DESIGN.md §3 "Hard metrics of an outer iteration").  The bookkeeping runs on the device (its
   buffers are kept in the context); the host polls the stop flag every opts->check_every steps, so
   the live `state` may run up to check_every steps past the stopping iterate (the snapshot, best_*
   and result->iterations follow the rule exactly).  Returns after synchronizing `stream` (the latched
   device status, as sqngd_sync). */
typedef struct {
  int32_t T;           /* maximum outer iterations (the paper's T = 2000)          */
  int32_t patience;    /* outer iterations without hard-WPSL improvement before stopping   */
  int32_t check_every; /* >= 1: host polls the device stop flag every check_every steps    */
  int32_t require_loss_decrease; /* 1: also require L below its value at the last improvement */
  double tol;          /* >= 0: minimum decrease of the hard WPSL (linear, / N) that counts */
} sqngd_run_opts;
typedef struct {
  int64_t iterations;  /* outer iterations until the rule stopped training (T if it did not) */
  int64_t steps_run;   /* sqngd_step calls made (iterations <= steps_run <= iterations + check_every
                          when stopped; T otherwise)                                          */
  int32_t stopped;     /* 1: stopped by the rule, 0: T reached                             */
  int32_t reserved;
} sqngd_run_result;
sqngd_status sqngd_run(sqngd_ctx ctx, sqngd_state* state, const sqngd_run_opts* opts, sqngd_state* best,
                       double* best_wpsl, int32_t* best_iter, double* wpsl_hist, double* loss_hist,
                       sqngd_run_result* result, sqngd_stream stream);

/* sqngd_step captures itself into a CUDA graph on the first call with a given (state
   buffers, block, outputs) on a non-legacy stream and replays the graph afterwards
   (single GPU; SQNGD_NO_GRAPH=1 disables).
   Profiling (for the roofline in bench.py): when enabled, sqngd_step runs eagerly and every
   launch of the dominant fused kernel (k_af for the FFT engine, k_lrt for the Chebyshev
   engine), and each generator update of Step B, is bracketed by CUDA events on its launch stream.
   sqngd_profile_read synchronizes and returns, per class (0 forward, 1 Step-A adjoint, 2 Step-B
   adjoint, 3 generator backward + Adam(theta) + forward), the summed device milliseconds ms[4]
   and counts count[4], plus `launches` = every kernel the
   library launched since the last reset (all classes, small kernels included). */
sqngd_status sqngd_profile_enable(sqngd_ctx ctx, int on);
sqngd_status sqngd_profile_read(sqngd_ctx ctx, double* ms, int64_t* count, int64_t* launches, int reset);

/* Debug: with the environment variable SQNGD_GUARD=1 at sqngd_create, every workspace buffer of the
   context is allocated with a 4 KiB guard band on each side (filled with 0x5A).  sqngd_check_guards
   synchronizes the device and sets *corrupted to the number of buffers whose guard bands changed (an
   out-of-bounds write by a kernel), or -1 when the context was created without guards. */
sqngd_status sqngd_check_guards(sqngd_ctx ctx, int64_t* corrupted);

/* Host utilities (no GPU needed). */
int64_t sqngd_num_units(const sqngd_config* cfg); /* R * M * K evaluation units */
/* Contiguous slice [lo, hi) of the units owned by `rank` of `world`. */
void sqngd_shard_range(int64_t units, int rank, int world, int64_t* lo, int64_t* hi);
const char* sqngd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SQNGD_H */
