// The multi-GPU combine of one evaluation as ONE kernel (DESIGN.md §7 "In-kernel
// all-reduce"): k_world_pack, the all-reduce over NVLink peer memory (comm.h k_peer_allreduce) and
// k_world_unpack fused.  Same window, flags and epochs as k_peer_allreduce; the grid is FIXED
// (peer_grid of the window capacity) so every block's epoch advances in lockstep and a block may compare
// another block's flag against its own epoch.  With stride = 1 + 2 M N (or 1 without a gradient) the
// payload index space [R stride] is cut into gridDim.x equal slices; block b
//   phase A  computes slice b of [wS_r | wG_r g_r] straight into its stage (no pack buffer), the block
//            that owns a restart's scalar (index r stride) also stages that restart's three keys;
//            fence; flag[rank][b] = e on every rank (remote stores over NVLink);
//   phase B  waits for (1) block b of every rank, (2) the scalar-owner block of every restart its slice
//            touches, on every rank (S_r normalises the gradient), and, if it owns restart r's scalar,
//            (3) the OWN rank's blocks that touch restart r: they have read the local record red[r] and
//            m_ref[r], which this block now overwrites with the global ones (the grid is <= 128 blocks of
//            256 threads, co-resident on 148 SMs; the clock watchdog bounds every wait regardless);
//            then sums slice b over the ranks' stages in rank order, normalises and writes the global
//            gradient, record and next reference shift -- the bits of pack + rank-ordered sum + unpack.
#pragma once
#include "comm.h"
#include "misc_kernels.cuh"

namespace sq {

__device__ __forceinline__ bool peer_wait(const unsigned long long* f, unsigned long long e, unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (peer_ld_acquire(f) < e) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > timeout_ns) return false;
    __nanosleep(64);
  }
  return true;
}

__global__ void __launch_bounds__(kPeerThreads) k_world_peer(WorldArgs a, PeerArgs pa, int phases, unsigned long long timeout_ns) {
  typedef unsigned long long u64;
  const int b = blockIdx.x, G = gridDim.x, t = threadIdx.x;
  u64* own = reinterpret_cast<u64*>(pa.win[pa.rank]);
  const u64 e = own[b] + 1;
  const size_t stage_off = peer_flags_bytes() + (size_t)(e & 1) * peer_stage_bytes(pa.cap_sum, pa.cap_max);
  const size_t n = a.with_grad ? (size_t)2 * a.M * a.N : 0, stride = 1 + n, T = (size_t)a.R * stride;
  const size_t cs = (T + G - 1) / G;
  const size_t i0 = min(T, (size_t)b * cs), i1 = min(T, i0 + cs);
  if (phases & kPeerPhaseA) {
    double* st_sum = reinterpret_cast<double*>(pa.win[pa.rank] + stage_off);
    u64* st_key = reinterpret_cast<u64*>(st_sum) + pa.cap_sum;
    int rc = -1;
    double wS = 0.0, wG = 0.0, m = 0.0;
    int r = (int)(min(T, i0 + t) / stride);
    size_t j = i0 + t - (size_t)r * stride;
#pragma unroll 2
    for (size_t i = i0 + t; i < i1; i += blockDim.x, j += blockDim.x) {
      while (j >= stride) {  // (restart, offset) of i without a 64-bit division per element
        j -= stride;
        ++r;
      }
      if (r != rc) {
        world_weights(a, r, wS, wG, m);
        rc = r;
      }
      if (j == 0) {
        st_sum[i] = (isfinite(wS) && isfinite(wG)) ? wS : INFINITY;  // fp64 weight overflow, as k_world_pack
        const Red rr = a.red[r];
        st_key[3 * r] = rr.key_a;
        st_key[3 * r + 1] = rr.key_c;
        st_key[3 * r + 2] = (rr.m > 0.0) ? (u64)__double_as_longlong(rr.m) : 0ull;
      } else {
        st_sum[i] = wG * (double)reinterpret_cast<const float*>(a.grad)[(size_t)r * n + (j - 1)];
      }
    }
    __syncthreads();  // (the release below is cumulative over the block's stage writes, as in k_peer_allreduce)
    if (t < pa.world) peer_st_release(reinterpret_cast<u64*>(pa.win[t]) + (size_t)(1 + pa.rank) * kPeerBlocks + b, e);
  }
  if (phases & kPeerPhaseB) {
    __shared__ int timed_out;
    if (t == 0) timed_out = 0;
    __syncthreads();
    const int W = pa.world;
    const int r_first = i0 < i1 ? (int)(i0 / stride) : 0, nr = i0 < i1 ? (int)((i1 - 1) / stride) - r_first + 1 : 0;
    // (1) block b of every rank, (2) the scalar owners of the touched restarts on every rank
    for (int it = t; it < W * (1 + nr); it += blockDim.x) {
      const int q = it % W, k = it / W;
      const int blk = k == 0 ? b : (int)(((size_t)(r_first + k - 1) * stride) / cs);
      if (!peer_wait(own + (size_t)(1 + q) * kPeerBlocks + blk, e, timeout_ns)) timed_out = 1;
    }
    // (3) for the restarts whose scalar this block owns: the own rank's blocks that touch the restart
    for (int k = 0; k < nr; ++k) {
      const size_t base = (size_t)(r_first + k) * stride;
      if (base < i0) continue;  // the scalar lies in an earlier block's slice
      const int lo = (int)(base / cs), hi = (int)((base + stride - 1) / cs);
      for (int blk = lo + t; blk <= hi; blk += blockDim.x)
        if (!peer_wait(own + (size_t)(1 + pa.rank) * kPeerBlocks + blk, e, timeout_ns)) timed_out = 1;
    }
    __syncthreads();
    if (timed_out) {
      if (t == 0) atomicOr(pa.status, kPeerTimeoutBit);
      return;
    }
    int rc = -1;
    double S = 0.0, norm = 0.0;
    int r = (int)(min(T, i0 + t) / stride);
    size_t j = i0 + t - (size_t)r * stride;
#pragma unroll 2
    for (size_t i = i0 + t; i < i1; i += blockDim.x, j += blockDim.x) {
      while (j >= stride) {  // (restart, offset) of i without a 64-bit division per element
        j -= stride;
        ++r;
      }
      if (r != rc) {
        S = 0.0;
        for (int q = 0; q < W; ++q)  // fixed rank order
          S += __ldcg(reinterpret_cast<const double*>(pa.win[q] + stage_off) + (size_t)r * stride);
        norm = 0.0;
        if (a.mode != 0 && S > 0.0) norm = a.mode == 1 ? 1.0 / S : pow(S, 1.0 / a.bp - 1.0);
        rc = r;
      }
      if (j == 0) {
        u64 key[3] = {0ull, 0ull, 0ull};
        for (int q = 0; q < W; ++q) {
          const u64* kq = reinterpret_cast<const u64*>(pa.win[q] + stage_off) + pa.cap_sum + 3 * (size_t)r;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const u64 v = __ldcg(kq + c);
            key[c] = v > key[c] ? v : key[c];
          }
        }
        const double mr = a.mref[r];
        Red rr;
        rr.m = (a.mode != 0 && S > 0.0) ? mr : -INFINITY;
        rr.S = a.mode != 0 ? S : 0.0;
        rr.key_a = key[0];
        rr.key_c = key[1];
        rr.tie = rr.pad = 0u;
        a.red[r] = rr;
        if (!isfinite(S)) atomicOr(pa.status, ST_NONFINITE);
        if (key[2] && a.mode != 0) a.mref[r] = __longlong_as_double((long long)key[2]);
      } else {
        double s = 0.0;
        for (int q = 0; q < W; ++q)
          s += __ldcg(reinterpret_cast<const double*>(pa.win[q] + stage_off) + i);
        reinterpret_cast<float*>(a.grad)[(size_t)r * n + (j - 1)] = (float)(s * norm);
      }
    }
    __syncthreads();
    if (t == 0) own[b] = e;
  }
}

inline bool PeerComm::fused(const WorldArgs* wa, cudaStream_t st, std::string* why) {
  k_world_peer<<<peer_grid(own.cap_sum, own.cap_max), kPeerThreads, 0, st>>>(*wa, args, kPeerPhaseA | kPeerPhaseB, timeout_ns);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { *why = cudaGetErrorString(e); return false; }
  return true;
}

// Loopback group in peer_fused mode: the same rendezvous as LoopComm::allreduce, the last-arriving rank
// launches phase A for every rank and then phase B for every rank (every wait already satisfied).
inline bool LoopComm::fused(const WorldArgs* wa, cudaStream_t st, std::string* why) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (cap_sum > g->cap_sum) g->cap_sum = cap_sum;
  if (cap_max > g->cap_max) g->cap_max = cap_max;
  if (g->arrived == 0) g->err.clear();
  g->wargs[rank] = wa;
  g->status[rank] = status;
  cudaEventRecord(g->ready[rank], st);
  const long long gen = g->generation;
  if (++g->arrived == g->world) {
    for (int r = 0; r < g->world; ++r) cudaStreamWaitEvent(st, g->ready[r], 0);
    for (int r = 0; r < g->world && g->err.empty(); ++r)
      if (!g->win[r].base && g->win[r].alloc(g->cap_sum, g->cap_max) != cudaSuccess)
        g->err = "loopback: peer window allocation";
    for (int ph = kPeerPhaseA; ph <= kPeerPhaseB && g->err.empty(); ph <<= 1)
      for (int r = 0; r < g->world; ++r) {
        if (ph == kPeerPhaseA && r == g->drop_signal_rank) continue;  // (tests) a rank that never signals
        PeerArgs a{};
        for (int q = 0; q < g->world; ++q) a.win[q] = g->win[q].base;
        a.world = g->world;
        a.rank = r;
        a.cap_sum = g->win[0].cap_sum;
        a.cap_max = g->win[0].cap_max;
        a.status = g->status[r];
        k_world_peer<<<peer_grid(a.cap_sum, a.cap_max), kPeerThreads, 0, st>>>(*g->wargs[r], a, ph, 2000000000ull);
      }
    cudaEventRecord(g->done, st);
    g->arrived = 0;
    ++g->generation;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->generation != gen; });
    if (g->err.empty()) cudaStreamWaitEvent(st, g->done, 0);
  }
  if (!g->err.empty()) { *why = g->err; return false; }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { *why = cudaGetErrorString(e); return false; }
  return true;
}

}  // namespace sq
