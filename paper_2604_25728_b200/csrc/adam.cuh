// Status bits and the Adam parameter block, shared by every translation unit (no device code
// with external linkage here: common.cuh's functions stay in one TU).
#pragma once

// Programmatic dependent launch: every kernel first waits for its programmatic predecessors (a
// no-op without one), so sqngd_step can turn the kernel-to-kernel edges of its CUDA graph into
// programmatic edges and overlap each launch with the previous kernel's tail.
#define SQ_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

namespace sq {

enum : int { ST_INVALID = 1, ST_DEGENERATE = 2, ST_NONFINITE = 4 };

// Adam hyper-parameters; the step count t = dt[which] + off + 1 is read on the device so a
// captured CUDA graph stays valid from one sqngd_step call to the next (bias corrections, Q15).
struct AdamP {
  float lr, b1, b2, eps;
  const long long* dt;
  int which, off;
  const float2* ct = nullptr;  // optional [2][cts] table of (c1, c2) per block and inner step (k_set_t)
  int cts = 0;
  __device__ __forceinline__ void corr(float& c1, float& c2) const {
    if (ct) {  // precomputed once per sqngd_step: one load instead of two fp64 pow chains
      const float2 v = ct[which * cts + off];
      c1 = v.x;
      c2 = v.y;
      return;
    }
    const double t = (double)(dt[which] + off + 1);
    c1 = (float)(1.0 - pow((double)b1, t));
    c2 = (float)(1.0 - pow((double)b2, t));
  }
};

}  // namespace sq
