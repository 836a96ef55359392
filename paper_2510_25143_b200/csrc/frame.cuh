// Per-frame parameters and small primitives shared by the frame kernels
// (fast.cu) and the block-scan chain (bscan.cuh).
#pragma once

#include "common.cuh"
#include "wavefront.cuh"

namespace vfcp {

struct PrepParams {
  int H, W, Wp, nchunks, nbx, nby, t;
  double S, cfl_x, cfl_y, d_max, lam, theta, rmeta;
  int n_max, stride, radius;
  int64_t tau;
  int mop;          // run the MoP trial for this frame
  int force_sl;     // predictor 'sl' (and t >= 1, tau > 0)
  uint32_t lossy_mask;   // bit c: code c quantises (e > 0)
  Ladder lad;
};

// exact rha(x / 2e) for integer x, e > 0, |x| < 2^31
__device__ __forceinline__ int32_t quant32(int32_t x, int32_t e, double inv2e) {
  const int32_t two_e = 2 * e;
  int32_t q = __double2int_rn(__dmul_rn((double)x, inv2e));
  int32_t rem = x - q * two_e;
  if (rem > e) { q += 1; rem -= two_e; }
  else if (rem < -e) { q -= 1; rem += two_e; }
  if (rem == e && x > 0) q += 1;
  else if (rem == -e && x < 0) q -= 1;
  return q;
}

// Warp-uniform wait for a shared-memory counter.  The chain warps poll
// tightly (they are on the critical path); the producers back off so their
// polling does not take issue slots and shared-memory bandwidth from the
// chain warp on the same sub-partition.
// The counters use acquire loads / release stores at CTA scope instead of
// full fences: a fence would also wait for the warp's outstanding global
// loads (the prefetched boundary slots).
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}
template <int SLEEP_NS = 0>
__device__ __forceinline__ void spin_ge(const int* p, int need) {
  while (!__all_sync(0xffffffffu, ld_acquire_cta(p) >= need)) {
    if (SLEEP_NS) __nanosleep(SLEEP_NS);
  }
}
__device__ __forceinline__ void signal_set(int* p, int v, int lane) {
  __syncwarp();   // the warp's writes happen before lane 0's release
  if (lane == 0) st_release_cta(p, v);
  __syncwarp();
}

}  // namespace vfcp
