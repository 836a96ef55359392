// Persistent space-time wavefront scheduling shared by the encoder and the
// decoder.
//
// The reference's frame loop (codec.py:359-376, 427-446) is sequential in t
// and raster-ordered inside a frame.  On the device a *task* is one 32-row
// strip of one frame, executed by one warp (lane = row) that sweeps the
// columns with a one-column skew per lane, so every Lorenzo neighbour
// (up / left / up-left) is final when it is read.  Tasks are handed out in
// (frame, strip) order by an atomic ticket; a task only waits on tasks with
// smaller tickets (the strip above in the same frame, and the strips of the
// previous frame within the semi-Lagrangian reach), which are already
// resident, so the schedule cannot deadlock.  Frames overlap: frame t+1's
// strip k starts as soon as frame t has progressed past the rows and columns
// it reads, so the critical path is ~(W + H + T * lag) steps instead of
// T * (W + H).
//
// Progress is published per 32-column chunk with release semantics
// (__threadfence + atomic store); consumers poll with volatile loads and read
// the produced data through L2 (ld.global.cg).
#pragma once

#include "common.cuh"

namespace vfcp {

struct WaveSched {
  int* ticket;     // [1]
  int* prog;       // [T * K] columns fully written (all rows of the strip)
  int* bprog;      // [T * K] columns of the strip's last row in `bnd`
  int K;           // strips per frame
  int reach_strips;  // previous-frame strips each side a strip reads
  int reach_cols;    // previous-frame columns ahead a chunk reads
  unsigned long long* stats;  // optional per-phase cycle counters (profiling)
};

// Phase timers (only when ws.stats != nullptr): accumulate clock64 deltas.
enum WavePhase { WP_WAITPREV, WP_PRE, WP_WAITBND, WP_CHAIN, WP_WRITE,
                 WP_TASKS, WP_TOTAL, WP_X1, WP_X2, WP_X3, WP_N };
struct PhaseClock {
  unsigned long long* stats;
  long long t0;
  __device__ __forceinline__ explicit PhaseClock(unsigned long long* s)
      : stats(s), t0(0) {
#ifdef __CUDA_ARCH__
    if (s) t0 = clock64();
#endif
  }
  __device__ __forceinline__ void lap(int phase, int lane) {
#ifdef __CUDA_ARCH__
    if (stats) {
      long long t1 = clock64();
      if (lane == 0) atomicAdd(stats + phase, (unsigned long long)(t1 - t0));
      t0 = t1;
    }
#endif
  }
};

__device__ __forceinline__ int ld_volatile(const int* p) {
  return *(volatile const int*)p;
}

__device__ __forceinline__ void publish(int* p, int v) {
  __threadfence();
  atomicMax(p, v);
}

// Spin until *p >= need, then acquire.  Every lane polls the same word and
// the loop condition is warp-uniform (__all_sync): a lane-0-only spin with
// __nanosleep leaves the warp split into lane groups afterwards, and every
// later shuffle then takes the slow divergent (WARPSYNC.COLLECTIVE) path.
__device__ __forceinline__ void wait_ge(const int* p, int need, int lane) {
  (void)lane;
  while (!__all_sync(0xffffffffu, ld_volatile(p) >= need)) __nanosleep(64);
  __threadfence();
}

// Asynchronous global->shared copies (cp.async, LDGSTS).  `valid` false
// zero-fills the destination without touching the source.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src,
                                         bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d),
               "l"(src), "n"(BYTES), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p,
                                                   unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

// Tagged single-copy-atomic handoff slots: each 64-bit word carries a 32-bit
// tag (the producer task's ticket + 1) and 32 bits of payload, so a consumer
// can spin on the data itself with no fence on the producer side (the strip
// boundary row is on the critical path of the wavefront).
template <typename IW>
struct TaggedSlot {
  static constexpr int SLOTS = sizeof(IW) / 4;
  __device__ __forceinline__ static void put(uint64_t* s, uint32_t tag, IW v) {
#pragma unroll
    for (int h = 0; h < SLOTS; h++) {
      uint64_t w = ((uint64_t)tag << 32) |
                   (uint32_t)((uint64_t)(int64_t)v >> (32 * h));
      st_relaxed_u64(s + h, w);
    }
  }
  // Warp-collective: every lane waits for its own slot (lanes with
  // valid == false pass immediately); the loop is warp-uniform.
  __device__ __forceinline__ static IW get(const uint64_t* s, uint32_t tag,
                                          bool valid) {
    uint64_t v = 0;
#pragma unroll
    for (int h = 0; h < SLOTS; h++) {
      uint64_t w = valid ? ld_relaxed_u64(s + h) : 0;
      bool ok = !valid || (uint32_t)(w >> 32) == tag;
      while (!__all_sync(0xffffffffu, ok)) {
        // poll again (no sleep: wake-up granularity exceeds the handoff)
        if (!ok) {
          w = ld_relaxed_u64(s + h);
          ok = (uint32_t)(w >> 32) == tag;
        }
      }
      v |= (uint64_t)(uint32_t)w << (32 * h);
    }
    return (IW)(int64_t)v;
  }
};

}  // namespace vfcp
