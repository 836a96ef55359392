// Microbenchmark: per-op latency of warp collectives for a lone warp, and
// with sibling warps spinning on shared memory (chain-kernel cost model).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__global__ void k(long long* out, int mode, int spin_ns) {
  __shared__ int flag;
  __shared__ int buf[64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) flag = 0;
  if (threadIdx.x < 64) buf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (w > 0) {
    if (mode == 0) return;
    // spin until warp 0 finishes
    while (!__all_sync(0xffffffffu, ld_acq(&flag) != 0)) {
      if (spin_ns) __nanosleep(spin_ns);
    }
    return;
  }
  const unsigned FULL = 0xffffffffu;
  int x = lane;
  long long t[8];
  t[0] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) x = __shfl_sync(FULL, x, (lane + 1) & 31) + 1;
  t[1] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) x = x * 3 + i;
  t[2] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) { int y = __shfl_up_sync(FULL, x, 1); if (lane == (i & 3)) x = y + 1; }
  t[3] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) { if (__any_sync(FULL, x == i)) x++; }
  t[4] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) x = buf[x & 63];
  t[5] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) { if (x > 1000) x -= 977; x += buf[lane]; if (x > 1000) x -= 977; }
  t[6] = clock64();
#pragma unroll
  for (int i = 0; i < 32; i++) { __syncwarp(); if (lane == 0) buf[32] = x + i; __syncwarp(); x += buf[32]; }
  t[7] = clock64();
  if (lane == 0) {
    for (int i = 0; i < 7; i++) out[i] = t[i + 1] - t[i];
    out[7] = x;
  }
  __syncwarp();
  if (lane == 0) { __threadfence_block(); *(volatile int*)&flag = 1; }
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h[8];
  const char* names[7] = {"shfl x32", "imad x32", "shfl_up+if(lane) x32", "any+if x32", "lds chain x32", "cond-sub x32", "syncwarp+sts+lds x32"};
  for (int mode = 0; mode < 3; mode++) {
    int ns = mode == 2 ? 64 : 0;
    for (int rep = 0; rep < 2; rep++) {
      k<<<1, 256>>>(d, mode ? 1 : 0, ns);
      cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    }
    printf("mode %d (%s):\n", mode, mode == 0 ? "lone warp" : mode == 1 ? "7 warps spinning" : "7 warps spinning, nanosleep 64");
    for (int i = 0; i < 7; i++) printf("  %-24s %6lld cycles (%.1f / op)\n", names[i], h[i], h[i] / 32.0);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
