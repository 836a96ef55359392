// Does a co-resident warp spinning on a shared flag (LDS + nanosleep) or on a
// global tag (ld.relaxed.gpu + nanosleep) slow a chain warp down?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t ldr(const uint64_t* p) {
  uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)); return v; }
__global__ void k(const uint32_t* in, uint32_t* out, long long* cyc, int nblk, int mode, uint64_t* g) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ uint32_t ring[4][32][64];
  __shared__ volatile int flag;
  if (threadIdx.x == 0) flag = 0;
  for (int q = threadIdx.x; q < 4 * 32 * 64; q += blockDim.x) (&ring[0][0][0])[q] = in[q & 4095];
  __syncthreads();
  if ((wid & 1) && mode) {   // spinner
    long long n = 0;
    while (flag == 0) {
      if (mode == 1) { __nanosleep(20); n++; }
      else if (mode == 2) { uint64_t w = ldr(g + lane); if (w == 12345) n++; __nanosleep(20); }
      else { n++; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)n;
    return;
  }
  uint32_t rl = 0, rul = 0, rlast = 0, acc = 0;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
    uint32_t av[32];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) av[jj] = ring[wid & 3][lane][(m * 32 + jj - lane) & 63];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      uint32_t ru = __shfl_up_sync(0xffffffffu, rlast, 1);
      if (lane == 0) ru = jj;
      uint32_t t = rl + (av[jj] - rul);
      uint32_t r = ((av[jj] & 7) == 0) ? av[jj] : ru + t;
      av[jj] = r; rl = r; rlast = r; rul = ru;
    }
#pragma unroll
    for (int jj = 0; jj < 32; jj++) ring[wid & 3][lane][(m * 32 + jj - lane) & 63] = av[jj];
    acc += rl;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * 32 + wid] = t1 - t0;
  __syncwarp();
  if (lane == 0 && wid == 0) { __threadfence_block(); flag = 1; }
}
int main() {
  uint32_t *in, *out; long long* cyc; uint64_t* g;
  cudaMalloc(&in, 4 * 4096); cudaMalloc(&out, 4 * 148 * 1024); cudaMalloc(&cyc, 8 * 148 * 32); cudaMalloc(&g, 8 * 64);
  cudaMemset(in, 1, 4 * 4096); cudaMemset(g, 0, 512);
  int nblk = 2000;
  for (int mode : {0, 1, 2, 3}) for (int wpb : {2, 8}) {
    k<<<148, 32 * wpb>>>(in, out, cyc, nblk, mode, g);
    cudaDeviceSynchronize();
    long long h[32]; cudaMemcpy(h, cyc, 8 * wpb, cudaMemcpyDeviceToHost);
    printf("mode %d warps %d: chain warp0 %.1f cycles/block\n", mode, wpb, (double)h[0] / nblk);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
