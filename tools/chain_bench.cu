// Microbenchmark: cycles per 32-step chain block for the decoder's chain
// loop shape (register-resident values, shfl-up recurrence), with and without
// co-resident warps.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__global__ void chain(const uint32_t* in, uint32_t* out, long long* cyc, int nblk, int mode) {
  const int lane = threadIdx.x & 31;
  __shared__ uint32_t ring[32][64];
  for (int k = threadIdx.x; k < 32 * 64; k += blockDim.x) (&ring[0][0])[k] = in[k];
  __syncthreads();
  uint32_t rl = 0, rul = 0, rlast = 0, acc = 0;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
    uint32_t av[32];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) av[jj] = ring[lane][(m * 32 + jj - lane) & 63];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      uint32_t ru = __shfl_up_sync(0xffffffffu, rlast, 1);
      if (lane == 0) ru = jj;
      uint32_t t = rl + (av[jj] - rul);
      uint32_t r = ((av[jj] & 7) == 0) ? av[jj] : ru + t;
      av[jj] = r; rl = r; rlast = r; rul = ru;
    }
#pragma unroll
    for (int jj = 0; jj < 32; jj++) ring[lane][(m * 32 + jj - lane) & 63] = av[jj];
    acc += rl;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}
int main() {
  uint32_t *in, *out; long long* cyc;
  cudaMalloc(&in, 4 * 4096); cudaMalloc(&out, 4 * 148 * 1024); cudaMalloc(&cyc, 8 * 148 * 32);
  cudaMemset(in, 1, 4 * 4096);
  int nblk = 2000;
  for (int wpb : {1, 4, 8, 16}) {
    chain<<<148, 32 * wpb>>>(in, out, cyc, nblk, 0);
    cudaDeviceSynchronize();
    long long h[32]; cudaMemcpy(h, cyc, 8 * wpb, cudaMemcpyDeviceToHost);
    printf("warps/SM %d: %.1f cycles per 32-step block (%.1f per step)\n", wpb, (double)h[0] / nblk, (double)h[0] / nblk / 32);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
