// Cycles per step of the encoder chain step used by chain_kernel<true>
// (enc_step_fast in chain.cuh) with per-pixel step sizes.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2510_25143_b200/csrc/chain.cuh"
using namespace vfcp;
__global__ void enc_sweep(const int32_t* in, int nblk, uint32_t pm, long long* out, int32_t* sink) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t rr[32], qq[32], ee[32];
  for (int jj = 0; jj < 32; jj++) { rr[jj] = in[lane * 32 + jj] % 100000; qq[jj] = in[lane * 32 + jj] % 7; ee[jj] = 1000 + (in[lane * 32 + jj] & 3); }
  int32_t l = 0, ul = 0, b = in[lane] % 100;
  const int32_t radius = in[5] | 32768;
  const bool lane0 = lane == 0;
  bool slow = false;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      const int32_t R0 = rr[jj], q0 = qq[jj], e = ee[jj];
      const int32_t rho = R0 - q0 * (2 * e);
      const int32_t bb = __shfl_sync(FULL, b, jj);
      const int32_t up = __shfl_up_sync(FULL, l, 1);
      const int32_t nu = lane0 ? bb : up;
      const int32_t d = nu + l - ul;
      uint32_t sy;
      const int32_t er = enc_step_fast(R0, q0, rho, e, d, radius, &sy);
      const bool pin = (pm >> jj) & 1u;
      const int32_t r = pin ? R0 : er;
      qq[jj] = pin ? 0 : (int32_t)sy;
      slow |= (e != 0) & ((uint32_t)(rho - d + 4 * e) > (uint32_t)(8 * e));
      rr[jj] = r;
      l = r;
      ul = nu;
    }
    if (__any_sync(FULL, slow)) b += 1;
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = t1 - t0;
  int32_t acc = 0;
  for (int jj = 0; jj < 32; jj++) acc += rr[jj] + qq[jj];
  sink[blockIdx.x * 32 + lane] = acc;
}
int main() {
  int32_t *in, *sink; long long* out;
  cudaMalloc(&in, 4096); cudaMalloc(&sink, 1 << 20); cudaMallocManaged(&out, 8 * 1024);
  cudaMemset(in, 1, 4096);
  const int nblk = 1000;
  enc_sweep<<<148, 32>>>(in, nblk, 0x10101010u, out, sink);
  cudaDeviceSynchronize();
  printf("enc_step_fast: %.1f cycles/step\n", (double)out[0] / nblk / 32);
  return 0;
}
