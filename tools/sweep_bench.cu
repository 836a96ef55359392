// Microbenchmark: cycles per step of the chain sweeps (chain.cuh) on
// register-resident operands, one warp alone on its SM sub-partition.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dec_sweep(const int32_t* in, int nblk, uint32_t pm, long long* out, int32_t* sink) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t av[32];
  for (int jj = 0; jj < 32; jj++) av[jj] = in[lane * 32 + jj];
  int32_t l = 0, ul = 0, b = in[lane];
  const bool lane0 = lane == 0;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      const int32_t bb = __shfl_sync(FULL, b, jj);
      const int32_t up = __shfl_up_sync(FULL, l, 1);
      const int32_t nu = lane0 ? bb : up;
      const int32_t t = (int32_t)((uint32_t)av[jj] - (uint32_t)ul);
      const int32_t r = ((pm >> jj) & 1u) ? av[jj]
          : (int32_t)((uint32_t)nu + (uint32_t)l + (uint32_t)t);
      av[jj] = r;
      l = r;
      ul = nu;
    }
    b += l;
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = t1 - t0;
  int32_t acc = 0;
  for (int jj = 0; jj < 32; jj++) acc += av[jj];
  sink[blockIdx.x * 32 + lane] = acc;
}

__global__ void enc_sweep(const int32_t* in, int nblk, uint32_t pm, long long* out, int32_t* sink) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t rr[32], qq[32], ee[32];
  for (int jj = 0; jj < 32; jj++) { rr[jj] = in[lane * 32 + jj] % 1000; qq[jj] = in[lane * 32 + jj] % 7; ee[jj] = 1000; }
  int32_t l = 0, ul = 0, b = in[lane] % 100;
  const int32_t radius = 32768;
  const bool lane0 = lane == 0;
  bool slow = false;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      const int32_t rho = rr[jj], q0 = qq[jj], e = ee[jj];
      const int32_t bb = __shfl_sync(FULL, b, jj);
      const int32_t up = __shfl_up_sync(FULL, l, 1);
      const int32_t nu = lane0 ? bb : up;
      const int32_t d = nu + l - ul;
      const int32_t y = rho - d;
      const int32_t e3 = 3 * e;
      const int32_t gf = (y >= e) + (y >= e3) - (y < -e) - (y < -e3);
      const int32_t ay = y < 0 ? -y : y;
      const bool tie = (ay == e) | (ay == e3);
      const int32_t qf = q0 + gf;
      const int32_t q = qf - ((tie && qf <= 0) ? 1 : 0);
      const bool esc = (uint32_t)(q + radius - 1) >= (uint32_t)(2 * radius - 1);
      const bool pin = (pm >> jj) & 1u;
      const int32_t r = pin ? rho : (esc ? 0 : (q - q0) * 2 * e - y);
      qq[jj] = (pin || esc) ? 0 : q + radius;
      slow |= (e != 0) & (ay >= 4 * e);
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


__global__ void enc_sweep2(const int32_t* in, int nblk, uint32_t pm, long long* out, int32_t* sink) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t rr[32], qq[32], ee[32];
  for (int jj = 0; jj < 32; jj++) { rr[jj] = in[lane * 32 + jj] % 1000; qq[jj] = in[lane * 32 + jj] % 7; ee[jj] = 1000; }
  int32_t l = 0, ul = 0, b = in[lane] % 100;
  const int32_t radius = 32768;
  const bool lane0 = lane == 0;
  bool slow = false;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      const int32_t rho = rr[jj], q0 = qq[jj], e = ee[jj];
      const int32_t e2 = 2 * e;
      const int32_t R0 = q0 * e2 + rho;
      const int32_t T1 = rho - e, T2 = T1 - e2, T3 = rho + e, T4 = T3 + e2;
      const int32_t bb = __shfl_sync(FULL, b, jj);
      const int32_t up = __shfl_up_sync(FULL, l, 1);
      const int32_t nu = lane0 ? bb : up;
      const int32_t d = nu + l - ul;
      const int32_t gu = (d <= T1) + (d <= T2) - (d > T3) - (d > T4);
      const int32_t gd = (d < T1) + (d < T2) - (d >= T3) - (d >= T4);
      const int32_t g = d < R0 ? gu : gd;
      const int32_t q = q0 + g;
      const bool esc = (uint32_t)(q + radius - 1) >= (uint32_t)(2 * radius - 1);
      const bool pin = (pm >> jj) & 1u;
      const int32_t er = g * e2 + (d - rho);
      const int32_t r = pin ? rho : (esc ? 0 : er);
      qq[jj] = (pin || esc) ? 0 : q + radius;
      slow |= (e != 0) & ((d <= T2 - e) | (d >= T4 + e));
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

template <int NC>
__global__ void enc_sweep3(const int32_t* in, int nblk, uint32_t pm, long long* out, int32_t* sink) {
  // NC independent chains (components) per lane, sign-shift threshold form
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t rr[NC][32], qq[NC][32], ee[32];
  for (int jj = 0; jj < 32; jj++) {
    for (int c = 0; c < NC; c++) { rr[c][jj] = (in[lane * 32 + jj] + c) % 1000; qq[c][jj] = in[lane * 32 + jj] % 7; }
    ee[jj] = 1000;
  }
  int32_t l[NC], ul[NC];
  for (int c = 0; c < NC; c++) { l[c] = 0; ul[c] = 0; }
  int32_t b = in[lane] % 100;
  const int32_t radius = 32768;
  const bool lane0 = lane == 0;
  bool slow = false;
  long long t0 = clock64();
  for (int m = 0; m < nblk; m++) {
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      const int32_t e = ee[jj], e2 = 2 * e;
      const bool pin = (pm >> jj) & 1u;
      const int32_t bb = __shfl_sync(FULL, b, jj);
#pragma unroll
      for (int c = 0; c < NC; c++) {
        const int32_t rho = rr[c][jj], q0 = qq[c][jj];
        const int32_t up = __shfl_up_sync(FULL, l[c], 1);
        const int32_t nu = lane0 ? bb : up;
        const int32_t d = nu + l[c] - ul[c];
        const int32_t x = rho - d;                       // y
        // g_up = 2 + sum sign((T - d)), T in {rho-e, rho-3e, rho+e, rho+3e}
        const int32_t gu = 2 + ((x - e) >> 31) + ((x - 3 * e) >> 31) +
                           ((x + e) >> 31) + ((x + 3 * e) >> 31);
        const int32_t gd = 2 + ((x - e - 1) >> 31) + ((x - 3 * e - 1) >> 31) +
                           ((x + e - 1) >> 31) + ((x + 3 * e - 1) >> 31);
        const int32_t R0 = q0 * e2 + rho;
        const int32_t g = d < R0 ? gu : gd;
        const int32_t q = q0 + g;
        const bool esc = (uint32_t)(q + radius - 1) >= (uint32_t)(2 * radius - 1);
        const int32_t er = g * e2 - x;
        const int32_t r = pin ? rho : (esc ? 0 : er);
        qq[c][jj] = (pin || esc) ? 0 : q + radius;
        slow |= (e != 0) & ((uint32_t)(x + 4 * e) > (uint32_t)(8 * e));
        rr[c][jj] = r;
        l[c] = r;
        ul[c] = nu;
      }
    }
    if (__any_sync(FULL, slow)) b += 1;
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = t1 - t0;
  int32_t acc = 0;
  for (int jj = 0; jj < 32; jj++) for (int c = 0; c < NC; c++) acc += rr[c][jj] + qq[c][jj];
  sink[blockIdx.x * 32 + lane] = acc;
}

int main() {
  int32_t *in, *sink; long long* out;
  cudaMalloc(&in, 4096); cudaMalloc(&sink, 1 << 20); cudaMallocManaged(&out, 8 * 1024);
  cudaMemset(in, 1, 4096);
  const int nblk = 1000;
  for (int warps = 1; warps <= 8; warps *= 2) {
    dec_sweep<<<148, 32 * warps>>>(in, nblk, 0x10101010u, out, sink);
    cudaDeviceSynchronize();
    printf("dec warps/CTA=%d: %.1f cycles/step\n", warps, (double)out[0] / nblk / 32);
    enc_sweep<<<148, 32 * warps>>>(in, nblk, 0x10101010u, out, sink);
    cudaDeviceSynchronize();
    printf("enc warps/CTA=%d: %.1f cycles/step\n", warps, (double)out[0] / nblk / 32);
    enc_sweep2<<<148, 32 * warps>>>(in, nblk, 0x10101010u, out, sink);
    cudaDeviceSynchronize();
    printf("enc2 warps/CTA=%d: %.1f cycles/step\n", warps, (double)out[0] / nblk / 32);
    enc_sweep3<1><<<148, 32 * warps>>>(in, nblk, 0x10101010u, out, sink);
    cudaDeviceSynchronize();
    printf("enc3x1 warps/CTA=%d: %.1f cycles/step\n", warps, (double)out[0] / nblk / 32);
    enc_sweep3<2><<<148, 32 * warps>>>(in, nblk, 0x10101010u, out, sink);
    cudaDeviceSynchronize();
    printf("enc3x2 warps/CTA=%d: %.1f cycles/step\n", warps, (double)out[0] / nblk / 32);
  }
  return 0;
}
