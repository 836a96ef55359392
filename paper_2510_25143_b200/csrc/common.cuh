// Device-side primitives shared by the vfcp B200 kernels.
//
// Every binary64 operation that the reference performs (numba, IEEE, no FMA
// contraction -- SURVEY.md V2) is written with explicit round-to-nearest
// intrinsics (__dmul_rn / __dadd_rn / __dsub_rn) and the whole library is
// compiled with -fmad=false, so the device reproduces the reference's float64
// results bit for bit.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace vfcp {

constexpr int CODE_LOSSLESS = 31;
constexpr int K_MAX = 30;

// Per-run constants for the quantisation ladder: e_k = tau' >> k.
struct Ladder {
  int64_t e[32];        // e per code (0 for code 31)
  double inv2e[32];     // 1 / (2 e) (0 for code 31)
};

// Per-frame settings of the compress kernels (codec.py:44-68 Config + the
// derived CFL factors of predictors.py:117-119).
struct FrameParams {
  int H, W, T, t;
  double S;
  int64_t tau;
  int radius;
  int bx, by, stride, nbx, nby;
  double lam, theta, rmeta, d_max;
  int n_max;
  double cfl_x, cfl_y;
  int use_modes;          // t >= 1 (modes of this frame valid)
};

// Per-frame settings of the decode kernels.
struct DecodeParams {
  int H, W, T, t;
  int64_t n_qd, n_ll;     // stream lengths (debug bounds checks)
  double inv_S, S;
  int radius;
  int bx, by, nbx;
  double d_max;
  int n_max;
  double cfl_x, cfl_y;
  int use_modes;
};

#ifdef VFCP_DEBUG
#define VFCP_CHECK(cond, tag)                                                \
  do {                                                                       \
    if (!(cond)) {                                                           \
      printf("VFCP_CHECK failed: %s (%s:%d) block %d thread %d\n", tag,      \
             __FILE__, __LINE__, blockIdx.x, threadIdx.x);                   \
      __trap();                                                              \
    }                                                                        \
  } while (0)
#else
#define VFCP_CHECK(cond, tag) \
  do {                        \
  } while (0)
#endif

// Host: a per-device "done" flag for one-time launch setup (kernel
// attributes, occupancy queries), so the per-frame launch loop of a small
// field does not pay for them at every frame.
struct OncePerDevice {
  int val[64];
  bool done[64] = {};
  template <typename Fn>
  cudaError_t get(Fn&& init, int* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return init(out);
    if (!done[dev]) {
      e = init(&val[dev]);
      if (e != cudaSuccess) return e;
      done[dev] = true;
    }
    *out = val[dev];
    return cudaSuccess;
  }
};

// predictors.py:25-30 _rha: round half away from zero (float64 -> int64).
__device__ __forceinline__ int64_t rha_d(double x) {
  if (x >= 0.0) return (int64_t)floor(__dadd_rn(x, 0.5));
  return -(int64_t)floor(__dadd_rn(-x, 0.5));
}

// the same for |x| < 2^31 - 1 (one 32-bit conversion)
__device__ __forceinline__ int32_t rha_d32(double x) {
  const int32_t r = __double2int_rd(__dadd_rn(fabs(x), 0.5));
  return x < 0.0 ? -r : r;
}

// field.py:295-297 / 313-336: sign(x*S) * floor(|x*S| + 0.5).
__device__ __forceinline__ int32_t fixed_of(double x, double S) {
  double y = __dmul_rn(x, S);
  double a = floor(__dadd_rn(fabs(y), 0.5));
  int32_t q = (int32_t)a;
  return y > 0.0 ? q : (y < 0.0 ? -q : 0);
}

// binary32 input: x*S is exact in binary32 (S = 2^k, |x*S| < 2^30), and so
// are its integer and fractional parts, so rounding half away from zero in
// binary32 gives the reference's binary64 result with a few FP32 ops.
__device__ __forceinline__ int32_t fixed_of_f32(float x, float S) {
  // below 2^23 the sum y +- 0.5 is exact (ulp(y) <= 0.5) and truncation
  // rounds half away from zero; from 2^23 on y is an integer
  const float y = __fmul_rn(x, S);
  const float h = fabsf(y) < 8388608.0f ? 0.5f : 0.0f;
  return __float2int_rz(__fadd_rn(y, copysignf(h, y)));
}
__device__ __forceinline__ int32_t fixed_t(float x, double S) {
  return fixed_of_f32(x, (float)S);
}
__device__ __forceinline__ int32_t fixed_t(double x, double S) {
  return fixed_of(x, S);
}

template <typename F>
__device__ __forceinline__ int32_t load_fixed(const F* p, int64_t k, double S) {
  return fixed_t(__ldg(p + k), S);
}

// Exact rha(x / (2e)) for integer x, e > 0 (equal to the reference's
// float64 _rha(r / two_e) for |x| < 2^51): the float64 estimate
// is corrected so that rem = x - q*2e lies in [-e, e], then ties go away
// from zero.
__device__ __forceinline__ int64_t quant_rha(int64_t x, int64_t e,
                                             double inv2e) {
  int64_t two_e = 2 * e;
  int64_t q = __double2ll_rn(__dmul_rn((double)x, inv2e));
  int64_t rem = x - q * two_e;
  if (rem > e) { q += 1; rem -= two_e; }
  else if (rem < -e) { q -= 1; rem += two_e; }
  if (rem > e) { q += 1; rem -= two_e; }
  else if (rem < -e) { q -= 1; rem += two_e; }
  if (rem == e && x > 0) q += 1;
  else if (rem == -e && x < 0) q -= 1;
  return q;
}

// Bilinear weights and corner indices of predictors.py:33-59 _bilinear,
// shared between the u and v samples at the same departure point.
struct BilinearTap {
  int64_t k00, k01, k10, k11;
  double w00, w01, w10, w11;
};

__device__ __forceinline__ BilinearTap bilinear_tap(int H, int W, double i_f,
                                                    double j_f, int pitch) {
  if (i_f < 0.0) i_f = 0.0;
  else if (i_f > (double)(H - 1)) i_f = (double)(H - 1);
  if (j_f < 0.0) j_f = 0.0;
  else if (j_f > (double)(W - 1)) j_f = (double)(W - 1);
  int i0 = (int)floor(i_f), j0 = (int)floor(j_f);
  if (i0 > H - 1) i0 = H - 1;
  if (j0 > W - 1) j0 = W - 1;
  int i1 = i0 + 1 < H - 1 ? i0 + 1 : H - 1;
  int j1 = j0 + 1 < W - 1 ? j0 + 1 : W - 1;
  double a = __dsub_rn(i_f, (double)i0), b = __dsub_rn(j_f, (double)j0);
  double oma = __dsub_rn(1.0, a), omb = __dsub_rn(1.0, b);
  BilinearTap t;
  t.k00 = (int64_t)i0 * pitch + j0;
  t.k01 = (int64_t)i0 * pitch + j1;
  t.k10 = (int64_t)i1 * pitch + j0;
  t.k11 = (int64_t)i1 * pitch + j1;
  t.w00 = __dmul_rn(oma, omb);
  t.w01 = __dmul_rn(oma, b);
  t.w10 = __dmul_rn(a, omb);
  t.w11 = __dmul_rn(a, b);
  return t;
}
__device__ __forceinline__ BilinearTap bilinear_tap(int H, int W, double i_f,
                                                    double j_f) {
  return bilinear_tap(H, W, i_f, j_f, W);
}

// Value sources for the semi-Lagrangian sampler: the value of frame entry k
// as the float64 the reference converts it to ((double) of an int64).
template <typename I>
struct IntSrc {
  const I* p;
  __device__ __forceinline__ double operator()(int64_t k) const {
    return (double)p[k];
  }
};
// an integer frame produced earlier in the same kernel (read through L2)
template <typename I>
struct IntSrcCG {
  const I* p;
  __device__ __forceinline__ double operator()(int64_t k) const {
    return (double)__ldcg(p + k);
  }
};
// a float64 frame holding recon * (1/S): times S is exact (S = 2^k)
struct F64Src {
  const double* p;
  double S;
  __device__ __forceinline__ double operator()(int64_t k) const {
    return __dmul_rn(__ldcg(p + k), S);
  }
};

template <typename Src>
__device__ __forceinline__ int64_t bilinear_src(const BilinearTap& t,
                                                const Src& f) {
  double val = __dmul_rn(t.w00, f(t.k00));
  val = __dadd_rn(val, __dmul_rn(t.w01, f(t.k01)));
  val = __dadd_rn(val, __dmul_rn(t.w10, f(t.k10)));
  val = __dadd_rn(val, __dmul_rn(t.w11, f(t.k11)));
  return rha_d(val);
}

template <typename I>
__device__ __forceinline__ int64_t bilinear_apply(const BilinearTap& t,
                                                  const I* f) {
  return bilinear_src(t, IntSrc<I>{f});
}

// predictors.py:76-108 _sl_departure on the reconstructed frame t-1.
template <typename Src>
__device__ __forceinline__ void sl_departure_src(const Src& up, const Src& vp,
                                                 int H, int W, int i, int j,
                                                 double cfl_x, double cfl_y,
                                                 double d_max, int n_max,
                                                 double* oi, double* oj,
                                                 int pitch) {
  int64_t k = (int64_t)i * pitch + j;
  double u0 = up(k), v0 = vp(k);
  double ax = __dmul_rn(fabs(u0), cfl_x), ay = __dmul_rn(fabs(v0), cfl_y);
  double d_inf = ay > ax ? ay : ax;
  if (d_inf <= d_max) {
    double ih = __dsub_rn((double)i, __dmul_rn(__dmul_rn(0.5, v0), cfl_y));
    double jh = __dsub_rn((double)j, __dmul_rn(__dmul_rn(0.5, u0), cfl_x));
    BilinearTap t = bilinear_tap(H, W, ih, jh, pitch);
    double um = (double)bilinear_src(t, up);
    double vm = (double)bilinear_src(t, vp);
    *oi = __dsub_rn((double)i, __dmul_rn(vm, cfl_y));
    *oj = __dsub_rn((double)j, __dmul_rn(um, cfl_x));
    return;
  }
  int64_t n = (int64_t)ceil(__ddiv_rn(d_inf, d_max));
  if (n > n_max) n = n_max;
  double dn = (double)n;
  double fi = (double)i, fj = (double)j;
  for (int64_t s = 0; s < n; s++) {
    BilinearTap t = bilinear_tap(H, W, fi, fj, pitch);
    double us = (double)bilinear_src(t, up);
    double vs = (double)bilinear_src(t, vp);
    fi = __dsub_rn(fi, __ddiv_rn(__dmul_rn(vs, cfl_y), dn));
    fj = __dsub_rn(fj, __ddiv_rn(__dmul_rn(us, cfl_x), dn));
    if (fi < 0.0) fi = 0.0;
    else if (fi > (double)(H - 1)) fi = (double)(H - 1);
    if (fj < 0.0) fj = 0.0;
    else if (fj > (double)(W - 1)) fj = (double)(W - 1);
  }
  *oi = fi;
  *oj = fj;
}

template <typename I>
__device__ __forceinline__ void sl_departure(const I* up, const I* vp, int H,
                                             int W, int i, int j,
                                             double cfl_x, double cfl_y,
                                             double d_max, int n_max,
                                             double* oi, double* oj) {
  sl_departure_src(IntSrc<I>{up}, IntSrc<I>{vp}, H, W, i, j, cfl_x, cfl_y,
                   d_max, n_max, oi, oj, W);
}

// Packed MSB-first bit (np.packbits) n of a byte stream viewed as u32 words.
__device__ __forceinline__ void set_packbit(uint32_t* words, int64_t n) {
  int64_t byte = n >> 3;
  uint32_t bit = 7u - (uint32_t)(n & 7);
  atomicOr(words + (byte >> 2), 1u << (8u * (uint32_t)(byte & 3) + bit));
}

__device__ __forceinline__ int get_packbit(const uint8_t* bytes, int64_t n) {
  return (bytes[n >> 3] >> (7 - (n & 7))) & 1;
}

}  // namespace vfcp
