// Host-side value range of a field that still lives in (pinned) host memory:
// min / max / max |x| over u and v (field.py:69-73 value_range, 300-310
// choose_scale's max_abs), reduced by a few threads at memory bandwidth while
// the same bytes cross PCIe.  The reference's global scale S and a relative
// eps need these three numbers before any vertex can be converted to fixed
// point, so a compress() of host data can only overlap its H2D copy with
// device work if they are known early.  The caller (codec.py
// _compress_streamed) hands this function the frames from the back of the
// field, which the DMA delivers last, while the device range kernel
// (analyze.cu range_kernel) reduces the frames that have arrived; the result
// is a *hint*: the device ends up reducing every frame and the caller
// compares the two.
//
// Minima and maxima of finite values are exact in any order; FieldSeries has
// already rejected NaN / Inf (field.py:37-51), so the comparisons need no
// NaN handling.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#define VFCP_X86 1
#endif

#include "../../include/vfcp_b200.h"

// capi.cu: sets the message vfcp_last_error() returns
int vfcp_record_error(int code, const char* msg);

namespace {

template <typename F>
void range_span(const F* __restrict__ x, int64_t n, double* out3) {
  // eight independent lanes so the compiler keeps the loop in vector
  // registers (-O2 vectorises min / max of this shape with the ?: form)
  constexpr int L = 16;
  F lo[L], hi[L];
  for (int k = 0; k < L; k++) { lo[k] = x[0]; hi[k] = x[0]; }
  int64_t i = 0;
  for (; i + L <= n; i += L) {
#pragma GCC unroll 16
    for (int k = 0; k < L; k++) {
      const F a = x[i + k];
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = a > hi[k] ? a : hi[k];
    }
  }
  F l = lo[0], h = hi[0];
  for (int k = 1; k < L; k++) {
    l = lo[k] < l ? lo[k] : l;
    h = hi[k] > h ? hi[k] : h;
  }
  for (; i < n; i++) {
    l = x[i] < l ? x[i] : l;
    h = x[i] > h ? x[i] : h;
  }
  out3[0] = (double)l;
  out3[1] = (double)h;
  out3[2] = std::fmax(std::fabs((double)l), std::fabs((double)h));
}

#ifdef VFCP_X86
// AVX2 forms (chosen at run time): four independent accumulators per bound
// keep the loads back to back; vminps / vmaxps on finite values are exact.
__attribute__((target("avx2"))) void range_span_avx2(const float* x, int64_t n,
                                                     double* out3) {
  __m256 lo[4], hi[4];
  for (int k = 0; k < 4; k++) lo[k] = hi[k] = _mm256_set1_ps(x[0]);
  int64_t i = 0;
  for (; i + 32 <= n; i += 32) {
    for (int k = 0; k < 4; k++) {
      const __m256 a = _mm256_loadu_ps(x + i + 8 * k);
      lo[k] = _mm256_min_ps(lo[k], a);
      hi[k] = _mm256_max_ps(hi[k], a);
    }
  }
  lo[0] = _mm256_min_ps(_mm256_min_ps(lo[0], lo[1]), _mm256_min_ps(lo[2], lo[3]));
  hi[0] = _mm256_max_ps(_mm256_max_ps(hi[0], hi[1]), _mm256_max_ps(hi[2], hi[3]));
  float l8[8], h8[8];
  _mm256_storeu_ps(l8, lo[0]);
  _mm256_storeu_ps(h8, hi[0]);
  float l = l8[0], h = h8[0];
  for (int k = 1; k < 8; k++) {
    l = l8[k] < l ? l8[k] : l;
    h = h8[k] > h ? h8[k] : h;
  }
  for (; i < n; i++) {
    l = x[i] < l ? x[i] : l;
    h = x[i] > h ? x[i] : h;
  }
  out3[0] = (double)l;
  out3[1] = (double)h;
  out3[2] = std::fmax(std::fabs((double)l), std::fabs((double)h));
}

__attribute__((target("avx2"))) void range_span_avx2(const double* x, int64_t n,
                                                     double* out3) {
  __m256d lo[4], hi[4];
  for (int k = 0; k < 4; k++) lo[k] = hi[k] = _mm256_set1_pd(x[0]);
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    for (int k = 0; k < 4; k++) {
      const __m256d a = _mm256_loadu_pd(x + i + 4 * k);
      lo[k] = _mm256_min_pd(lo[k], a);
      hi[k] = _mm256_max_pd(hi[k], a);
    }
  }
  lo[0] = _mm256_min_pd(_mm256_min_pd(lo[0], lo[1]), _mm256_min_pd(lo[2], lo[3]));
  hi[0] = _mm256_max_pd(_mm256_max_pd(hi[0], hi[1]), _mm256_max_pd(hi[2], hi[3]));
  double l4[4], h4[4];
  _mm256_storeu_pd(l4, lo[0]);
  _mm256_storeu_pd(h4, hi[0]);
  double l = l4[0], h = h4[0];
  for (int k = 1; k < 4; k++) {
    l = l4[k] < l ? l4[k] : l;
    h = h4[k] > h ? h4[k] : h;
  }
  for (; i < n; i++) {
    l = x[i] < l ? x[i] : l;
    h = x[i] > h ? x[i] : h;
  }
  out3[0] = l;
  out3[1] = h;
  out3[2] = std::fmax(std::fabs(l), std::fabs(h));
}
#endif

template <typename F>
void range_any(const F* x, int64_t n, double* out3, bool avx2) {
#ifdef VFCP_X86
  if (avx2) return range_span_avx2(x, n, out3);
#endif
  (void)avx2;
  range_span(x, n, out3);
}

template <typename F>
void host_range(const F* u, const F* v, int64_t n, int nthreads, double* out3) {
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, n / (1 << 16) + 1));
  // spans in frame order: thread k takes chunk k, k + nt, ... of each
  // component, so the early chunks (the first to cross PCIe) are read first
  const int64_t chunk = 1 << 20;
  const int64_t nchunks = (n + chunk - 1) / chunk;
#ifdef VFCP_X86
  const bool avx2 = __builtin_cpu_supports("avx2");
#else
  const bool avx2 = false;
#endif
  std::vector<double> part((size_t)nt * 3);
  std::vector<std::thread> th;
  auto work = [&](int k) {
    double lo = INFINITY, hi = -INFINITY, ma = 0.0;
    for (int64_t c = k; c < nchunks; c += nt) {
      const int64_t a = c * chunk, len = std::min(chunk, n - a);
      double r[3];
      range_any(u + a, len, r, avx2);
      lo = std::fmin(lo, r[0]); hi = std::fmax(hi, r[1]); ma = std::fmax(ma, r[2]);
      range_any(v + a, len, r, avx2);
      lo = std::fmin(lo, r[0]); hi = std::fmax(hi, r[1]); ma = std::fmax(ma, r[2]);
    }
    part[3 * k] = lo; part[3 * k + 1] = hi; part[3 * k + 2] = ma;
  };
  for (int k = 1; k < nt; k++) th.emplace_back(work, k);
  work(0);
  for (auto& t : th) t.join();
  double lo = INFINITY, hi = -INFINITY, ma = 0.0;
  for (int k = 0; k < nt; k++) {
    lo = std::fmin(lo, part[3 * k]);
    hi = std::fmax(hi, part[3 * k + 1]);
    ma = std::fmax(ma, part[3 * k + 2]);
  }
  out3[0] = lo; out3[1] = hi; out3[2] = ma;
}

}  // namespace

extern "C" int vfcp_host_range(const void* u, const void* v, int dtype,
                               int64_t n, int nthreads, double* out3) {
  if (n <= 0 || !u || !v || !out3)
    return vfcp_record_error(VFCP_EINVAL, "vfcp_host_range: empty field");
  if (dtype == VFCP_F32)
    host_range((const float*)u, (const float*)v, n, nthreads, out3);
  else if (dtype == VFCP_F64)
    host_range((const double*)u, (const double*)v, n, nthreads, out3);
  else
    return vfcp_record_error(VFCP_EINVAL, "vfcp_host_range: unknown dtype");
  return VFCP_OK;
}
