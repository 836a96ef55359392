// Exact face predicate (fixed-point, simulation of simplicity) and the exact
// L-infinity face error bound, device side.
//
// Restates predicates.py:156-287 (_sos_sign, _face_cp_sos, _face_scan) and
// ebounds.py:101-148 (_edge_eb, _eb_one) for |values| < 2^30, where every
// product fits int64 exactly.
#pragma once

#include "common.cuh"

namespace vfcp {

// predicates.py:156-254: sign of the homogeneous 3x3 orientation determinant
// under SoS (ids distinct; the origin carries id -1).
__device__ __noinline__ int sos_sign(int64_t x0, int64_t y0, int64_t x1,
                                     int64_t y1, int64_t x2, int64_t y2,
                                     int64_t id0, int64_t id1, int64_t id2) {
  int64_t det = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
  if (det > 0) return 1;
  if (det < 0) return -1;
  int64_t id[3] = {id0, id1, id2}, xs[3] = {x0, x1, x2}, ys[3] = {y0, y1, y2};
  int parity = 1;
#pragma unroll
  for (int i = 1; i < 3; i++) {
    for (int k = i; k > 0 && id[k - 1] > id[k]; k--) {
      int64_t t = id[k - 1]; id[k - 1] = id[k]; id[k] = t;
      t = xs[k - 1]; xs[k - 1] = xs[k]; xs[k] = t;
      t = ys[k - 1]; ys[k - 1] = ys[k]; ys[k] = t;
      parity = -parity;
    }
  }
  // lexicographically smallest descending key (2*id + choice, padded with
  // -2^62) among the 26 perturbation terms with a non-zero coefficient
  const int64_t PAD = -(((int64_t)1) << 62);
  int64_t b0 = ((int64_t)1) << 62, b1 = 0, b2 = 0, bc = 0;
  for (int code = 1; code < 27; code++) {
    int ch[3] = {code % 3 - 1, (code / 3) % 3 - 1, code / 9 - 1};
    int64_t r[3][3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
      if (ch[q] == -1) { r[q][0] = xs[q]; r[q][1] = ys[q]; r[q][2] = 1; }
      else if (ch[q] == 0) { r[q][0] = 1; r[q][1] = 0; r[q][2] = 0; }
      else { r[q][0] = 0; r[q][1] = 1; r[q][2] = 0; }
    }
    int64_t coeff = r[0][0] * (r[1][1] * r[2][2] - r[1][2] * r[2][1]) -
                    r[0][1] * (r[1][0] * r[2][2] - r[1][2] * r[2][0]) +
                    r[0][2] * (r[1][0] * r[2][1] - r[1][1] * r[2][0]);
    if (coeff == 0) continue;
    int64_t k0 = PAD, k1 = PAD, k2 = PAD;
    int nf = 0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
      if (ch[q] == -1) continue;
      int64_t f = 2 * id[q] + ch[q];
      if (nf == 0) k0 = f; else if (nf == 1) k1 = f; else k2 = f;
      nf++;
    }
    int64_t t;
    if (k1 > k0) { t = k0; k0 = k1; k1 = t; }
    if (k2 > k1) { t = k1; k1 = k2; k2 = t; }
    if (k1 > k0) { t = k0; k0 = k1; k1 = t; }
    bool smaller = (k0 < b0) || (k0 == b0 && k1 < b1) ||
                   (k0 == b0 && k1 == b1 && k2 < b2);
    if (smaller) { b0 = k0; b1 = k1; b2 = k2; bc = coeff; }
  }
  return bc > 0 ? parity : -parity;
}

// predicates.py:257-267 _face_cp_sos.
__device__ __noinline__ bool face_cp_sos(int64_t ua, int64_t va, int64_t ub,
                                         int64_t vb, int64_t uc, int64_t vc,
                                         int64_t ida, int64_t idb,
                                         int64_t idc) {
  int s = sos_sign(ua, va, ub, vb, uc, vc, ida, idb, idc);
  if (sos_sign(0, 0, ub, vb, uc, vc, -1, idb, idc) != s) return false;
  if (sos_sign(ua, va, 0, 0, uc, vc, ida, -1, idc) != s) return false;
  if (sos_sign(ua, va, ub, vb, 0, 0, ida, idb, -1) != s) return false;
  return true;
}

// predicates.py:278-287: positive iff the origin is inside the value triangle.
__device__ __forceinline__ bool face_positive(int64_t ua, int64_t va,
                                              int64_t ub, int64_t vb,
                                              int64_t uc, int64_t vc,
                                              int64_t a, int64_t b,
                                              int64_t c) {
  int64_t d1 = ua * vb - va * ub;
  int64_t d2 = ub * vc - vb * uc;
  int64_t d3 = uc * va - vc * ua;
  if (d1 != 0 && d2 != 0 && d3 != 0)
    return (d1 > 0 && d2 > 0 && d3 > 0) || (d1 < 0 && d2 < 0 && d3 < 0);
  return face_cp_sos(ua, va, ub, vb, uc, vc, a, b, c);
}

__device__ __forceinline__ int64_t floordiv_pos(int64_t a, int64_t d) {
  int64_t q = a / d;
  if ((a % d != 0) && (a < 0)) q--;
  return q;
}

// ebounds.py:101-134 _edge_eb: largest integer strictly below the exact
// L-inf distance from the origin to the segment p-q.
__device__ __noinline__ int64_t edge_eb(int64_t px, int64_t py, int64_t qx,
                                       int64_t qy) {
  int64_t dx = qx - px, dy = qy - py;
  int64_t best = max(llabs(px), llabs(py)) - 1;
  int64_t e1 = max(llabs(qx), llabs(qy)) - 1;
  if (e1 < best) best = e1;
#pragma unroll
  for (int which = 0; which < 4; which++) {
    int64_t n, d;
    if (which == 0) { if (dx == 0) continue; n = -px; d = dx; }
    else if (which == 1) { if (dy == 0) continue; n = -py; d = dy; }
    else if (which == 2) { if (dx == dy) continue; n = py - px; d = dx - dy; }
    else { if (dx + dy == 0) continue; n = -(px + py); d = dx + dy; }
    if (d < 0) { n = -n; d = -d; }
    if (0 <= n && n <= d) {
      int64_t a = max(llabs(px * d + n * dx), llabs(py * d + n * dy));
      int64_t e = floordiv_pos(a - 1, d);
      if (e < best) best = e;
    }
  }
  return best;
}

// codec.py:80-90 quantize_eb for 0 < xi < tau (the other cases are handled
// by the callers): k = bitlen(ceil(tau/xi) - 1), code 31 past the ladder.
__device__ __forceinline__ int ladder_code(int64_t xi, int64_t tau) {
  int64_t m = (tau + xi - 1) / xi;
  int k = 64 - __clzll((unsigned long long)(m - 1));
  if (k > K_MAX || (tau >> k) == 0) return CODE_LOSSLESS;
  return k;
}

// Vertex "value" of a bound: 0..31 = its ladder code, 32 = xi == 0 (l_d).
// quantize_eb is monotone non-increasing in xi, so the code of the
// per-vertex minimum is the maximum of these values.
__device__ __forceinline__ int eb_value(int64_t xi, int64_t tau) {
  if (xi <= 0) return 32;
  if (xi >= tau) return 0;
  return ladder_code(xi, tau);
}

}  // namespace vfcp
