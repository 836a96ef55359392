// K0 value-range reduction and K1 fused critical-face / error-bound analysis.
//
// K1 replaces, in one pass over the input, the reference's
//   field.to_fixed conversion          field.py:313-336
//   build_critical_face_set            predicates.py:270-301
//   derive_all (+ _eb_scan/_edge_eb)   ebounds.py:101-206
//   _quantize_eb_vec                   codec.py:97-115
// A CTA owns a TI x TJ spatial tile and marches through time keeping frames
// t and t+1 (with a one-vertex halo) in shared memory.  Faces are enumerated
// implicitly per anchor vertex (12 classes, mesh.py:91-128).  Only the
// per-vertex eb *code* leaves the kernel (plus l_d bits and, optionally, a
// 12-bit positive-face mask per anchor); xi itself is never stored: since
// quantize_eb is monotone non-increasing in xi, code(min over faces) equals
// max over faces of code(face bound), which is reduced with shared-memory
// atomicMax.  A vertex class byte (|u|,|v| >= tau'+1 with a sign, and strict
// signs) lets whole space-time cubes skip the exact integer work:
// such faces can neither be positive nor lower xi below tau'.
#include <cub/cub.cuh>

#include "predicates.cuh"

namespace vfcp {

// ---------------------------------------------------------------- K0
// min / max / max |.| over u and v (field.py:69-73, 300-310).  Element
// minima and maxima are exact in the input precision; binary32 input is
// read as 16-byte vectors, four in flight per thread.
__device__ __forceinline__ void range_acc(float x, float& lo, float& hi,
                                          float& ma) {
  lo = fminf(lo, x);
  hi = fmaxf(hi, x);
  ma = fmaxf(ma, fabsf(x));
}
__device__ __forceinline__ void range_acc(double x, double& lo, double& hi,
                                          double& ma) {
  lo = fmin(lo, x);
  hi = fmax(hi, x);
  ma = fmax(ma, fabs(x));
}

template <typename F>
__global__ void __launch_bounds__(256) range_kernel(const F* __restrict__ u,
                                                    const F* __restrict__ v,
                                                    int64_t n,
                                                    double* __restrict__ part) {
  F lo = F(INFINITY), hi = F(-INFINITY), ma = F(0);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int c = 0; c < 2; c++) {
    const F* p = c ? v : u;
    int64_t head = 0;
    if (sizeof(F) == 4 && ((uintptr_t)p & 15) == 0) {
      const float4* p4 = reinterpret_cast<const float4*>(p);
      const int64_t n4 = n / 4;
      constexpr int U = 4;
      int64_t k = tid;
      for (; k + (U - 1) * stride < n4; k += U * stride) {
        float4 q[U];
#pragma unroll
        for (int e = 0; e < U; e++) q[e] = __ldg(p4 + k + e * stride);
#pragma unroll
        for (int e = 0; e < U; e++) {
          range_acc((F)q[e].x, lo, hi, ma);
          range_acc((F)q[e].y, lo, hi, ma);
          range_acc((F)q[e].z, lo, hi, ma);
          range_acc((F)q[e].w, lo, hi, ma);
        }
      }
      for (; k < n4; k += stride) {
        const float4 q = __ldg(p4 + k);
        range_acc((F)q.x, lo, hi, ma);
        range_acc((F)q.y, lo, hi, ma);
        range_acc((F)q.z, lo, hi, ma);
        range_acc((F)q.w, lo, hi, ma);
      }
      head = 4 * n4;
    }
    for (int64_t k = head + tid; k < n; k += stride) range_acc(__ldg(p + k), lo, hi, ma);
  }
  double dlo = (double)lo, dhi = (double)hi, dma = (double)ma;
  for (int o = 16; o; o >>= 1) {
    dlo = fmin(dlo, __shfl_xor_sync(0xffffffffu, dlo, o));
    dhi = fmax(dhi, __shfl_xor_sync(0xffffffffu, dhi, o));
    dma = fmax(dma, __shfl_xor_sync(0xffffffffu, dma, o));
  }
  __shared__ double s[3][8];
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s[0][w] = dlo; s[1][w] = dhi; s[2][w] = dma; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); q++) {
      dlo = fmin(dlo, s[0][q]); dhi = fmax(dhi, s[1][q]); dma = fmax(dma, s[2][q]);
    }
    part[3 * blockIdx.x + 0] = dlo;
    part[3 * blockIdx.x + 1] = dhi;
    part[3 * blockIdx.x + 2] = dma;
  }
}

// ---------------------------------------------------------------- K1
constexpr int TI = 32;             // owned rows per tile
constexpr int TJ = 64;             // owned columns per tile
constexpr int RH = TI + 2;         // region rows (1-vertex halo)
constexpr int RW = TJ + 2;         // region columns
constexpr int NA = (TI + 1) * (TJ + 1);  // anchors touching owned vertices
constexpr int K1_THREADS = 256;

// face classes (mesh.py:100-128): vertex offsets (dt, di, dj) of a < b < c
__constant__ int8_t c_off[12][3][3] = {
    {{0, 0, 0}, {0, 1, 0}, {0, 1, 1}},  // slice_lower
    {{0, 0, 0}, {0, 0, 1}, {0, 1, 1}},  // slice_upper
    {{0, 0, 0}, {0, 0, 1}, {1, 0, 1}},  // wall_h1
    {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}},  // wall_h2
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 0}},  // wall_v1
    {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}},  // wall_v2
    {{0, 0, 0}, {0, 1, 1}, {1, 1, 1}},  // wall_d1
    {{0, 0, 0}, {1, 0, 0}, {1, 1, 1}},  // wall_d2
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 1}},  // int_lower_a
    {{0, 0, 0}, {1, 1, 0}, {1, 1, 1}},  // int_lower_b
    {{0, 0, 0}, {0, 0, 1}, {1, 1, 1}},  // int_upper_a
    {{0, 0, 0}, {1, 0, 1}, {1, 1, 1}},  // int_upper_b
};
// anchor range: t < T - lim_t, i < H - lim_i, j < W - lim_j
__constant__ int8_t c_lim[12][3] = {
    {0, 1, 1}, {0, 1, 1}, {1, 0, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 0},
    {1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {1, 1, 1}};

struct K1Smem {
  int32_t u[2][RH][RW];
  int32_t v[2][RH][RW];
  uint8_t cls[2][RH][RW];    // low nibble: |.|>=tau'+1 by sign; high: strict sign
  int32_t acc[2][TI][TJ];    // max eb value (0..32) per owned vertex
  uint16_t mask[TI][TJ];     // positive-face classes per owned anchor
  uint16_t list[NA];         // anchors that need exact work
  int nlist;
};

__device__ __forceinline__ uint8_t vertex_class(int32_t x, int32_t y,
                                                int64_t thr) {
  uint8_t c = 0;
  if (x >= thr) c |= 1;
  if (-(int64_t)x >= thr) c |= 2;
  if (y >= thr) c |= 4;
  if (-(int64_t)y >= thr) c |= 8;
  if (x > 0) c |= 16;
  if (x < 0) c |= 32;
  if (y > 0) c |= 64;
  if (y < 0) c |= 128;
  return c;
}

template <typename F>
__global__ void __launch_bounds__(K1_THREADS)
analyze_kernel(const F* __restrict__ u, const F* __restrict__ v, int H, int W,
               int T, double S, int64_t tau, uint8_t* __restrict__ codes,
               uint32_t* __restrict__ ld_words, uint16_t* __restrict__ mask,
               int32_t* __restrict__ row_n31, const int* __restrict__ run_if) {
  // the fallback of the split analysis (below) when its anchor list
  // overflowed; run_if == nullptr: always
  if (run_if && *run_if == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K1Smem& sm = *reinterpret_cast<K1Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int i0 = blockIdx.y * TI, j0 = blockIdx.x * TJ;
  const int64_t HW = (int64_t)H * W;
  const int64_t thr = tau + 1;

  for (int k = tid; k < 2 * TI * TJ; k += K1_THREADS)
    (&sm.acc[0][0][0])[k] = 0;
  for (int k = tid; k < TI * TJ; k += K1_THREADS) (&sm.mask[0][0])[k] = 0;

  // Frame loads are software-pipelined: the raw values of frame t+2 are in
  // flight (registers) while slab (t, t+1) is processed, and converted into
  // shared memory at the start of the next iteration.
  constexpr int NL = (RH * RW + K1_THREADS - 1) / K1_THREADS;
  F ru[NL], rv[NL];
  auto issue = [&](int t) {
    const int64_t base = (int64_t)t * HW;
#pragma unroll
    for (int q = 0; q < NL; q++) {
      const int k = tid + q * K1_THREADS;
      const int lr = k / RW, lc = k - lr * RW;
      const int gi = i0 - 1 + lr, gj = j0 - 1 + lc;
      const bool ok = k < RH * RW && gi >= 0 && gi < H && gj >= 0 && gj < W;
      const int64_t n = ok ? base + (int64_t)gi * W + gj : 0;
      ru[q] = ok ? __ldg(u + n) : F(0);
      rv[q] = ok ? __ldg(v + n) : F(0);
    }
  };
  auto commit = [&](int t) {
    const int s = t & 1;
#pragma unroll
    for (int q = 0; q < NL; q++) {
      const int k = tid + q * K1_THREADS;
      if (k >= RH * RW) break;
      const int lr = k / RW, lc = k - lr * RW;
      const int gi = i0 - 1 + lr, gj = j0 - 1 + lc;
      int32_t x = 0, y = 0;
      uint8_t c = 0;
      if (gi >= 0 && gi < H && gj >= 0 && gj < W) {
        x = fixed_t(ru[q], S);
        y = fixed_t(rv[q], S);
        c = vertex_class(x, y, thr);
      }
      sm.u[s][lr][lc] = x;
      sm.v[s][lr][lc] = y;
      sm.cls[s][lr][lc] = c;
    }
  };

  issue(0);
  commit(0);
  if (T > 1) issue(1);
  for (int t = 0; t < T; t++) {
    const bool slab = t + 1 < T;
    if (slab) commit(t + 1);
    if (t + 2 < T) issue(t + 2);
    if (tid == 0) sm.nlist = 0;
    __syncthreads();

    // -- 1. cube test per anchor; compact the anchors needing exact work
    const int s0 = t & 1, s1 = (t + 1) & 1;
    for (int k = tid; k < NA; k += K1_THREADS) {
      int lr = k / (TJ + 1), lc = k - lr * (TJ + 1);
      int gi = i0 - 1 + lr, gj = j0 - 1 + lc;
      if (gi < 0 || gj < 0 || gi >= H || gj >= W) continue;
      // vertices that exist around the anchor (edges of the grid clip)
      int r1 = gi + 1 < H ? lr + 1 : lr, c1 = gj + 1 < W ? lc + 1 : lc;
      uint8_t a = sm.cls[s0][lr][lc] & sm.cls[s0][lr][c1] &
                  sm.cls[s0][r1][lc] & sm.cls[s0][r1][c1];
      if (slab)
        a &= sm.cls[s1][lr][lc] & sm.cls[s1][lr][c1] & sm.cls[s1][r1][lc] &
             sm.cls[s1][r1][c1];
      if ((a & 0x0F) == 0) {
        int p = atomicAdd(&sm.nlist, 1);
        sm.list[p] = (uint16_t)k;
      }
    }
    __syncthreads();

    // -- 2. exact predicate + bound for every (anchor, class) on the list
    const int nitems = sm.nlist * 12;
    for (int w = tid; w < nitems; w += K1_THREADS) {
      int k = sm.list[w / 12], c = w % 12;
      int lr = k / (TJ + 1), lc = k - lr * (TJ + 1);
      int gi = i0 - 1 + lr, gj = j0 - 1 + lc;
      if (t >= T - c_lim[c][0] || gi >= H - c_lim[c][1] ||
          gj >= W - c_lim[c][2])
        continue;
      int vs[3], vr[3], vc[3];
      int64_t id[3], X[3], Y[3];
      uint8_t cl[3];
#pragma unroll
      for (int q = 0; q < 3; q++) {
        int dt = c_off[c][q][0], di = c_off[c][q][1], dj = c_off[c][q][2];
        vs[q] = (t + dt) & 1;
        vr[q] = lr + di;
        vc[q] = lc + dj;
        X[q] = sm.u[vs[q]][vr[q]][vc[q]];
        Y[q] = sm.v[vs[q]][vr[q]][vc[q]];
        cl[q] = sm.cls[vs[q]][vr[q]][vc[q]];
        id[q] = (int64_t)(t + dt) * HW + (int64_t)(gi + di) * W + (gj + dj);
      }
      uint8_t fa = cl[0] & cl[1] & cl[2];
      if (fa & 0x0F) continue;  // neither positive nor below tau'
      bool pos = false;
      if ((fa & 0xF0) == 0)
        pos = face_positive(X[0], Y[0], X[1], Y[1], X[2], Y[2], id[0], id[1],
                            id[2]);
      int val;
      if (pos) {
        val = 32;
        if (mask && lr >= 1 && lc >= 1)
          atomicOr((unsigned int*)&sm.mask[0][0] +
                       (((lr - 1) * TJ + (lc - 1)) >> 1),
                   (1u << c) << (16 * ((lc - 1) & 1)));
      } else {
        int64_t xi = tau;
#pragma unroll
        for (int q = 0; q < 3; q++) {
          int q2 = q == 2 ? 0 : q + 1;
          if ((cl[q] & cl[q2] & 0x0F) == 0) {
            int64_t e = edge_eb(X[q], Y[q], X[q2], Y[q2]);
            if (e < xi) xi = e;
          }
        }
        if (xi < 0) xi = 0;
        val = eb_value(xi, tau);
      }
      if (val == 0) continue;
#pragma unroll
      for (int q = 0; q < 3; q++) {
        int orr = vr[q] - 1, occ = vc[q] - 1;
        if (orr >= 0 && orr < TI && occ >= 0 && occ < TJ)
          atomicMax(&sm.acc[vs[q]][orr][occ], val);
      }
    }
    __syncthreads();

    // -- 3. frame t is final: emit codes, l_d bits, row counts, face mask
    {
      const int lc = tid & (TJ - 1);
      const int gj = j0 + lc;
      const int lane = tid & 31;
      for (int lr = tid / TJ; lr < TI; lr += K1_THREADS / TJ) {
        const int gi = i0 + lr;
        bool inb = gi < H && gj < W;
        int val = sm.acc[s0][lr][lc];
        if (tau <= 0) val = 32;
        int code = val > 31 ? 31 : val;
        if (inb) {
          int64_t n = (int64_t)t * HW + (int64_t)gi * W + gj;
          codes[n] = (uint8_t)code;
          if (val == 32) set_packbit(ld_words, n);
          if (mask) mask[n] = sm.mask[lr][lc];
        }
        unsigned b = __ballot_sync(0xffffffffu, inb && code == 31);
        if (lane == 0 && b && gi < H)
          atomicAdd(row_n31 + (int64_t)t * H + gi, __popc(b));
        sm.acc[s0][lr][lc] = 0;
        sm.mask[lr][lc] = 0;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------- K1, split in two
// The common case has almost no anchor whose space-time cube can carry a
// positive face or lower a bound below tau' (the vertex class
// test above).  So the analysis runs as
//   cube_kernel   streaming over the field once (8 B/vertex): fixed point,
//                 the vertex class, the cube test of every anchor; only the
//                 failing anchors are appended to a list (codes are 0 for
//                 everything else: set by a memset beforehand);
//   exact_kernel  the 12 faces of each listed anchor, exactly (SoS, int64
//                 edge bounds); the code of a vertex is the max over its
//                 faces' values (quantize_eb is monotone), applied with a
//                 byte atomicMax; l_d bits, the per-row code-31 counts (a
//                 vertex is counted when its byte first reaches 31) and the
//                 face mask likewise.
// A list that would overflow its buffer hands the frame set to the fused
// kernel above (analyze_kernel with run_if = the overflow flag).
constexpr int CTI = 32, CTJ = 128;           // owned anchors per tile
constexpr int CRH = CTI + 1;                 // vertex rows (+1 below)
constexpr int CQW = CTJ / 4 + 1;             // 4-vertex groups per row (+1 right)
constexpr int C_THREADS = 256;

// Low nibble of the vertex class (analyze_kernel's vertex_class) straight
// from the float input: fixed(x) >= thr <=> x*S >= thr - 0.5 (rha rounds
// half away from zero) <=> x >= T with T = (thr - 0.5) / S exact, i.e. x >=
// Tf for the smallest float Tf >= T (x is a float); -x likewise.  Vertices
// outside the frame get 0xFF, so a cube clipped at the frame edge (the
// reference's anchor ranges) ANDs only its existing vertices.
__device__ __forceinline__ uint32_t cls_nib(float x, float y, float Tf) {
  return (x >= Tf ? 1u : 0u) | (-x >= Tf ? 2u : 0u) | (y >= Tf ? 4u : 0u) |
         (-y >= Tf ? 8u : 0u);
}
__device__ __forceinline__ uint32_t cls_nib(double x, double y, double Td) {
  return (x >= Td ? 1u : 0u) | (-x >= Td ? 2u : 0u) | (y >= Td ? 4u : 0u) |
         (-y >= Td ? 8u : 0u);
}

// CTA = 32 x 128 anchors, marching over the frames with the class bytes of
// frames t and t+1 in shared memory (frame t+2's values in flight); a thread
// tests four anchors of one row at once (byte-SIMD AND of 32-bit words).
template <typename F>
__global__ void __launch_bounds__(C_THREADS, 4)
cube_kernel(const F* __restrict__ u, const F* __restrict__ v, int H, int W,
            int T, int t0, int t1, F Tq, uint64_t* __restrict__ list,
            unsigned long long* __restrict__ count, unsigned long long cap) {
  __shared__ uint32_t cls[2][CRH][CQW + 1];   // 4 class bytes per word
  const int tid = threadIdx.x, lane = tid & 31;
  const int i0 = blockIdx.y * CTI, j0 = blockIdx.x * CTJ;
  const int64_t HW = (int64_t)H * W;
  const bool vec = sizeof(F) == 4 && (W & 3) == 0 &&
                   (((uintptr_t)u | (uintptr_t)v) & 15) == 0;
  constexpr int NG = CRH * CQW;                           // groups per frame
  constexpr int NL = (NG + C_THREADS - 1) / C_THREADS;
  float4 ru[NL], rv[NL];
  auto issue = [&](int t) {
    const int64_t base = (int64_t)t * HW;
#pragma unroll
    for (int q = 0; q < NL; q++) {
      const int k = tid + q * C_THREADS;
      const int lr = k / CQW, g = k - lr * CQW;
      const int gi = i0 + lr, gj = j0 + 4 * g;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (k < NG && gi < H) {
        const int64_t n = base + (int64_t)gi * W + gj;
        if (vec && gj + 3 < W) {
          a = __ldg(reinterpret_cast<const float4*>(u + n));
          b = __ldg(reinterpret_cast<const float4*>(v + n));
        } else {
          float xa[4] = {0.f, 0.f, 0.f, 0.f}, xb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (gj + e < W) { xa[e] = (float)__ldg(u + n + e); xb[e] = (float)__ldg(v + n + e); }
          a = make_float4(xa[0], xa[1], xa[2], xa[3]);
          b = make_float4(xb[0], xb[1], xb[2], xb[3]);
          if (sizeof(F) == 8) {
            // float64 input: the class is taken in double below; keep the
            // raw values by reloading there (rare path)
          }
        }
      }
      ru[q] = a;
      rv[q] = b;
    }
  };
  auto commit = [&](int t) {
    const int s = t & 1;
    const int64_t base = (int64_t)t * HW;
#pragma unroll
    for (int q = 0; q < NL; q++) {
      const int k = tid + q * C_THREADS;
      if (k >= NG) break;
      const int lr = k / CQW, g = k - lr * CQW;
      const int gi = i0 + lr, gj = j0 + 4 * g;
      uint32_t w = 0;
      const float xs[4] = {ru[q].x, ru[q].y, ru[q].z, ru[q].w};
      const float ys[4] = {rv[q].x, rv[q].y, rv[q].z, rv[q].w};
      const bool inside = gi < H && gj + 3 < W;   // the usual group
#pragma unroll
      for (int e = 0; e < 4; e++) {
        uint32_t c = 0xffu;
        if (inside || (gi < H && gj + e < W)) {
          if (sizeof(F) == 4) {
            c = cls_nib(xs[e], ys[e], (float)Tq);
          } else {
            const int64_t n = base + (int64_t)gi * W + gj + e;
            c = cls_nib((double)__ldg(u + n), (double)__ldg(v + n), (double)Tq);
          }
        }
        w |= c << (8 * e);
      }
      cls[s][lr][g] = w;
    }
  };
  // anchors of frames [t0, t1): reads frames t0 .. min(t1, T - 1)
  issue(t0);
  commit(t0);
  if (t0 + 1 < T) issue(t0 + 1);
  const unsigned FULL = 0xffffffffu;
  for (int t = t0; t < t1; t++) {
    const bool slab = t + 1 < T;
    if (slab) commit(t + 1);
    if (t + 2 < T && t + 1 < t1) issue(t + 2);
    __syncthreads();
    const int s0 = t & 1, s1 = (t + 1) & 1;
    // thread: row lr, anchors 4g .. 4g+3 (CTJ / 4 = 32 groups per row)
    const int g = tid & 31;
#pragma unroll
    for (int lr = tid >> 5; lr < CTI; lr += C_THREADS / 32) {
      const int gi = i0 + lr;
      auto band = [&](int s, int r) {
        const uint32_t w0 = cls[s][r][g], w1 = cls[s][r][g + 1];
        return w0 & __funnelshift_r(w0, w1, 8);   // (c, c+1) pairs
      };
      uint32_t a = band(s0, lr) & band(s0, lr + 1);
      if (slab) a &= band(s1, lr) & band(s1, lr + 1);
      // anchor e needs exact work iff its nibble AND is 0 (and it exists)
      uint32_t need = __vcmpeq4(a & 0x0f0f0f0fu, 0u);   // 0xff per byte
      uint32_t m4 = 0;
#pragma unroll
      for (int e = 0; e < 4; e++)
        if (((need >> (8 * e)) & 1u) && gi < H && j0 + 4 * g + e < W) m4 |= 1u << e;
      const int n = __popc(m4);
      // (almost every row of 128 anchors lists nothing: one vote instead of
      // the scan)
      if (!__any_sync(FULL, n != 0)) continue;
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(FULL, incl, 31);
      if (tot) {
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(count, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 31);
        unsigned long long k = base + (incl - n);
        while (m4) {
          const int e = __ffs(m4) - 1;
          m4 &= m4 - 1u;
          if (k < cap)
            list[k] = ((uint64_t)t << 48) | ((uint64_t)gi << 24) |
                      (uint64_t)(j0 + 4 * g + e);
          k++;
        }
      }
    }
    __syncthreads();
  }
}

// byte-wise atomic max on a byte array; returns the previous byte
__device__ __forceinline__ unsigned atomic_max_u8(uint8_t* a, int64_t k,
                                                  unsigned val) {
  unsigned int* w = reinterpret_cast<unsigned int*>(
      reinterpret_cast<uintptr_t>(a + k) & ~(uintptr_t)3);
  const unsigned sh = 8u * (unsigned)(reinterpret_cast<uintptr_t>(a + k) & 3);
  unsigned old = *reinterpret_cast<volatile unsigned int*>(w);
  for (;;) {
    const unsigned ob = (old >> sh) & 0xffu;
    if (ob >= val) return ob;
    const unsigned nw = (old & ~(0xffu << sh)) | (val << sh);
    const unsigned prev = atomicCAS(w, old, nw);
    if (prev == old) return ob;
    old = prev;
  }
}

template <typename F>
__global__ void __launch_bounds__(128)
exact_kernel(const F* __restrict__ u, const F* __restrict__ v, int H, int W,
             int T, double S, int64_t tau, const uint64_t* __restrict__ list,
             const unsigned long long* __restrict__ count,
             unsigned long long cap, const int* __restrict__ skip_if,
             uint8_t* __restrict__ codes, uint32_t* __restrict__ ld_words,
             uint16_t* __restrict__ mask, int32_t* __restrict__ row_n31) {
  if (*skip_if) return;
  const unsigned long long n = min(*count, cap);
  const int64_t HW = (int64_t)H * W;
  const int64_t thr = tau + 1;
  for (unsigned long long k = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
       k < n; k += (unsigned long long)gridDim.x * blockDim.x) {
    const uint64_t e = list[k];
    const int t = (int)(e >> 48), gi = (int)((e >> 24) & 0xffffff), gj = (int)(e & 0xffffff);
    // the anchor's cube: q = dt * 4 + di * 2 + dj
    int64_t X[8], Y[8];
    uint8_t cl[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int dt = q >> 2, di = (q >> 1) & 1, dj = q & 1;
      const bool ok = t + dt < T && gi + di < H && gj + dj < W;
      const int64_t id = (int64_t)(t + dt) * HW + (int64_t)(gi + di) * W + gj + dj;
      const int32_t x = ok ? fixed_t(__ldg(u + id), S) : 0;
      const int32_t y = ok ? fixed_t(__ldg(v + id), S) : 0;
      X[q] = x;
      Y[q] = y;
      cl[q] = vertex_class(x, y, thr);
    }
    const int64_t an = (int64_t)t * HW + (int64_t)gi * W + gj;
    unsigned mbits = 0;
#pragma unroll 1
    for (int c = 0; c < 12; c++) {
      if (t >= T - c_lim[c][0] || gi >= H - c_lim[c][1] || gj >= W - c_lim[c][2])
        continue;
      int qv[3];
      int64_t id[3];
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const int dt = c_off[c][r][0], di = c_off[c][r][1], dj = c_off[c][r][2];
        qv[r] = dt * 4 + di * 2 + dj;
        id[r] = an + (int64_t)dt * HW + (int64_t)di * W + dj;
      }
      const uint8_t fa = cl[qv[0]] & cl[qv[1]] & cl[qv[2]];
      if (fa & 0x0F) continue;   // neither positive nor below tau'
      bool pos = false;
      if ((fa & 0xF0) == 0)
        pos = face_positive(X[qv[0]], Y[qv[0]], X[qv[1]], Y[qv[1]], X[qv[2]],
                            Y[qv[2]], id[0], id[1], id[2]);
      int val;
      if (pos) {
        val = 32;
        mbits |= 1u << c;
      } else {
        int64_t xi = tau;
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const int r2 = r == 2 ? 0 : r + 1;
          if ((cl[qv[r]] & cl[qv[r2]] & 0x0F) == 0) {
            const int64_t eb = edge_eb(X[qv[r]], Y[qv[r]], X[qv[r2]], Y[qv[r2]]);
            if (eb < xi) xi = eb;
          }
        }
        if (xi < 0) xi = 0;
        val = eb_value(xi, tau);
      }
      if (val == 0 || tau <= 0) continue;   // tau' <= 0: every code is 31
      const unsigned v31 = val > 31 ? 31u : (unsigned)val;
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const unsigned old = atomic_max_u8(codes, id[r], v31);
        if (val == 32) set_packbit(ld_words, id[r]);
        if (old < 31u && v31 == 31u) {
          const int64_t row = id[r] / W;   // t * H + i
          atomicAdd(row_n31 + row, 1);
        }
      }
    }
    if (mask && mbits)
      atomicOr(reinterpret_cast<unsigned int*>(mask) + (an >> 1),
               mbits << (16 * (unsigned)(an & 1)));
  }
}

__global__ void ovf_flag_kernel(const unsigned long long* count,
                                unsigned long long cap, int* ovf) {
  *ovf = *count > cap ? 1 : 0;
}

// the same for a slab of anchors: the flag of earlier slabs stays set
__global__ void ovf_or_kernel(const unsigned long long* count,
                              unsigned long long cap, int* ovf) {
  if (*count > cap) *ovf = 1;
}

// every vertex lossless (tau' <= 0): l_d all ones (packbits of N bits,
// zero padded), W code-31 vertices per row (the codes: a memset); skipped
// when the fused fallback runs
__global__ void lossless_fill_kernel(int64_t N, int64_t nrows, int W,
                                     uint8_t* __restrict__ ld_bytes,
                                     int32_t* __restrict__ row_n31,
                                     const int* __restrict__ skip_if) {
  if (*skip_if) return;
  const int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = k0; r < nrows; r += step) row_n31[r] = W;
  for (int64_t b = k0; b < (N >> 3); b += step) ld_bytes[b] = 0xff;
  if (k0 == 0 && (N & 7)) ld_bytes[N >> 3] = (uint8_t)(0xffu << (8 - (N & 7)));
}

// ------------------------------------------------- row offsets (exclusive)
// out[r] = base + sum_{q < r} mul * (W - cnt[q])   (qd symbol offsets), or
// out[r] = sum_{q < r} cnt[q] when W == 0 (plain exclusive scan).
// CTA b scans rows [1024 b, 1024 b + 1024): its carry-in is a coalesced
// block reduction over all earlier rows (at most T*H 4-byte loads per CTA,
// L2-resident), so the CTAs need no inter-CTA handoff.
constexpr int RS_T = 1024;
__device__ __forceinline__ int64_t row_term(const int32_t* cnt, int64_t r,
                                            int W, int mul) {
  return W ? (int64_t)mul * (W - __ldg(cnt + r)) : (int64_t)__ldg(cnt + r);
}
__global__ void __launch_bounds__(RS_T)
row_scan_kernel(const int32_t* __restrict__ cnt, int64_t nrows, int W,
                int mul, int64_t* __restrict__ out) {
  typedef cub::BlockReduce<int64_t, RS_T> BR;
  typedef cub::BlockScan<int64_t, RS_T> BS;
  __shared__ union {
    typename BR::TempStorage r;
    typename BS::TempStorage s;
  } tmp;
  __shared__ int64_t carry;
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * RS_T;
  int64_t acc = 0;
  int64_t r = tid;
  for (; r + 3 * RS_T < r0; r += 4 * RS_T)
    acc += row_term(cnt, r, W, mul) + row_term(cnt, r + RS_T, W, mul) +
           row_term(cnt, r + 2 * RS_T, W, mul) + row_term(cnt, r + 3 * RS_T, W, mul);
  for (; r < r0; r += RS_T) acc += row_term(cnt, r, W, mul);
  const int64_t pre = BR(tmp.r).Sum(acc);
  if (tid == 0) carry = pre;
  __syncthreads();
  const int64_t me = r0 + tid;
  const int64_t x = me < nrows ? row_term(cnt, me, W, mul) : 0;
  int64_t excl, tot;
  BS(tmp.s).ExclusiveSum(x, excl, tot);
  if (me < nrows) out[me] = carry + excl;
  if (r0 + RS_T >= nrows && tid == 0) out[nrows] = carry + tot;
}

// ------------------------------------------------------------ launchers
template <typename F>
cudaError_t launch_range(const F* u, const F* v, int64_t n, double* part,
                         int nblocks, cudaStream_t st) {
  range_kernel<F><<<nblocks, 256, 0, st>>>(u, v, n, part);
  return cudaGetLastError();
}

// ld_words and row_n31 zeroed by the caller; scratch: the anchor list
// (cap entries), its count and the overflow flag (zeroed here)
template <typename F>
cudaError_t launch_analyze(const F* u, const F* v, int H, int W, int T,
                           double S, int64_t tau, uint8_t* codes,
                           uint32_t* ld_words, uint16_t* mask,
                           int32_t* row_n31, uint64_t* list,
                           unsigned long long* count, int* ovf,
                           unsigned long long cap, int nsm, cudaStream_t st) {
  const int64_t N = (int64_t)H * W * T;
  cudaError_t e;
  if ((e = cudaMemsetAsync(codes, tau > 0 ? 0 : CODE_LOSSLESS, (size_t)N, st)) != cudaSuccess)
    return e;
  if (mask && (e = cudaMemsetAsync(mask, 0, sizeof(uint16_t) * (size_t)N, st)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), st)) != cudaSuccess) return e;
  // the class threshold in the input's own precision (cls_nib)
  const double Td = ((double)(tau + 1) - 0.5) / S;
  F Tq;
  if (sizeof(F) == 4) {
    float tf = (float)Td;
    if ((double)tf < Td) tf = nextafterf(tf, INFINITY);
    Tq = (F)tf;
  } else {
    Tq = (F)Td;
  }
  cube_kernel<F><<<dim3((W + CTJ - 1) / CTJ, (H + CTI - 1) / CTI), C_THREADS, 0, st>>>(
      u, v, H, W, T, 0, T, Tq, list, count, cap);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ovf_flag_kernel<<<1, 1, 0, st>>>(count, cap, ovf);
  exact_kernel<F><<<nsm * 8, 128, 0, st>>>(u, v, H, W, T, S, tau, list, count,
                                          cap, ovf, codes, ld_words, mask,
                                          row_n31);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (tau <= 0) {
    lossless_fill_kernel<<<1184, 256, 0, st>>>(N, (int64_t)T * H, W,
                                               reinterpret_cast<uint8_t*>(ld_words),
                                               row_n31, ovf);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // fallback: the fused kernel, which rewrites codes / l_d / counts / mask
  size_t smem = sizeof(K1Smem);
  e = cudaFuncSetAttribute(analyze_kernel<F>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + TJ - 1) / TJ, (H + TI - 1) / TI);
  analyze_kernel<F><<<grid, K1_THREADS, smem, st>>>(
      u, v, H, W, T, S, tau, codes, ld_words, mask, row_n31, ovf);
  return cudaGetLastError();
}

// The anchors of frames [t0, t1) only (they read frames t0 .. min(t1, T-1)):
// every update of codes / l_d / row counts / mask is an atomic max / or /
// first-touch count, so the slabs of a field may run in any partition and
// leave the same arrays as launch_analyze.  codes, ld_words, mask, row_n31
// and *ovf are zeroed by the caller before the first slab; a list overflow
// sets *ovf (the caller then redoes the field with launch_analyze).  tau > 0.
template <typename F>
cudaError_t launch_analyze_slab(const F* u, const F* v, int H, int W, int T,
                                int t0, int t1, double S, int64_t tau,
                                uint8_t* codes, uint32_t* ld_words,
                                uint16_t* mask, int32_t* row_n31,
                                uint64_t* list, unsigned long long* count,
                                int* ovf, unsigned long long cap, int nsm,
                                cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), st)) != cudaSuccess) return e;
  const double Td = ((double)(tau + 1) - 0.5) / S;
  F Tq;
  if (sizeof(F) == 4) {
    float tf = (float)Td;
    if ((double)tf < Td) tf = nextafterf(tf, INFINITY);
    Tq = (F)tf;
  } else {
    Tq = (F)Td;
  }
  cube_kernel<F><<<dim3((W + CTJ - 1) / CTJ, (H + CTI - 1) / CTI), C_THREADS, 0, st>>>(
      u, v, H, W, T, t0, t1, Tq, list, count, cap);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ovf_or_kernel<<<1, 1, 0, st>>>(count, cap, ovf);
  exact_kernel<F><<<nsm * 8, 128, 0, st>>>(u, v, H, W, T, S, tau, list, count,
                                          cap, ovf, codes, ld_words, mask,
                                          row_n31);
  return cudaGetLastError();
}

cudaError_t launch_row_scan(const int32_t* cnt, int64_t nrows, int W, int mul,
                            int64_t* out, cudaStream_t st) {
  const unsigned nb = (unsigned)((nrows + RS_T - 1) / RS_T);
  row_scan_kernel<<<nb ? nb : 1, RS_T, 0, st>>>(cnt, nrows, W, mul, out);
  return cudaGetLastError();
}

template cudaError_t launch_range<float>(const float*, const float*, int64_t,
                                         double*, int, cudaStream_t);
template cudaError_t launch_range<double>(const double*, const double*,
                                          int64_t, double*, int, cudaStream_t);
template cudaError_t launch_analyze<float>(const float*, const float*, int,
                                           int, int, double, int64_t,
                                           uint8_t*, uint32_t*, uint16_t*,
                                           int32_t*, uint64_t*,
                                           unsigned long long*, int*,
                                           unsigned long long, int,
                                           cudaStream_t);
template cudaError_t launch_analyze<double>(const double*, const double*, int,
                                            int, int, double, int64_t,
                                            uint8_t*, uint32_t*, uint16_t*,
                                            int32_t*, uint64_t*,
                                            unsigned long long*, int*,
                                            unsigned long long, int,
                                            cudaStream_t);

template cudaError_t launch_analyze_slab<float>(
    const float*, const float*, int, int, int, int, int, double, int64_t,
    uint8_t*, uint32_t*, uint16_t*, int32_t*, uint64_t*, unsigned long long*,
    int*, unsigned long long, int, cudaStream_t);
template cudaError_t launch_analyze_slab<double>(
    const double*, const double*, int, int, int, int, int, double, int64_t,
    uint8_t*, uint32_t*, uint16_t*, int32_t*, uint64_t*, unsigned long long*,
    int*, unsigned long long, int, cudaStream_t);

}  // namespace vfcp
