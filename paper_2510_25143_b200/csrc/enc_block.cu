// The encoder's per-block preparation of one frame: one CTA per 32x32 block
// does everything that does not depend on the raster recurrence, in one pass
// over the block's inputs (codec.py:118-164 _encode_frame, mop.py:68-151
// _score_frame):
//
//   * the tiles of orig(t) (fixed point) and recon(t-1) with a one-pixel halo
//     above and to the left (delta = orig - recon(t-1));
//   * R0 = orig - Lorenzo(orig, prev) = D(delta), the 2D difference of
//     delta, against the escape limits -- skipped when 4 max|delta| is below
//     them, which bounds every |R0|;
//   * the MoP mode (t >= 1): Lorenzo trial (two warps, rows streamed) and
//     semi-Lagrangian trial at the stride samples (the other two warps),
//     first-touch entropy rates, the theta gate;
//   * semi-Lagrangian blocks: every pixel's prediction (the trial's sample
//     predictions reused), symbol, recon(t) and the block's err edges;
//   * Lorenzo blocks: the class for the block scan (bscan.cuh) and its edge
//     data, or recon(t) = orig for all-lossless blocks, or the R0 plane for
//     the blocks the chain sweeps exactly.
//
// Why no prefix sums are needed.  In a block whose pixels share one step e
// (m = 2e), carry no pins and cannot escape, Z = recon - recon(t-1) satisfies
// D(Z) = q*m, so Z (mod m) is separable: Z(i,j) = Z(top, j) + Z(i, left) -
// Z(corner) (mod m).  With err = recon - orig = Z - delta that gives every
// error directly from the block boundary:
//   err(i, j) = rep(errT(j) + errL(i) - errC - Pd(i, j))  (mod m)
// where Pd(i, j) = delta(i,j) - delta(top,j) - delta(i,left) +
// delta(corner) is the telescoped 2D prefix sum of R0 and rep() the
// representative in [-e, e] (a residue of exactly e is a tie, decided by the
// sign of x = R0 - (errU + errL - errUL) in raster order).  The MoP Lorenzo
// trial is the same identity with zero boundary errors (the candidate frame
// is the original outside the block, mop.py:88-110).  The chain (bscan.cuh
// phase B) needs only the block's bottom row and right column of -Pd; the
// interior pass recomputes the rest from orig / recon(t-1) and the exact
// boundary.
//
// Exactness: |orig| < 2^30 and |recon| < 2^31, so delta fits int64 and its
// residues come from res_i64.  When every |delta| of the tile is below 2^29
// ("narrow", the normal case) R0 = D(delta) is computed in int32 (|R0| <
// 2^31); otherwise in int64.
#include "bscan.cuh"
#include "predict.cuh"

namespace vfcp {

struct EncBlockSmem {
  int32_t o[2][33][33];     // fixed orig(t), [comp][1+i][1+j], halo row/col 0
  int32_t d[2][33][33];     // delta = orig - recon(t-1) (wrapping int32)
  uint8_t cd[32][36];       // codes of the block (31 outside)
  int32_t spu[256], spv[256];   // SL trial predictions at the samples
  int16_t samp[2][512];     // |idx| per trial sample (-1: escape)
  int16_t order[2][ETB];
  alignas(16) int16_t cnt[2][ETB];
  double rate[2];
  int flag[8];              // see F_* below
  int32_t etab[32];         // e per code (tau' < 2^29 on this path)
};
enum {
  F_NONUNI = 0,   // a valid code differs from code0
  F_LOSSY = 1,    // some valid pixel has e > 0
  F_LOSSLESS = 2, // some valid pixel has e == 0
  F_MAXD = 3,     // max |delta| over the tile (clamped to 2^31 - 1)
  F_UNSAFE_T = 4, // bit c: comp c has |R0| >= lim(tau') (trial sweep)
  F_UNSAFE_0 = 5, // bit c: comp c has |R0| >= lim(e0)
  F_OVF = 6,      // some |R0| >= 2^31 - 1
  F_TIE = 7,      // the sample-parallel Lorenzo trial met a tie
};

// recon(t-1) of component c at delta-tile coordinates (rr, cc) (row 0 =
// r0 - 1, column 0 = c0 - 1)
struct PvTile {
  const int32_t (*o)[33][33];
  const int32_t (*d)[33][33];
  __device__ __forceinline__ int32_t at(int c, int rr, int cc) const {
    return (int32_t)((uint32_t)o[c][rr][cc] - (uint32_t)d[c][rr][cc]);
  }
};

// residue in [0, m) of delta = o - p: int32 when the tile is narrow
// (|delta| < 2^29), else int64 (|delta| < 2^32)
__device__ __forceinline__ uint32_t res_delta(int32_t d, uint32_t m, uint32_t M,
                                              uint32_t) {
  return bs_res_any(d, m, M);
}
__device__ __forceinline__ uint32_t res_delta(int64_t d, uint32_t m, uint32_t M,
                                              uint32_t c32) {
  return res_i64(d, m, M, c32);
}

// MoP Lorenzo trial of one component (mop.py:88-110): step tau' everywhere,
// zero error boundary, rows streamed (lane = column):
//   err'(i, j) = rep(dT(j) + dL(i) - dC - d(i, j))  (mod m)
// with D(err') and R0 from the row above (registers) and the left
// neighbour (shuffles); ties in raster order.  |idx| = |R0 + D(err')| / m at
// the stride samples (STRIDE: 2, or 0 for the runtime stride).
template <typename I, int STRIDE>
__device__ __forceinline__ void trial_rows(const int32_t (*o)[33],
                                           PvTile pp, int nr,
                                           int ncl, int stride, int nsx,
                                           int32_t e, uint32_t m, uint32_t M,
                                           uint32_t c32, int16_t* samp,
                                           int comp, int lane) {
  const unsigned FULL = 0xffffffffu;
  const uint32_t ue = (uint32_t)e;
  const bool colok = lane < ncl;
  auto dlt = [&](int rr, int cc) -> I {
    if (sizeof(I) == 4) return (I)pp.d[comp][rr][cc];
    return (I)o[rr][cc] - (I)pp.at(comp, rr, cc);
  };
  const I dT = dlt(0, lane + 1), dC = dlt(0, 0);
  const I hL = dlt(lane + 1, 0);   // lane = row: the left halo of row lane
  const uint32_t rL = res_delta(hL, m, M, c32);
  const uint32_t base = bs_msub(res_delta(dT, m, M, c32), res_delta(dC, m, M, c32), m);
  I dU = dT, hU = dC;
  int32_t eU = 0;
  const int sj = STRIDE == 2 ? (lane >> 1) : lane / stride;
  const bool scol = colok && (STRIDE == 2 ? (lane & 1) == 0 : (lane % stride) == 0);
  int rph = 0, srow = 0;   // row phase (runtime stride) and sample row
#pragma unroll 2
  for (int i = 0; i < nr; i++) {
    const I d = dlt(i + 1, lane + 1);
    const I hl = (I)__shfl_sync(FULL, hL, i);
    const uint32_t zl = __shfl_sync(FULL, rL, i);
    const uint32_t s = bs_msub(bs_madd(base, zl, m), res_delta(d, m, M, c32), m);
    const bool tie = colok && s == ue;
    int32_t er = colok ? bs_rep(s, ue, m) : 0;
    I dl = (I)__shfl_up_sync(FULL, d, 1);
    I dul = (I)__shfl_up_sync(FULL, dU, 1);
    if (lane == 0) { dl = hl; dul = hU; }
    const int32_t R0 = (int32_t)(d - dU - dl + dul);
    uint32_t tm = __ballot_sync(FULL, tie);
    while (tm) {   // raster order: x = R0 - (eU + eL - eUL)
      const int jj = __ffs(tm) - 1;
      tm &= tm - 1u;
      int32_t el = __shfl_up_sync(FULL, er, 1);
      int32_t eul = __shfl_up_sync(FULL, eU, 1);
      if (lane == 0) { el = 0; eul = 0; }
      if (lane == jj)
        er = ((int64_t)R0 - ((int64_t)eU + el - eul)) > 0 ? e : -e;
    }
    int32_t el = __shfl_up_sync(FULL, er, 1);
    int32_t eul = __shfl_up_sync(FULL, eU, 1);
    if (lane == 0) { el = 0; eul = 0; }
    const bool srw = STRIDE == 2 ? (i & 1) == 0 : rph == 0;
    if (scol && srw) {
      // |idx| = |R0 + D(err')| / m, an exact multiple
      const int64_t n = (int64_t)R0 + er - eU - el + eul;
      const uint32_t an = (uint32_t)(n < 0 ? -n : n);
      uint32_t qa = __umulhi(an, M);
      if (qa * m != an) qa++;
      const int sr = STRIDE == 2 ? (i >> 1) : srow;
      samp[2 * (sr * nsx + sj) + comp] = (int16_t)qa;
    }
    if (STRIDE != 2) {
      if (++rph == stride) { rph = 0; srow++; }
    }
    eU = er;
    dU = d;
    hU = hl;
  }
}

// The same trial without the row recurrence (stride 2, narrow tile, no
// escapes).  With s(i, j) = dT(j) + dL(i) - dC - d(i, j) (integers, |s| <
// 2^31) the trial error is err' = s - k m, k the integer nearest to s / m,
// and since D(s) = -D(d) = -R0 the symbol R0 + D(err') = -m D(k): one
// rounding per pixel, no shuffles, k = 0 on the halo row / column.  A task is
// one (sample, component): the 2x2 pixels ending at the sample.  A tie
// (s - k m = +-e, decided in raster order by the sign of x) sends the block
// to trial_rows.
__device__ __forceinline__ bool trial_sample(const int32_t (*dt)[33], int i,
                                             int j, uint32_t e, uint32_t m,
                                             uint32_t M, int* qabs) {
  // tile coordinates: pixel (a, b) of the block is [a + 1][b + 1]
  auto dl = [&](int rr, int cc) -> int32_t { return dt[rr][cc]; };
  const int32_t dC = dl(0, 0);
  const int32_t bT0 = dl(0, j) - dC, bT1 = dl(0, j + 1) - dC;
  const int32_t dL0 = dl(i, 0), dL1 = dl(i + 1, 0);
  bool t00, t01, t10, t11;
  const int32_t k00 = bs_knear(bT0 + dL0 - dl(i, j), e, m, M, &t00);
  const int32_t k01 = bs_knear(bT1 + dL0 - dl(i, j + 1), e, m, M, &t01);
  const int32_t k10 = bs_knear(bT0 + dL1 - dl(i + 1, j), e, m, M, &t10);
  const int32_t k11 = bs_knear(bT1 + dL1 - dl(i + 1, j + 1), e, m, M, &t11);
  const int32_t q = k11 - k01 - k10 + k00;
  *qabs = q < 0 ? -q : q;
  return t00 | t01 | t10 | t11;
}

// the runtime-stride / wide-tile trial (rare) out of line
static __device__ __noinline__ void trial_rows_generic(
    const int32_t (*o)[33], PvTile pp, int nr, int ncl,
    int stride, int nsx, int32_t e, uint32_t m, uint32_t M, uint32_t c32,
    int16_t* samp, int comp, int lane) {
  trial_rows<int64_t, 0>(o, pp, nr, ncl, stride, nsx, e, m, M, c32, samp, comp, lane);
}

// the row-streamed narrow trial (a tie in the sample-parallel trial, or a
// component that may escape next to one that cannot) out of line
static __device__ __noinline__ void trial_rows_n2(
    const int32_t (*o)[33], PvTile pp, int nr, int ncl, int nsx, int32_t e,
    uint32_t m, uint32_t M, uint32_t c32, int16_t* samp, int comp, int lane) {
  trial_rows<int32_t, 2>(o, pp, nr, ncl, 2, nsx, e, m, M, c32, samp, comp, lane);
}

template <typename F>
__device__ __forceinline__ void enc_block_body(
    const F* __restrict__ u, const F* __restrict__ v,
    const uint8_t* __restrict__ codes_t, const int2* __restrict__ prev,
    int2* __restrict__ rec, const PrepParams& p, const BScanIO& bio,
    const double* __restrict__ log2tab, uint8_t* __restrict__ modes_t,
    const int64_t* __restrict__ qd_row_off, const int32_t* __restrict__ pre_nl,
    uint16_t* __restrict__ qd, int32_t* __restrict__ row_ll,
    int* __restrict__ overflow, EncBlockSmem& sm);

template <typename F>
__global__ void __launch_bounds__(128, 8)
enc_block_kernel(const F* __restrict__ u, const F* __restrict__ v,
                 const uint8_t* __restrict__ codes_t,   // frame t, pitch W
                 const int2* __restrict__ prev,         // recon(t-1), pitch Wp
                 int2* __restrict__ rec,                // recon(t), pitch Wp
                 PrepParams p, BScanIO bio, const double* __restrict__ log2tab,
                 uint8_t* __restrict__ modes_t, const int64_t* __restrict__ qd_row_off,
                 const int32_t* __restrict__ pre_nl, uint16_t* __restrict__ qd,
                 int32_t* __restrict__ row_ll, int* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EncBlockSmem& sm = *reinterpret_cast<EncBlockSmem*>(smem_raw);
  enc_block_body<F>(u, v, codes_t, prev, rec, p, bio, log2tab, modes_t,
                    qd_row_off, pre_nl, qd, row_ll, overflow, sm);
}

template <typename F>
__device__ __forceinline__ void enc_block_body(
    const F* __restrict__ u, const F* __restrict__ v,
    const uint8_t* __restrict__ codes_t, const int2* __restrict__ prev,
    int2* __restrict__ rec, const PrepParams& p, const BScanIO& bio,
    const double* __restrict__ log2tab, uint8_t* __restrict__ modes_t,
    const int64_t* __restrict__ qd_row_off, const int32_t* __restrict__ pre_nl,
    uint16_t* __restrict__ qd, int32_t* __restrict__ row_ll,
    int* __restrict__ overflow, EncBlockSmem& sm) {
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int bj = blockIdx.x, bi = blockIdx.y;
  const int H = p.H, W = p.W, Wp = p.Wp;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const int64_t HW = (int64_t)H * W;
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  const int64_t blk = (int64_t)bi * p.nbx + bj;
  const F* uo = u + (int64_t)p.t * HW;
  const F* vo = v + (int64_t)p.t * HW;
  const bool has_prev = prev != nullptr;

  // ---- tiles: orig(t) (fixed point) and delta = orig - recon(t-1) at rows
  // r0-1 .. r0+31, columns c0-1 .. c0+31 (recon(t-1) is zero outside the
  // frame, as the reference's Lorenzo terms vanish there); max |delta| on
  // the way (|o - p| < 2^32: exact in uint32)
  if (tid < 8) sm.flag[tid] = 0;
  if (tid < 32) sm.etab[tid] = bio.e_tab[tid];
  reinterpret_cast<uint4*>(&sm.cnt[0][0])[tid] = make_uint4(0, 0, 0, 0);
  static_assert(2 * ETB * sizeof(int16_t) == 128 * sizeof(uint4), "cnt zeroing");
  uint32_t maxd = 0;
  auto put = [&](int rr, int cc, F xu, F xv, int2 pr, bool ok) {
    const int32_t ou = ok ? fixed_t(xu, p.S) : 0, ov = ok ? fixed_t(xv, p.S) : 0;
    sm.o[0][rr][cc] = ou;
    sm.o[1][rr][cc] = ov;
    sm.d[0][rr][cc] = (int32_t)((uint32_t)ou - (uint32_t)pr.x);
    sm.d[1][rr][cc] = (int32_t)((uint32_t)ov - (uint32_t)pr.y);
    const uint32_t du = ou > pr.x ? (uint32_t)ou - (uint32_t)pr.x : (uint32_t)pr.x - (uint32_t)ou;
    const uint32_t dv = ov > pr.y ? (uint32_t)ov - (uint32_t)pr.y : (uint32_t)pr.y - (uint32_t)ov;
    maxd = max(maxd, max(du, dv));
  };
  const bool full = nr == 32 && ncl == 32;
  const bool vec = full && sizeof(F) == 4 && (W & 3) == 0 &&
                   (((uintptr_t)uo | (uintptr_t)vo | (uintptr_t)codes_t) & 15) == 0;
  if (vec) {
    // interior: 16-byte loads, four pixels per thread and step
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int idx = tid + 128 * q;     // 256 = 32 rows x 8 quads
      const int i = idx >> 3, c4 = (idx & 7) * 4;
      const int64_t n = (int64_t)(r0 + i) * W + c0 + c4;
      const float4 a = __ldg(reinterpret_cast<const float4*>(uo + n));
      const float4 b = __ldg(reinterpret_cast<const float4*>(vo + n));
      int4 p01 = make_int4(0, 0, 0, 0), p23 = make_int4(0, 0, 0, 0);
      if (has_prev) {
        const int4* pp = reinterpret_cast<const int4*>(prev + (int64_t)(r0 + i) * Wp + c0 + c4);
        p01 = __ldg(pp);
        p23 = __ldg(pp + 1);
      }
      put(i + 1, c4 + 1, (F)a.x, (F)b.x, make_int2(p01.x, p01.y), true);
      put(i + 1, c4 + 2, (F)a.y, (F)b.y, make_int2(p01.z, p01.w), true);
      put(i + 1, c4 + 3, (F)a.z, (F)b.z, make_int2(p23.x, p23.y), true);
      put(i + 1, c4 + 4, (F)a.w, (F)b.w, make_int2(p23.z, p23.w), true);
    }
    // halo: row r0-1 (33 values incl. the corner), column c0-1
    if (tid < 65) {
      const bool rowh = tid < 33;
      const int rr = rowh ? 0 : tid - 32, cc = rowh ? tid : 0;
      const int i = r0 - 1 + rr, j = c0 - 1 + cc;
      const bool ok = i >= 0 && j >= 0;
      F xu = 0, xv = 0;
      int2 pr = make_int2(0, 0);
      if (ok) {
        xu = __ldg(uo + (int64_t)i * W + j);
        xv = __ldg(vo + (int64_t)i * W + j);
        if (has_prev) pr = __ldg(prev + (int64_t)i * Wp + j);
      }
      put(rr, cc, xu, xv, pr, ok);
    }
    // codes: 4-byte loads
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int idx = tid + 128 * q;     // 256 = 32 rows x 8 words
      const int i = idx >> 3, c4 = (idx & 7) * 4;
      const uint32_t w4 = __ldg(reinterpret_cast<const uint32_t*>(
          codes_t + (int64_t)(r0 + i) * W + c0 + c4));
      *reinterpret_cast<uint32_t*>(&sm.cd[i][c4]) = w4;
    }
  } else {
#pragma unroll 3
    for (int k = tid; k < 33 * 33; k += 128) {
      const int rr = k / 33, cc = k - 33 * rr;
      const int i = r0 - 1 + rr, j = c0 - 1 + cc;
      const bool ok = i >= 0 && j >= 0 && i < H && j < W;
      F xu = 0, xv = 0;
      int2 pr = make_int2(0, 0);
      if (ok) {
        xu = __ldg(uo + (int64_t)i * W + j);
        xv = __ldg(vo + (int64_t)i * W + j);
        if (has_prev) pr = __ldg(prev + (int64_t)i * Wp + j);
      }
      put(rr, cc, xu, xv, pr, ok);
    }
#pragma unroll 2
    for (int k = tid; k < 1024; k += 128) {
      const int i = k >> 5, j = k & 31;
      sm.cd[i][j] = (i < nr && j < ncl) ? codes_t[(int64_t)(r0 + i) * W + c0 + j]
                                        : (uint8_t)CODE_LOSSLESS;
    }
  }
  __syncthreads();   // flag[] zeroed before the atomics below
  {
    int md = (int)min(maxd, (uint32_t)INT32_MAX);
    md = __reduce_max_sync(FULL, md);
    if (lane == 0) atomicMax(&sm.flag[F_MAXD], md);
  }
  const PvTile pvt{sm.o, sm.d};
  // ---- code checks (whole words in a full block)
  const int code0 = sm.cd[0][0];
  {
    bool nonuni = false, lossy = false, lossless = false;
    if (full) {
      const uint32_t cm4 = 0x01010101u * (uint32_t)__popc(p.lossy_mask);
      const uint32_t c04 = 0x01010101u * (uint32_t)code0;
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int idx = tid + 128 * q;
        const uint32_t w4 = *reinterpret_cast<const uint32_t*>(&sm.cd[idx >> 3][(idx & 7) * 4]);
        const uint32_t lt = __vcmpltu4(w4, cm4);   // 0xff where the code quantises
        nonuni |= w4 != c04;
        lossy |= lt != 0u;
        lossless |= lt != 0xffffffffu;
      }
    } else {
      for (int i = wid; i < nr; i += 4) {
        if (lane >= ncl) continue;
        const int cd = sm.cd[i][lane];
        const bool ls = sm.etab[cd & 31] > 0;
        nonuni |= cd != code0;
        lossy |= ls;
        lossless |= !ls;
      }
    }
    if (__any_sync(FULL, nonuni) && lane == 0) sm.flag[F_NONUNI] = 1;
    if (__any_sync(FULL, lossy) && lane == 0) sm.flag[F_LOSSY] = 1;
    if (__any_sync(FULL, lossless) && lane == 0) sm.flag[F_LOSSLESS] = 1;
  }
  __syncthreads();

  // ---- unless 4 max|delta| bounds them, the exact R0 escape checks (warp
  // w: rows w, w+4, ...; lane = column)
  const int64_t e0 = p.lad.e[code0];
  const int64_t tau = p.tau;
  auto lim_of = [&](int64_t e) -> int64_t {
    const int64_t l = (2 * (int64_t)p.radius - 4) * e;
    return l > ((int64_t)1 << 30) ? ((int64_t)1 << 30) : l;
  };
  const int64_t limT = lim_of(tau), lim0 = lim_of(e0);
  const int64_t maxd4 = 4 * (int64_t)sm.flag[F_MAXD];
  const bool narrow = sm.flag[F_MAXD] < (1 << 29);
  const bool colok = lane < ncl;
  // R0 of pixel (i, j) from the tiles (exact)
  auto R0_at = [&](int c, int i, int j) -> int64_t {
    if (narrow) {
      const int32_t(*dt)[33] = sm.d[c];
      return (int64_t)(dt[i + 1][j + 1] - dt[i][j + 1] - dt[i + 1][j] + dt[i][j]);
    }
    const int32_t(*o)[33] = sm.o[c];
    return ((int64_t)o[i + 1][j + 1] - pvt.at(c, i + 1, j + 1)) -
           ((int64_t)o[i][j + 1] - pvt.at(c, i, j + 1)) -
           ((int64_t)o[i + 1][j] - pvt.at(c, i + 1, j)) +
           ((int64_t)o[i][j] - pvt.at(c, i, j));
  };
  if (maxd4 >= lim0) {   // (uniform over the CTA)
    {
      bool ovf = false;
      bool unT[2] = {false, false}, un0[2] = {false, false};
      for (int i = wid; i < nr; i += 4) {
        if (!colok) continue;
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int64_t R0 = R0_at(c, i, lane);
          const int64_t a = R0 < 0 ? -R0 : R0;
          ovf |= a >= 2147483647LL;
          unT[c] |= a >= limT;
          un0[c] |= a >= lim0;
        }
      }
      if (__any_sync(FULL, ovf) && lane == 0) sm.flag[F_OVF] = 1;
      const unsigned ut = (__any_sync(FULL, unT[0]) ? 1u : 0u) | (__any_sync(FULL, unT[1]) ? 2u : 0u);
      const unsigned u0 = (__any_sync(FULL, un0[0]) ? 1u : 0u) | (__any_sync(FULL, un0[1]) ? 2u : 0u);
      if (lane == 0 && ut) atomicOr(&sm.flag[F_UNSAFE_T], (int)ut);
      if (lane == 0 && u0) atomicOr(&sm.flag[F_UNSAFE_0], (int)u0);
    }
    __syncthreads();
    if (tid == 0 && sm.flag[F_OVF]) atomicOr(overflow, 1);
  }

  // ---- MoP mode decision (mop.py:68-151)
  const int nsx = (ncl + p.stride - 1) / p.stride;
  const int nsy = (nr + p.stride - 1) / p.stride;
  const int nsamp = nsx * nsy;
  int mode = p.force_sl;
  if (p.mop) {
    const int32_t e = (int32_t)tau;   // fast path: tau' < 2^29
    const double inv = p.lad.inv2e[0];
    const int32_t radius = p.radius;
    // sample-parallel trial when the tile is narrow and cannot escape
    const bool kform = narrow && p.stride == 2 && (sm.flag[F_UNSAFE_T] & 3) == 0;
    if (kform) {
      const uint32_t ue = (uint32_t)e, m = 2u * ue, M = bio.mag_tab[0];
      const int comp = lane >> 4, sj = lane & 15;
      const int32_t(*dt)[33] = sm.d[comp];
      bool tie = false;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int si = wid + 4 * r;
        if (2 * si < nr && 2 * sj < ncl) {
          int qa;
          tie |= trial_sample(dt, 2 * si, 2 * sj, ue, m, M, &qa);
          sm.samp[0][2 * (si * nsx + sj) + comp] = (int16_t)qa;
        }
      }
      if (__any_sync(FULL, tie) && lane == 0) sm.flag[F_TIE] = 1;
    } else
    if (wid < 2) {
      // Lorenzo trial of component wid with the step tau' everywhere and a
      // zero error boundary (candidate = orig outside the block)
      const int comp = wid;
      const uint32_t m = 2u * (uint32_t)e, ue = (uint32_t)e;
      const uint32_t M = bio.mag_tab[0], c32 = bio.c32_tab[0];
      const int32_t(*o)[33] = sm.o[comp];
      const PvTile pp = pvt;
      if (!((sm.flag[F_UNSAFE_T] >> comp) & 1)) {
        int16_t* samp = &sm.samp[0][0];
        if (narrow && p.stride == 2)
          trial_rows_n2(o, pp, nr, ncl, nsx, e, m, M, c32, samp, comp, lane);
        else
          trial_rows_generic(o, pp, nr, ncl, p.stride, nsx, e, m, M, c32, samp, comp, lane);
      } else {
        // escapes possible: the exact raster sweep of the trial (skewed:
        // lane = row, step s visits column s - lane)
        const int i = lane;
        const bool rowok = i < nr;
        int32_t eL = 0, eUL = 0;
        const bool srow = (i % p.stride) == 0;
        const int sbase = 2 * ((i / p.stride) * nsx) + comp;
        int jm = 0, jq = 0;
#pragma unroll 1
        for (int s = 0; s < 63; s++) {
          const int jj = s - lane;
          const bool act = rowok && jj >= 0 && jj < ncl;
          const int32_t x0 = act ? (int32_t)R0_at(comp, i, jj) : 0;
          const int32_t q0 = act ? quant32(x0, e, inv) : 0;
          const int32_t rho = x0 - q0 * 2 * e;
          const int32_t up = __shfl_up_sync(FULL, eL, 1);
          const int32_t eU = (lane == 0 || !act) ? 0 : up;
          const int32_t dd = eU + (jj > 0 ? eL : 0) - ((jj > 0 && lane > 0) ? eUL : 0);
          int32_t qa;
          const int32_t er = trial_step(rho, q0, e, dd, radius, &qa);
          eUL = eU;
          if (act) eL = er;
          if (act && srow && jm == 0) sm.samp[0][sbase + 2 * jq] = (int16_t)qa;
          if (jj >= 0) {
            if (++jm == p.stride) { jm = 0; jq++; }
          }
        }
      }
    }
    {
      // semi-Lagrangian trial at the stride samples, two per lane in lockstep
      // so the departure-point gathers overlap: warps 2 and 3 take samples
      // [0, 128) at once, warps 0 and 1 [128, 256) after their Lorenzo trial;
      // the predictions are kept for the block's encode
      const int t2 = wid >= 2 ? tid - 64 : tid + 128;
      int64_t pr_u[2], pr_v[2];
      int si_i[2], si_j[2];
      bool slow[2];
#pragma unroll
      for (int b = 0; b < 2; b++) {
        const int sidx = min(t2 + 64 * b, nsamp - 1);
        const int si = sidx / nsx, sj = sidx - si * nsx;
        si_i[b] = r0 + si * p.stride;
        si_j[b] = c0 + sj * p.stride;
        slow[b] = !sl_predict_rk2(PairPlane{prev, Wp}, H, W, si_i[b], si_j[b],
                                  p.cfl_x, p.cfl_y, p.d_max, &pr_u[b], &pr_v[b]);
      }
#pragma unroll 1
      for (int b = 0; b < 2; b++) {
        const int sidx = t2 + 64 * b;
        if (sidx >= nsamp) continue;
        if (slow[b])
          sl_general(prev, Wp, H, W, si_i[b], si_j[b], p.cfl_x, p.cfl_y, p.d_max,
                     p.n_max, &pr_u[b], &pr_v[b]);
        const int li = si_i[b] - r0 + 1, lj = si_j[b] - c0 + 1;
        const int64_t ru = (int64_t)sm.o[0][li][lj] - pr_u[b];
        const int64_t rv = (int64_t)sm.o[1][li][lj] - pr_v[b];
        // |idx| = |rha(r / 2 tau')|, |r| < 2^32
        const uint32_t mt = 2u * (uint32_t)e, Mt = bio.mag_tab[0];
        const uint32_t qu = bs_qabs((uint32_t)(ru < 0 ? -ru : ru), (uint32_t)e, mt, Mt);
        const uint32_t qv = bs_qabs((uint32_t)(rv < 0 ? -rv : rv), (uint32_t)e, mt, Mt);
        sm.samp[1][2 * sidx] = (int16_t)(qu < (uint32_t)radius ? (int)qu : -1);
        sm.samp[1][2 * sidx + 1] = (int16_t)(qv < (uint32_t)radius ? (int)qv : -1);
        sm.spu[sidx] = (int32_t)pr_u[b];
        sm.spv[sidx] = (int32_t)pr_v[b];
      }
    }
    __syncthreads();
    if (kform && sm.flag[F_TIE]) {
      // rare: a tie somewhere in the block, the trial in raster order
      if (wid < 2)
        trial_rows_n2(sm.o[wid], pvt, nr, ncl, nsx, e, 2u * (uint32_t)e,
                      bio.mag_tab[0], bio.c32_tab[0], &sm.samp[0][0], wid, lane);
      __syncthreads();
    }
    if (wid == 0 || wid == 2) {
      const int tr = wid >> 1;
      const double r = block_rate(sm.samp[tr], 2 * nsamp, sm.cnt[tr], sm.order[tr],
                                  log2tab, p.lam, p.rmeta, lane);
      if (lane == 0) sm.rate[tr] = r;
    }
    __syncthreads();
    const double r_lor = sm.rate[0], r_sl = sm.rate[1];
    mode = (r_lor > 0.0 && __ddiv_rn(__dsub_rn(r_lor, r_sl), r_lor) > p.theta) ? 1 : 0;
    if (tid == 0) modes_t[blk] = (uint8_t)mode;
  }

  const int64_t rowbase = (int64_t)p.t * H;
  if (mode == 1) {
    // ---- semi-Lagrangian block (codec.py:140-155 with the SL prediction):
    // every pixel is pinned (its value does not depend on the recurrence)
    const PairPlane src{prev, Wp};
    const int j = c0 + lane;
    const bool sc = (lane % p.stride) == 0;
    const double* inv2e = p.lad.inv2e;
#pragma unroll 1
    for (int i0 = wid; i0 < nr; i0 += 8) {
      // two rows per step (i0, i0 + 4) so their gathers overlap
      int64_t pu[2], pv[2];
      bool need[2], slow[2], have[2];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int i = i0 + 4 * q;
        const bool rv_ = i < nr;
        const int cd = rv_ && colok ? sm.cd[i][lane] : CODE_LOSSLESS;
        need[q] = rv_ && colok && sm.etab[cd & 31] > 0;
        have[q] = p.mop && sc && (i % p.stride) == 0;
        pu[q] = pv[q] = 0;
        slow[q] = false;
        if (have[q] && need[q]) {
          const int sidx = (i / p.stride) * nsx + lane / p.stride;
          pu[q] = sm.spu[sidx];
          pv[q] = sm.spv[sidx];
        }
      }
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int i = min(i0 + 4 * q, nr - 1);
        if (__any_sync(FULL, need[q] && !have[q]) && !have[q])
          slow[q] = !sl_predict_rk2(src, H, W, r0 + i, min(j, W - 1), p.cfl_x,
                                    p.cfl_y, p.d_max, &pu[q], &pv[q]);
      }
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int i = i0 + 4 * q;
        if (i >= nr) break;   // warp-uniform
        if (slow[q] && need[q])
          sl_general(prev, Wp, H, W, r0 + i, j, p.cfl_x, p.cfl_y, p.d_max,
                     p.n_max, &pu[q], &pv[q]);
        const int cd = colok ? sm.cd[i][lane] : CODE_LOSSLESS;
        const int64_t e = sm.etab[cd & 31];
        const bool nl = colok && e > 0;
        const int32_t ou = colok ? sm.o[0][i + 1][lane + 1] : 0;
        const int32_t ov = colok ? sm.o[1][i + 1][lane + 1] : 0;
        int32_t ru = ou, rv = ov;
        int nll = (colok && !nl) ? 2 : 0;
        const unsigned bnl = __ballot_sync(FULL, nl);
        if (nl) {
          // idx = rha(r / 2e) from its magnitude (|r| < 2^32); recon fits
          // int32, so pred + idx * 2e may wrap on the way
          const uint32_t ue = (uint32_t)e, m = 2u * ue, M = bio.mag_tab[cd & 31];
          const int64_t du = (int64_t)ou - pu[q], dv = (int64_t)ov - pv[q];
          const uint32_t au = bs_qabs((uint32_t)(du < 0 ? -du : du), ue, m, M);
          const uint32_t av = bs_qabs((uint32_t)(dv < 0 ? -dv : dv), ue, m, M);
          const bool oku = au < (uint32_t)p.radius, okv = av < (uint32_t)p.radius;
          const int32_t qu = du < 0 ? -(int32_t)au : (int32_t)au;
          const int32_t qv = dv < 0 ? -(int32_t)av : (int32_t)av;
          if (oku) ru = (int32_t)((uint32_t)pu[q] + (uint32_t)qu * m);
          if (okv) rv = (int32_t)((uint32_t)pv[q] + (uint32_t)qv * m);
          const uint32_t syu = oku ? (uint32_t)(qu + p.radius) : 0u;
          const uint32_t syv = okv ? (uint32_t)(qv + p.radius) : 0u;
          const int64_t row = rowbase + r0 + i;
          const int64_t pos = qd_row_off[row] +
                              2 * ((int64_t)pre_nl[row * p.nchunks + bj] + __popc(bnl & lt));
          *reinterpret_cast<uint32_t*>(qd + pos) = syu | (syv << 16);
          nll = (oku ? 0 : 1) + (okv ? 0 : 1);
        }
        if (colok) rec[(int64_t)(r0 + i) * Wp + j] = make_int2(ru, rv);
        const int tot = __reduce_add_sync(FULL, nll);
        if (lane == 0 && tot) atomicAdd(row_ll + rowbase + r0 + i, tot);
        // the block's err edges for the chain
        if (i == nr - 1) {
          bio.lb[blk * 32 + lane] = colok ? ru - ou : 0;
          bio.lb[(nblk + blk) * 32 + lane] = colok ? rv - ov : 0;
        }
        if (lane == ncl - 1) {
          bio.lr[blk * 32 + i] = ru - ou;
          bio.lr[(nblk + blk) * 32 + i] = rv - ov;
        }
      }
    }
    if (tid < 64) {
      // rows past the frame of a ragged block: zero right-column entries
      const int c = tid >> 5;
      if (lane >= nr) bio.lr[(c * nblk + blk) * 32 + lane] = 0;
      if (lane == 0) bio.cls[c * nblk + blk] = BS_KNOWN;
    }
    return;
  }

  // ---- Lorenzo block
  const bool any_lossy = sm.flag[F_LOSSY] != 0;
  const bool any_lossless = sm.flag[F_LOSSLESS] != 0;
  if (!any_lossy) {
    // every pixel lossless: recon = orig, err edges 0, two ll values each
    for (int i = wid; i < nr; i += 4) {
      if (colok)
        rec[(int64_t)(r0 + i) * Wp + c0 + lane] =
            make_int2(sm.o[0][i + 1][lane + 1], sm.o[1][i + 1][lane + 1]);
      if (lane == 0) atomicAdd(row_ll + rowbase + r0 + i, 2 * ncl);
    }
    if (tid < 64) {
      const int c = tid >> 5;
      bio.lb[(c * nblk + blk) * 32 + lane] = 0;
      bio.lr[(c * nblk + blk) * 32 + lane] = 0;
      if (lane == 0) bio.cls[c * nblk + blk] = BS_KNOWN;
    }
    return;
  }
  if (any_lossless) {
    // two ll values per lossless pixel (the chain sweeps such a block)
    for (int i = wid; i < nr; i += 4) {
      const bool ll = colok && sm.etab[sm.cd[i][lane] & 31] == 0;
      const int nll = 2 * __popc(__ballot_sync(FULL, ll));
      if (lane == 0 && nll) atomicAdd(row_ll + rowbase + r0 + i, nll);
    }
  }
  const bool uniform = !sm.flag[F_NONUNI] && !any_lossless && e0 > 0;
  if (wid < 2) {
    const int c = wid;
    const bool reg = uniform && !((sm.flag[F_UNSAFE_0] >> c) & 1);
    if (reg) {
      // edges of -Pd (mod m0) for the chain: bottom row and right column,
      // from the residues of the four deltas
      const uint32_t m = 2u * (uint32_t)e0;
      const uint32_t M = bio.mag_tab[code0], c32 = bio.c32_tab[code0];
      const int32_t(*o)[33] = sm.o[c];
      auto rd = [&](int rr, int cc) -> uint32_t {
        if (narrow) return bs_res_any(sm.d[c][rr][cc], m, M);
        return res_i64((int64_t)o[rr][cc] - pvt.at(c, rr, cc), m, M, c32);
      };
      const uint32_t rc = rd(0, 0);
      int32_t lbv = 0, lrv = 0;
      if (lane < ncl) {
        // -Pd = -d(nr-1, j) + d(-1, j) + d(nr-1, -1) - d(-1, -1)
        const uint32_t s = bs_msub(bs_madd(rd(0, lane + 1), rd(nr, 0), m),
                                   bs_madd(rd(nr, lane + 1), rc, m), m);
        lbv = (int32_t)s;
      }
      if (lane < nr) {
        const uint32_t s = bs_msub(bs_madd(rd(0, ncl), rd(lane + 1, 0), m),
                                   bs_madd(rd(lane + 1, ncl), rc, m), m);
        lrv = (int32_t)s;
      }
      bio.lb[(c * nblk + blk) * 32 + lane] = lbv;
      bio.lr[(c * nblk + blk) * 32 + lane] = lrv;
      if (lane == 0)
        bio.cls[c * nblk + blk] = BS_REG | (code0 << 2) |
                                  (sm.flag[F_MAXD] < (1 << 27) ? BS_NARROW : 0);
    } else if (lane == 0) {
      bio.cls[c * nblk + blk] = BS_SLOW;
    }
  }
  // R0 plane for the components the chain sweeps
  const int slow_mask = uniform ? (sm.flag[F_UNSAFE_0] & 3) : 3;
  if (slow_mask) {
    for (int i = wid; i < nr; i += 4) {
      if (!colok) continue;
      const int64_t k = (int64_t)(r0 + i) * Wp + c0 + lane;
      if (slow_mask & 1) bio.a_w[0][k] = (int32_t)R0_at(0, i, lane);
      if (slow_mask & 2) bio.a_w[1][k] = (int32_t)R0_at(1, i, lane);
    }
  }
}

template <typename F>
cudaError_t launch_enc_block(const F* u, const F* v, const uint8_t* codes_t,
                             const int32_t* prev, int32_t* rec,
                             const PrepParams& p, const BScanIO& bio,
                             const double* log2tab, uint8_t* modes_t,
                             const int64_t* qd_row_off, const int32_t* pre_nl,
                             uint16_t* qd, int32_t* row_ll, int* overflow,
                             cudaStream_t st) {
  const size_t smem = sizeof(EncBlockSmem);
  static OncePerDevice once;
  int dummy = 0;
  const cudaError_t e = once.get(
      [&](int*) {
        return cudaFuncSetAttribute(enc_block_kernel<F>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
      },
      &dummy);
  if (e != cudaSuccess) return e;
  enc_block_kernel<F><<<dim3(p.nbx, p.nby), 128, smem, st>>>(
      u, v, codes_t, reinterpret_cast<const int2*>(prev),
      reinterpret_cast<int2*>(rec), p, bio, log2tab, modes_t, qd_row_off,
      pre_nl, qd, row_ll, overflow);
  return cudaGetLastError();
}

template cudaError_t launch_enc_block<float>(
    const float*, const float*, const uint8_t*, const int32_t*, int32_t*,
    const PrepParams&, const BScanIO&, const double*, uint8_t*, const int64_t*,
    const int32_t*, uint16_t*, int32_t*, int*, cudaStream_t);
template cudaError_t launch_enc_block<double>(
    const double*, const double*, const uint8_t*, const int32_t*, int32_t*,
    const PrepParams&, const BScanIO&, const double*, uint8_t*, const int64_t*,
    const int32_t*, uint16_t*, int32_t*, int*, cudaStream_t);

}  // namespace vfcp
