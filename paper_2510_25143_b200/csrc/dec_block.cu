// The decoder's per-block preparation of one frame (codec.py:167-206
// _decode_frame): one CTA per 32x32 block reads the block's eb codes,
// symbols and lossless values once and
//   * semi-Lagrangian blocks (mode 1, t >= 1): predicts every pixel from
//     recon(t-1) (predictors.py:76-108) and writes recon(t), the float64
//     output and the Z = recon - recon(t-1) edges for the chain -- the block
//     is KNOWN;
//   * Lorenzo blocks, per component: with no pinned pixel (no lossless
//     vertex, no escape) the component is REG and only the bottom row /
//     right column of the 2D prefix sums of A = (sym - radius) * 2e go to the
//     chain (the decoder's recurrence Z = ZU + ZL - ZUL + A is exact in
//     wrapping uint32 arithmetic, so the interior is that prefix sum plus the
//     exact boundary, rebuilt by the chain's interior pass, bscan.cuh); with
//     every pixel pinned it is KNOWN (recon = the ll values, written here);
//     otherwise SLOW: the A / Z plane and the pin words go to the chain,
//     which sweeps it.
#include "bscan.cuh"
#include "predict.cuh"

namespace vfcp {

constexpr int DB_NW = 8;           // warps per block (rows w, w + 8, ...)
constexpr int DB_OCC = 4;          // CTAs per SM of the general kernel (register cap)

struct DecBlockSmem {
  alignas(16) uint32_t colsum[2][DB_NW][32];   // per warp: column sums of A (REG edges)
  uint32_t rowsum[2][32];      // row sums of A
  int anypin[2], notall[2];
  int32_t etab[32];            // e per code
  alignas(16) int2 pv[SLT][SLT];   // recon(t-1) tile (semi-Lagrangian blocks)
};

template <typename SYM>
__device__ __forceinline__ void dec_block_body(
    const uint8_t* __restrict__ codes_t, const SYM* __restrict__ qd,
    const int64_t* __restrict__ ll, const uint8_t* __restrict__ modes_t,
    const int2* __restrict__ prev, int2* __restrict__ rec,
    const int64_t* __restrict__ qd_row_off,
    const int64_t* __restrict__ ll_row_off, const int32_t* __restrict__ pre_nl,
    const int32_t* __restrict__ pre_ll, const PrepParams& p, const BScanIO& bio,
    uint32_t* __restrict__ pin_u, uint32_t* __restrict__ pin_v,
    double* __restrict__ f64u, double* __restrict__ f64v,
    int64_t* __restrict__ fixu, int64_t* __restrict__ fixv, double inv_S,
    DecBlockSmem& sm, int bi, int bj);

template <typename SYM>
__global__ void __launch_bounds__(32 * DB_NW, DB_OCC)
dec_block_kernel(const uint8_t* __restrict__ codes_t,   // frame t, pitch W
                 const SYM* __restrict__ qd, const int64_t* __restrict__ ll,
                 const uint8_t* __restrict__ modes_t,
                 const int2* __restrict__ prev,         // recon(t-1), pitch Wp
                 int2* __restrict__ rec,                // recon(t), pitch Wp
                 const int64_t* __restrict__ qd_row_off,
                 const int64_t* __restrict__ ll_row_off,
                 const int32_t* __restrict__ pre_nl,
                 const int32_t* __restrict__ pre_ll, PrepParams p, BScanIO bio,
                 uint32_t* __restrict__ pin_u, uint32_t* __restrict__ pin_v,
                 double* __restrict__ f64u, double* __restrict__ f64v,
                 int64_t* __restrict__ fixu, int64_t* __restrict__ fixv,
                 double inv_S, const int* __restrict__ list,
                 const int* __restrict__ count) {
  __shared__ DecBlockSmem sm;
  if (!list) {
    // every block of the frame (grid nbx x nby)
    dec_block_body<SYM>(codes_t, qd, ll, modes_t, prev, rec, qd_row_off,
                        ll_row_off, pre_nl, pre_ll, p, bio, pin_u, pin_v, f64u,
                        f64v, fixu, fixv, inv_S, sm, blockIdx.y, blockIdx.x);
    return;
  }
  // the blocks the fast kernel listed
  const int n = *count;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int blk = list[k];
    const int bi = blk / p.nbx, bj = blk - bi * p.nbx;
    dec_block_body<SYM>(codes_t, qd, ll, modes_t, prev, rec, qd_row_off,
                        ll_row_off, pre_nl, pre_ll, p, bio, pin_u, pin_v, f64u,
                        f64v, fixu, fixv, inv_S, sm, bi, bj);
    __syncthreads();
  }
}

// The usual block on its own: a full block whose pixels share one quantising
// code and hold no escape is REG in both components, its symbols are dense
// (64 per row) and A = (sym - radius) * 2e needs no per-pixel table: four
// pixels per thread (row tid / 8, column quad tid % 8), row sums over the 8
// lanes of a row, column sums over the warp's four rows and then the CTA's
// warps.  Any other block (semi-Lagrangian, ragged, mixed codes, lossless
// pixels, an escape) goes to the list for dec_block_kernel.
template <typename SYM>
__global__ void __launch_bounds__(32 * DB_NW, 8)
dec_block_fast_kernel(const uint8_t* __restrict__ codes_t,
                      const SYM* __restrict__ qd,
                      const uint8_t* __restrict__ modes_t,
                      const int64_t* __restrict__ qd_row_off,
                      const int32_t* __restrict__ pre_nl, PrepParams p,
                      int32_t* __restrict__ lb, int32_t* __restrict__ lr,
                      int32_t* __restrict__ cls, int32_t e_of_code0_unused,
                      const int32_t* __restrict__ e_tab_g,
                      int* __restrict__ list, int* __restrict__ count) {
  __shared__ alignas(16) uint32_t s_colsum[2][DB_NW][32];
  __shared__ uint32_t s_rowsum[2][32];
  __shared__ int s_esc;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int bj = blockIdx.x, bi = blockIdx.y;
  const int H = p.H, W = p.W, nchunks = p.nchunks;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  const int64_t blk = (int64_t)bi * p.nbx + bj;
  const int64_t rowbase = (int64_t)p.t * H;
  auto defer = [&]() {
    if (tid == 0) list[atomicAdd(count, 1)] = (int)blk;
  };
  const bool sl_blk = modes_t && modes_t[blk] == 1;
  if (sl_blk || nr != 32 || ncl != 32) {
    defer();
    return;
  }
  if (tid == 0) s_esc = 0;
  const int i = tid >> 3, cq = tid & 7;
  const int code0 = __ldg(codes_t + (int64_t)r0 * W + c0);
  const uint32_t w4 = __ldg(reinterpret_cast<const uint32_t*>(
      codes_t + (int64_t)(r0 + i) * W + c0 + 4 * cq));
  const int32_t e = __ldg(e_tab_g + (code0 & 31));
  const int64_t row = rowbase + r0 + i;
  const int64_t qoff = qd_row_off[row] + 2 * (int64_t)pre_nl[row * nchunks + bj];
  // (uniform over the CTA; also orders s_esc = 0 before the votes below)
  if (__syncthreads_or(w4 != 0x01010101u * (uint32_t)code0 || e == 0)) {
    defer();
    return;
  }
  const uint32_t* sp = reinterpret_cast<const uint32_t*>(qd + qoff) + 4 * cq;
  uint32_t sq[4];
#pragma unroll
  for (int k = 0; k < 4; k++) sq[k] = __ldg(sp + k);
  const uint32_t e2 = 2u * (uint32_t)e, rad = (uint32_t)p.radius;
  uint32_t au[4], av[4];
  bool esc = false;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t su = sq[k] & 0xffffu, sv = sq[k] >> 16;
    esc |= su == 0u || sv == 0u;
    au[k] = (su - rad) * e2;
    av[k] = (sv - rad) * e2;
  }
  // row sums (8 lanes of the row)
  uint32_t ru = au[0] + au[1] + au[2] + au[3], rv = av[0] + av[1] + av[2] + av[3];
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    ru += __shfl_xor_sync(FULL, ru, o);
    rv += __shfl_xor_sync(FULL, rv, o);
  }
  if (cq == 0) {
    s_rowsum[0][i] = ru;
    s_rowsum[1][i] = rv;
  }
  // column sums (the warp's four rows; lanes 0-7 hold columns 4 cq + k)
#pragma unroll
  for (int k = 0; k < 4; k++) {
    au[k] += __shfl_xor_sync(FULL, au[k], 8);
    av[k] += __shfl_xor_sync(FULL, av[k], 8);
    au[k] += __shfl_xor_sync(FULL, au[k], 16);
    av[k] += __shfl_xor_sync(FULL, av[k], 16);
  }
  if (lane < 8) {
    *reinterpret_cast<uint4*>(&s_colsum[0][wid][4 * cq]) = make_uint4(au[0], au[1], au[2], au[3]);
    *reinterpret_cast<uint4*>(&s_colsum[1][wid][4 * cq]) = make_uint4(av[0], av[1], av[2], av[3]);
  }
  if (__any_sync(FULL, esc) && lane == 0) s_esc = 1;
  __syncthreads();
  if (s_esc) {
    defer();
    return;
  }
  if (tid >= 64) return;
  const int c = tid >> 5;
  uint32_t cs = 0u;
#pragma unroll
  for (int w = 0; w < DB_NW; w++) cs += s_colsum[c][w][lane];
  uint32_t rs = s_rowsum[c][lane];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t pc = __shfl_up_sync(FULL, cs, o);
    const uint32_t pr = __shfl_up_sync(FULL, rs, o);
    if (lane >= o) { cs += pc; rs += pr; }
  }
  lb[(c * nblk + blk) * 32 + lane] = (int32_t)cs;
  lr[(c * nblk + blk) * 32 + lane] = (int32_t)rs;
  // (BS_NARROW: one code, dense symbols -- the interior pass's vector form)
  if (lane == 0) cls[c * nblk + blk] = BS_REG | (code0 << 2) | BS_NARROW;
}

template <typename SYM>
__device__ __forceinline__ void dec_block_body(
    const uint8_t* __restrict__ codes_t, const SYM* __restrict__ qd,
    const int64_t* __restrict__ ll, const uint8_t* __restrict__ modes_t,
    const int2* __restrict__ prev, int2* __restrict__ rec,
    const int64_t* __restrict__ qd_row_off,
    const int64_t* __restrict__ ll_row_off, const int32_t* __restrict__ pre_nl,
    const int32_t* __restrict__ pre_ll, const PrepParams& p, const BScanIO& bio,
    uint32_t* __restrict__ pin_u, uint32_t* __restrict__ pin_v,
    double* __restrict__ f64u, double* __restrict__ f64v,
    int64_t* __restrict__ fixu, int64_t* __restrict__ fixv, double inv_S,
    DecBlockSmem& sm, int bi, int bj) {
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int H = p.H, W = p.W, Wp = p.Wp, nchunks = p.nchunks;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  const int64_t blk = (int64_t)bi * p.nbx + bj;
  const bool has_prev = prev != nullptr;
  const bool sl_blk = has_prev && modes_t && modes_t[blk] == 1;
  const bool colok = lane < ncl;
  const int j = c0 + (colok ? lane : ncl - 1);
  const int64_t rowbase = (int64_t)p.t * H;
  const int64_t fbase = (int64_t)p.t * H * W;
  int32_t* recw = reinterpret_cast<int32_t*>(rec);
  if (tid < 2) { sm.anypin[tid] = 0; sm.notall[tid] = 0; }
  if (tid < 32) sm.etab[tid] = bio.e_tab[tid];
  if (sl_blk) load_prev_tile(sm.pv, prev, H, W, Wp, r0, c0, tid, 32 * DB_NW);
  __syncthreads();

  // ---- warp w: rows w, w+8, ... (lane = column); the loads of all four
  // rows are issued together, in dependent rounds: codes and the rows'
  // stream offsets (lane q loads row q's, then shuffled); symbols; ll values
  // and recon(t-1) only for rows with a pinned pixel (and SL blocks)
  constexpr int NR = 32 / DB_NW;
  const int32_t* etab = sm.etab;
  int cd[NR];
  int64_t qo = 0, lo = 0;   // lane q < NR: offsets of row wid + DB_NW * q
  if (lane < NR) {
    const int i = min(wid + DB_NW * lane, nr - 1);
    const int64_t row = rowbase + r0 + i;
    qo = qd_row_off[row] + 2 * (int64_t)pre_nl[row * nchunks + bj];
  }
#pragma unroll
  for (int q = 0; q < NR; q++) {
    const int i = min(wid + DB_NW * q, nr - 1);
    cd[q] = (wid + DB_NW * q < nr && colok) ? __ldg(codes_t + (int64_t)(r0 + i) * W + j) : CODE_LOSSLESS;
  }
  uint32_t sy[NR];
  bool nlq[NR];
#pragma unroll
  for (int q = 0; q < NR; q++) {
    nlq[q] = colok && etab[cd[q] & 31] != 0;
    const unsigned bnl = __ballot_sync(FULL, nlq[q]);
    const int64_t qoff = __shfl_sync(FULL, qo, q);
    sy[q] = 0u;
    if (nlq[q]) {
      const int64_t k = qoff + 2 * __popc(bnl & lt);
      if (sizeof(SYM) == 2)
        sy[q] = __ldg(reinterpret_cast<const uint32_t*>(qd + k));
      else
        sy[q] = (uint32_t)qd[k] | ((uint32_t)qd[k + 1] << 16);
    }
  }
  int32_t lu[NR], lv[NR];
  int2 pp[NR];
  unsigned peu[NR], pev[NR];
  unsigned pinrows = 0;
#pragma unroll
  for (int q = 0; q < NR; q++) {
    const int i = wid + DB_NW * q;
    const bool rv = i < nr;
    const uint32_t syu = sy[q] & 0xffffu, syv = sy[q] >> 16;
    const bool eu = rv && ((colok && !nlq[q]) || (nlq[q] && syu == 0));
    const bool ev = rv && ((colok && !nlq[q]) || (nlq[q] && syv == 0));
    peu[q] = __ballot_sync(FULL, eu);
    pev[q] = __ballot_sync(FULL, ev);
    if (peu[q] | pev[q]) pinrows |= 1u << q;
  }
  if (pinrows && lane < NR) {
    const int i = min(wid + DB_NW * lane, nr - 1);
    const int64_t row = rowbase + r0 + i;
    lo = ll_row_off[row] + pre_ll[row * nchunks + bj];
  }
#pragma unroll
  for (int q = 0; q < NR; q++) {
    const int i = wid + DB_NW * q;
    lu[q] = 0;
    lv[q] = 0;
    const bool eu = (peu[q] >> lane) & 1u, ev = (pev[q] >> lane) & 1u;
    if ((pinrows >> q) & 1u) {
      int64_t lidx = __shfl_sync(FULL, lo, q) + __popc(peu[q] & lt) + __popc(pev[q] & lt);
      if (eu) { lu[q] = (int32_t)ll[lidx]; lidx++; }
      if (ev) lv[q] = (int32_t)ll[lidx];
    }
    pp[q] = (i < nr && has_prev && (sl_blk || eu || ev))
                ? __ldg(prev + (int64_t)(r0 + min(i, nr - 1)) * Wp + j)
                : make_int2(0, 0);
  }
  // per row: A (quantised pixels) or Z = recon - prev (pinned ones)
  uint32_t a[2][NR];
  uint32_t csum[2] = {0u, 0u};
  bool anyp[2] = {false, false}, notall[2] = {false, false};
  if (sl_blk) {
    // every pixel known: the SL predictions (two rows at a time so their
    // gathers overlap), recon, the float64 output, Z edges
    const TileSrc src{sm.pv, r0 - SLH, c0 - SLH, prev, Wp};
#pragma unroll
    for (int q0 = 0; q0 < NR; q0 += 2) {
      int64_t pu[2] = {0, 0}, pv[2] = {0, 0};
      bool slow[2] = {false, false}, need[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int q = q0 + h;
        const int i = min(wid + DB_NW * q, nr - 1);
        need[h] = wid + DB_NW * q < nr && nlq[q] &&
                  !(((peu[q] & pev[q]) >> lane) & 1u);
        if (__any_sync(FULL, need[h]))
          slow[h] = !sl_predict_rk2(src, H, W, r0 + i, j, p.cfl_x, p.cfl_y,
                                    p.d_max, &pu[h], &pv[h]);
      }
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int q = q0 + h;
        const int i = wid + DB_NW * q;
        if (i >= nr) break;   // warp-uniform
        if (slow[h] && need[h])
          sl_general(prev, Wp, H, W, r0 + i, j, p.cfl_x, p.cfl_y, p.d_max,
                     p.n_max, &pu[h], &pv[h]);
        const int64_t two_e = 2 * (int64_t)etab[cd[q] & 31];
        const bool eu = (peu[q] >> lane) & 1u, ev = (pev[q] >> lane) & 1u;
        const int64_t qu = (int64_t)(sy[q] & 0xffffu) - p.radius;
        const int64_t qv = (int64_t)(sy[q] >> 16) - p.radius;
        const int32_t ru = eu ? lu[q] : (int32_t)(pu[h] + qu * two_e);
        const int32_t rv = ev ? lv[q] : (int32_t)(pv[h] + qv * two_e);
        const int64_t pk = (int64_t)(r0 + i) * Wp + j;
        if (colok) {
          rec[pk] = make_int2(ru, rv);
          const int64_t ko = fbase + (int64_t)(r0 + i) * W + j;
          f64u[ko] = __dmul_rn((double)ru, inv_S);
          f64v[ko] = __dmul_rn((double)rv, inv_S);
          if (fixu) { fixu[ko] = ru; fixv[ko] = rv; }
        }
        const int32_t zu = ru - pp[q].x, zv = rv - pp[q].y;
        if (i == nr - 1) {
          bio.lb[blk * 32 + lane] = colok ? zu : 0;
          bio.lb[(nblk + blk) * 32 + lane] = colok ? zv : 0;
        }
        if (lane == ncl - 1) {
          bio.lr[blk * 32 + i] = zu;
          bio.lr[(nblk + blk) * 32 + i] = zv;
        }
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < NR; q++) {
      const int i = wid + DB_NW * q;
      a[0][q] = a[1][q] = 0u;
      if (i >= nr) continue;   // warp-uniform
      const bool eu = (peu[q] >> lane) & 1u, ev = (pev[q] >> lane) & 1u;
      const int64_t two_e = 2 * (int64_t)etab[cd[q] & 31];
      const int64_t qu = (int64_t)(sy[q] & 0xffffu) - p.radius;
      const int64_t qv = (int64_t)(sy[q] >> 16) - p.radius;
      a[0][q] = colok ? (eu ? (uint32_t)(lu[q] - pp[q].x) : (uint32_t)(qu * two_e)) : 0u;
      a[1][q] = colok ? (ev ? (uint32_t)(lv[q] - pp[q].y) : (uint32_t)(qv * two_e)) : 0u;
      anyp[0] |= eu;
      anyp[1] |= ev;
      notall[0] |= colok && !eu;
      notall[1] |= colok && !ev;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        csum[c] += a[c][q];
        const uint32_t rs = __reduce_add_sync(FULL, a[c][q]);
        if (lane == 0) sm.rowsum[c][i] = rs;
      }
    }
  }
  if (sl_blk) {
    if (tid < 64) {
      const int c = tid >> 5;
      if (lane >= nr) bio.lr[(c * nblk + blk) * 32 + lane] = 0;
      if (lane == 0) bio.cls[c * nblk + blk] = BS_KNOWN;
    }
    return;
  }
#pragma unroll
  for (int c = 0; c < 2; c++) {
    sm.colsum[c][wid][lane] = csum[c];
    if (__any_sync(FULL, anyp[c]) && lane == 0) atomicOr(&sm.anypin[c], 1);
    if (__any_sync(FULL, notall[c]) && lane == 0) atomicOr(&sm.notall[c], 1);
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const bool known = !sm.notall[c];
    const bool slow = !known && sm.anypin[c];
    uint32_t* pinp = c ? pin_v : pin_u;
    double* f64 = c ? f64v : f64u;
    int64_t* fix = c ? fixv : fixu;
    if (known || slow) {
#pragma unroll
      for (int q = 0; q < NR; q++) {
        const int i = wid + DB_NW * q;
        if (i >= nr) break;
        const int64_t pk = (int64_t)(r0 + i) * Wp + j;
        if (known) {
          // recon = the lossless / escaped value of every pixel
          const int32_t rv = c ? lv[q] : lu[q];
          if (colok) {
            recw[2 * pk + c] = rv;
            const int64_t ko = fbase + (int64_t)(r0 + i) * W + j;
            f64[ko] = __dmul_rn((double)rv, inv_S);
            if (fix) fix[ko] = rv;
          }
          if (i == nr - 1) bio.lb[(c * nblk + blk) * 32 + lane] = colok ? (int32_t)a[c][q] : 0;
          if (lane == ncl - 1) bio.lr[(c * nblk + blk) * 32 + i] = (int32_t)a[c][q];
        } else {
          if (colok) bio.a_w[c][pk] = (int32_t)a[c][q];
          if (lane == 0) pinp[(int64_t)(r0 + i) * nchunks + bj] = c ? pev[q] : peu[q];
        }
      }
    }
  }
  if (tid >= 64) return;
  const int c = tid >> 5;
  const bool known = !sm.notall[c];
  const bool anypin = sm.anypin[c] != 0;
  if (known) {
    if (lane >= nr) bio.lr[(c * nblk + blk) * 32 + lane] = 0;
    if (lane == 0) bio.cls[c * nblk + blk] = BS_KNOWN;
    return;
  }
  if (anypin) {
    if (lane == 0) bio.cls[c * nblk + blk] = BS_SLOW;
    return;
  }
  // REG: LB(j) = sum_{b<=j} colsum(b), LR(i) = sum_{a<=i} rowsum(a)
  uint32_t cs = 0u;
#pragma unroll
  for (int w = 0; w < DB_NW; w++) cs += sm.colsum[c][w][lane];
  uint32_t rs = lane < nr ? sm.rowsum[c][lane] : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t pc = __shfl_up_sync(FULL, cs, o);
    const uint32_t pr = __shfl_up_sync(FULL, rs, o);
    if (lane >= o) { cs += pc; rs += pr; }
  }
  bio.lb[(c * nblk + blk) * 32 + lane] = (int32_t)cs;
  bio.lr[(c * nblk + blk) * 32 + lane] = (int32_t)rs;
  if (lane == 0) bio.cls[c * nblk + blk] = BS_REG;
}

// true when the frame's usual blocks go through the fast kernel (a large
// frame of 16-bit symbols with 4-byte-aligned code rows)
template <typename SYM>
bool dec_block_split(const uint8_t* codes_t, const PrepParams& p) {
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  return sizeof(SYM) == 2 && nblk >= 1024 && (p.W & 3) == 0 &&
         ((uintptr_t)codes_t & 3) == 0;
}

// The usual blocks of a frame; needs nothing of frame t - 1, so the caller
// may run it ahead on a side stream.
template <typename SYM>
cudaError_t launch_dec_block_fast(const uint8_t* codes_t, const SYM* qd,
                                  const uint8_t* modes_t, bool has_prev,
                                  const int64_t* qd_row_off,
                                  const int32_t* pre_nl, const PrepParams& p,
                                  const BScanIO& bio, const int32_t* e_tab_dev,
                                  int* list, int* count, cudaStream_t st) {
  dec_block_fast_kernel<SYM><<<dim3(p.nbx, p.nby), 32 * DB_NW, 0, st>>>(
      codes_t, qd, has_prev ? modes_t : nullptr, qd_row_off, pre_nl, p, bio.lb,
      bio.lr, bio.cls, 0, e_tab_dev, list, count);
  return cudaGetLastError();
}

// The general kernel: the listed blocks (list != nullptr, after the fast
// kernel) or every block of the frame.
template <typename SYM>
cudaError_t launch_dec_block(const uint8_t* codes_t, const SYM* qd,
                             const int64_t* ll, const uint8_t* modes_t,
                             const int32_t* prev, int32_t* rec,
                             const int64_t* qd_row_off,
                             const int64_t* ll_row_off, const int32_t* pre_nl,
                             const int32_t* pre_ll, const PrepParams& p,
                             const BScanIO& bio, uint32_t* pin_u,
                             uint32_t* pin_v, double* f64u, double* f64v,
                             int64_t* fixu, int64_t* fixv, double inv_S,
                             const int* list, const int* count, int nsm,
                             cudaStream_t st) {
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  if (list) {
    const int64_t cap = (int64_t)nsm * DB_OCC;
    dec_block_kernel<SYM><<<(int)(nblk < cap ? nblk : cap), 32 * DB_NW, 0, st>>>(
        codes_t, qd, ll, modes_t, reinterpret_cast<const int2*>(prev),
        reinterpret_cast<int2*>(rec), qd_row_off, ll_row_off, pre_nl, pre_ll, p,
        bio, pin_u, pin_v, f64u, f64v, fixu, fixv, inv_S, list, count);
    return cudaGetLastError();
  }
  dec_block_kernel<SYM><<<dim3(p.nbx, p.nby), 32 * DB_NW, 0, st>>>(
      codes_t, qd, ll, modes_t, reinterpret_cast<const int2*>(prev),
      reinterpret_cast<int2*>(rec), qd_row_off, ll_row_off, pre_nl, pre_ll, p,
      bio, pin_u, pin_v, f64u, f64v, fixu, fixv, inv_S, nullptr, nullptr);
  return cudaGetLastError();
}

template bool dec_block_split<uint16_t>(const uint8_t*, const PrepParams&);
template cudaError_t launch_dec_block_fast<uint16_t>(
    const uint8_t*, const uint16_t*, const uint8_t*, bool, const int64_t*,
    const int32_t*, const PrepParams&, const BScanIO&, const int32_t*, int*,
    int*, cudaStream_t);
template cudaError_t launch_dec_block<uint16_t>(
    const uint8_t*, const uint16_t*, const int64_t*, const uint8_t*,
    const int32_t*, int32_t*, const int64_t*, const int64_t*, const int32_t*,
    const int32_t*, const PrepParams&, const BScanIO&, uint32_t*, uint32_t*,
    double*, double*, int64_t*, int64_t*, double, const int*, const int*, int,
    cudaStream_t);

}  // namespace vfcp
