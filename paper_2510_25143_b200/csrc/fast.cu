// Frame-parallel preparation kernels + the chain wavefront (chain.cuh).
//
// Per frame t the compress path runs
//   enc_prep_kernel  one warp per 32x32 block: MoP mode selection
//                    (mop.py:68-151: Lorenzo trial with block-local
//                    write-back, semi-Lagrangian trial at the stride samples,
//                    first-touch entropy, theta gate), then every pixel that
//                    does not need its reconstructed neighbours: lossless
//                    pins, semi-Lagrangian pixels (prediction, symbol, err)
//                    and, for Lorenzo pixels, R0 = orig - Lorenzo(orig, prev)
//                    for the error-form chain;
//   chain_kernel<ENC>  the raster recurrence (chain.cuh);
// and the decompress path
//   dec_prep_kernel  one warp per 32x32 block: pins (lossless, escapes,
//                    semi-Lagrangian pixels) and A = Pd + (sym-radius)*2e;
//   chain_kernel<DEC>.
// The reconstruction of frame t-1 is read as orig + err (encoder) or the int
// recon frame (decoder).  Stream positions come from per-(row, chunk) prefix
// counts, so any block can place its symbols and ll values.
#include "chain.cuh"

namespace vfcp {

// ----------------------------------------------------------- prefix counts
// Per frame row: for each 32-column chunk, the number of non-lossless
// pixels (and, for the decoder, ll entries) before it in the row.
// One warp per row.
template <typename SYM>
__global__ void chunk_prefix_kernel(const uint8_t* __restrict__ codes,
                                    const SYM* __restrict__ qd,
                                    const int64_t* __restrict__ qd_row_off,
                                    int64_t nrows, int W, int nchunks,
                                    int64_t tau, int32_t* __restrict__ pre_nl,
                                    int32_t* __restrict__ pre_ll) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int64_t rb = row * W;
  int32_t nl_run = 0, ll_run = 0;
  int64_t qp = qd ? qd_row_off[row] : 0;
  for (int x = 0; x < nchunks; x++) {
    const int j = 32 * x + lane;
    bool nl = false, ll0 = false;
    if (j < W) {
      const int c = codes[rb + j];
      nl = !(c >= CODE_LOSSLESS || tau <= 0 || (tau >> c) == 0);
    }
    const unsigned b = __ballot_sync(0xffffffffu, nl);
    int esc = 0;
    if (qd && nl) {
      const int64_t q = qp + 2 * __popc(b & ((1u << lane) - 1u));
      esc = (qd[q] == 0) + (qd[q + 1] == 0);
    }
    if (j < W && !nl) ll0 = true;
    int cnt = esc + (ll0 ? 2 : 0);
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      pre_nl[row * nchunks + x] = nl_run;
      if (pre_ll) pre_ll[row * nchunks + x] = ll_run;
    }
    nl_run += __popc(b);
    ll_run += cnt;
    qp += 2 * __popc(b);
  }
}

// ------------------------------------------------------ 2D value sources
// frame t-1 reconstruction seen by the encoder: orig fixed + err
template <typename F>
struct EncPrev {
  const F* o;        // frame t-1 input (pitch W)
  const int32_t* e;  // frame t-1 err (pitch Wp)
  double S;
  int W, Wp;
  __device__ __forceinline__ int64_t ival(int i, int j) const {
    return (int64_t)load_fixed(o, (int64_t)i * W + j, S) + e[(int64_t)i * Wp + j];
  }
  __device__ __forceinline__ double operator()(int i, int j) const {
    return (double)ival(i, j);
  }
};
struct DecPrev {
  const int32_t* r;  // frame t-1 recon (pitch Wp)
  int Wp;
  __device__ __forceinline__ int64_t ival(int i, int j) const {
    return r[(int64_t)i * Wp + j];
  }
  __device__ __forceinline__ double operator()(int i, int j) const {
    return (double)r[(int64_t)i * Wp + j];
  }
};

// predictors.py:33-59 with a 2D source (shared weights for u and v)
template <typename Src>
__device__ __forceinline__ void bilinear2(const Src& su, const Src& sv, int H,
                                          int W, double i_f, double j_f,
                                          int64_t* pu, int64_t* pv) {
  if (i_f < 0.0) i_f = 0.0;
  else if (i_f > (double)(H - 1)) i_f = (double)(H - 1);
  if (j_f < 0.0) j_f = 0.0;
  else if (j_f > (double)(W - 1)) j_f = (double)(W - 1);
  int i0 = (int)floor(i_f), j0 = (int)floor(j_f);
  if (i0 > H - 1) i0 = H - 1;
  if (j0 > W - 1) j0 = W - 1;
  const int i1 = i0 + 1 < H - 1 ? i0 + 1 : H - 1;
  const int j1 = j0 + 1 < W - 1 ? j0 + 1 : W - 1;
  const double a = __dsub_rn(i_f, (double)i0), b = __dsub_rn(j_f, (double)j0);
  const double oma = __dsub_rn(1.0, a), omb = __dsub_rn(1.0, b);
  const double w00 = __dmul_rn(oma, omb), w01 = __dmul_rn(oma, b);
  const double w10 = __dmul_rn(a, omb), w11 = __dmul_rn(a, b);
  double vu = __dmul_rn(w00, su(i0, j0));
  vu = __dadd_rn(vu, __dmul_rn(w01, su(i0, j1)));
  vu = __dadd_rn(vu, __dmul_rn(w10, su(i1, j0)));
  vu = __dadd_rn(vu, __dmul_rn(w11, su(i1, j1)));
  double vv = __dmul_rn(w00, sv(i0, j0));
  vv = __dadd_rn(vv, __dmul_rn(w01, sv(i0, j1)));
  vv = __dadd_rn(vv, __dmul_rn(w10, sv(i1, j0)));
  vv = __dadd_rn(vv, __dmul_rn(w11, sv(i1, j1)));
  *pu = rha_d(vu);
  *pv = rha_d(vv);
}

// predictors.py:76-108 + the prediction sample at the departure point
template <typename Src>
__device__ __forceinline__ void sl_predict2(const Src& su, const Src& sv,
                                            int H, int W, int i, int j,
                                            double cfl_x, double cfl_y,
                                            double d_max, int n_max,
                                            int64_t* pu, int64_t* pv) {
  const double u0 = su(i, j), v0 = sv(i, j);
  const double ax = __dmul_rn(fabs(u0), cfl_x), ay = __dmul_rn(fabs(v0), cfl_y);
  const double d_inf = ay > ax ? ay : ax;
  double fi, fj;
  if (d_inf <= d_max) {
    const double ih = __dsub_rn((double)i, __dmul_rn(__dmul_rn(0.5, v0), cfl_y));
    const double jh = __dsub_rn((double)j, __dmul_rn(__dmul_rn(0.5, u0), cfl_x));
    int64_t um, vm;
    bilinear2(su, sv, H, W, ih, jh, &um, &vm);
    fi = __dsub_rn((double)i, __dmul_rn((double)vm, cfl_y));
    fj = __dsub_rn((double)j, __dmul_rn((double)um, cfl_x));
  } else {
    int64_t n = (int64_t)ceil(__ddiv_rn(d_inf, d_max));
    if (n > n_max) n = n_max;
    const double dn = (double)n;
    fi = (double)i;
    fj = (double)j;
    for (int64_t s = 0; s < n; s++) {
      int64_t us, vs;
      bilinear2(su, sv, H, W, fi, fj, &us, &vs);
      fi = __dsub_rn(fi, __ddiv_rn(__dmul_rn((double)vs, cfl_y), dn));
      fj = __dsub_rn(fj, __ddiv_rn(__dmul_rn((double)us, cfl_x), dn));
      if (fi < 0.0) fi = 0.0;
      else if (fi > (double)(H - 1)) fi = (double)(H - 1);
      if (fj < 0.0) fj = 0.0;
      else if (fj > (double)(W - 1)) fj = (double)(W - 1);
    }
  }
  bilinear2(su, sv, H, W, fi, fj, pu, pv);
}

// ------------------------------------------------ first-touch block entropy
// mop.py:118-138.  samp[sp] = |idx| of sample sp (sequence order: raster
// (i, j), u then v) or -1 for an overflow sample.
constexpr int ETB = 1024;
__device__ double block_rate(const int32_t* samp, int ns, int32_t* first,
                             int32_t* cnt, const double* log2tab, double lam,
                             double rmeta, int lane) {
  int n_ok = 0, lp = 0;
  for (int sp = lane; sp < ns; sp += 32) {
    const int a = samp[sp];
    if (a < 0) { lp++; continue; }
    n_ok++;
    if (a < ETB) { atomicMin(first + a, sp); atomicAdd(cnt + a, 1); }
  }
  for (int o = 16; o; o >>= 1) {
    n_ok += __shfl_xor_sync(0xffffffffu, n_ok, o);
    lp += __shfl_xor_sync(0xffffffffu, lp, o);
  }
  __syncwarp();
  double acc = 0.0;
  for (int c = 0; c < ns; c += 32) {
    const int sp = c + lane;
    bool ft = false;
    int h = 0;
    if (sp < ns) {
      const int a = samp[sp];
      if (a >= 0 && a < ETB) {
        ft = first[a] == sp;
        h = cnt[a];
      } else if (a >= ETB) {
        ft = true;
        for (int q = 0; q < sp; q++)
          if (samp[q] == a) { ft = false; break; }
        if (ft)
          for (int q = 0; q < ns; q++) h += samp[q] == a;
      }
    }
    const double term = ft ? __dmul_rn((double)h, log2tab[h]) : 0.0;
    unsigned bal = __ballot_sync(0xffffffffu, ft);
    while (bal) {
      const int b = __ffs(bal) - 1;
      bal &= bal - 1;
      acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, term, b));
    }
  }
  __syncwarp();
  for (int sp = lane; sp < ns; sp += 32) {
    const int a = samp[sp];
    if (a >= 0 && a < ETB) { first[a] = 0x7fffffff; cnt[a] = 0; }
  }
  __syncwarp();
  double h0 = 0.0;
  if (n_ok > 0) h0 = __dsub_rn(log2tab[n_ok], __ddiv_rn(acc, (double)n_ok));
  if (n_ok + lp > 0)
    return __dadd_rn(__dadd_rn(h0, __ddiv_rn(__dmul_rn(lam, (double)lp),
                                             (double)(n_ok + lp))),
                     rmeta);
  return rmeta;
}


// ---------------------------------------------------------- encoder prep
struct EncPrepSmem {
  // R0 tile [comp][row][col]; row stride 32 keeps both the column-wise
  // writes and the trial's anti-diagonal reads bank-conflict free
  int32_t r0[2][32][32];
  int32_t samp[512];
  int32_t first[ETB];
  int32_t cnt[ETB];
};

template <typename F>
__global__ void __launch_bounds__(128)
enc_prep_kernel(const F* __restrict__ u, const F* __restrict__ v,
                const uint8_t* __restrict__ codes,
                const int32_t* __restrict__ err_prev_u,
                const int32_t* __restrict__ err_prev_v,
                const int64_t* __restrict__ qd_row_off,
                const int32_t* __restrict__ pre_nl, PrepParams p,
                const double* __restrict__ log2tab,
                uint8_t* __restrict__ modes_t, int32_t* __restrict__ a0,
                int32_t* __restrict__ a1, uint32_t* __restrict__ pin_u,
                uint32_t* __restrict__ pin_v, uint32_t* __restrict__ nlw,
                uint32_t* __restrict__ symw, uint16_t* __restrict__ qd,
                int32_t* __restrict__ row_ll, int* __restrict__ overflow,
                uint8_t* __restrict__ codes_p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  EncPrepSmem& sm = reinterpret_cast<EncPrepSmem*>(smem_raw)[wid];
  const int blk = blockIdx.x * 4 + wid;
  if (blk >= p.nbx * p.nby) return;
  const int bi = blk / p.nbx, bj = blk - bi * p.nbx;
  const int H = p.H, W = p.W, Wp = p.Wp;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const int j = c0 + lane;
  const bool colok = lane < ncl;
  const int64_t HW = (int64_t)H * W;
  const F* uo = u + (int64_t)p.t * HW;
  const F* vo = v + (int64_t)p.t * HW;
  const bool has_prev = p.t > 0;
  const EncPrev<F> su{u + (int64_t)(p.t - 1) * HW, err_prev_u, p.S, W, Wp};
  const EncPrev<F> sv{v + (int64_t)(p.t - 1) * HW, err_prev_v, p.S, W, Wp};
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;

  // ---- R0 for the block (lane = column), Lorenzo on orig and on frame t-1
  auto orig = [&](const F* f, int i, int jj) -> int64_t {
    return (i >= 0 && jj >= 0) ? (int64_t)load_fixed(f, (int64_t)i * W + jj, p.S) : 0;
  };
  auto prevv = [&](const EncPrev<F>& s, int i, int jj) -> int64_t {
    return (has_prev && i >= 0 && jj >= 0) ? s.ival(i, jj) : 0;
  };
  int64_t oU_u = 0, oU_v = 0, pU_u = 0, pU_v = 0;     // row above, column j
  int64_t oUL_u = 0, oUL_v = 0, pUL_u = 0, pUL_v = 0; // lane 0: (r-1, c0-1)
  if (colok && r0 > 0) {
    oU_u = orig(uo, r0 - 1, j); oU_v = orig(vo, r0 - 1, j);
    pU_u = prevv(su, r0 - 1, j); pU_v = prevv(sv, r0 - 1, j);
  }
  if (lane == 0 && r0 > 0 && c0 > 0) {
    oUL_u = orig(uo, r0 - 1, c0 - 1); oUL_v = orig(vo, r0 - 1, c0 - 1);
    pUL_u = prevv(su, r0 - 1, c0 - 1); pUL_v = prevv(sv, r0 - 1, c0 - 1);
  }
  bool ovf = false;
  for (int r = 0; r < nr; r++) {
    const int i = r0 + r;
    int64_t o_u = 0, o_v = 0, pp_u = 0, pp_v = 0, oL_u = 0, oL_v = 0,
            pL_u = 0, pL_v = 0;
    if (colok) {
      o_u = orig(uo, i, j); o_v = orig(vo, i, j);
      pp_u = prevv(su, i, j); pp_v = prevv(sv, i, j);
    }
    if (lane == 0 && c0 > 0) {
      oL_u = orig(uo, i, c0 - 1); oL_v = orig(vo, i, c0 - 1);
      pL_u = prevv(su, i, c0 - 1); pL_v = prevv(sv, i, c0 - 1);
    }
    // left neighbours via shuffles (lane 0: the column left of the block)
    int64_t tl_ou = __shfl_up_sync(FULL, o_u, 1), tl_ov = __shfl_up_sync(FULL, o_v, 1);
    int64_t tl_pu = __shfl_up_sync(FULL, pp_u, 1), tl_pv = __shfl_up_sync(FULL, pp_v, 1);
    int64_t tul_ou = __shfl_up_sync(FULL, oU_u, 1), tul_ov = __shfl_up_sync(FULL, oU_v, 1);
    int64_t tul_pu = __shfl_up_sync(FULL, pU_u, 1), tul_pv = __shfl_up_sync(FULL, pU_v, 1);
    if (lane == 0) {
      tl_ou = oL_u; tl_ov = oL_v; tl_pu = pL_u; tl_pv = pL_v;
      tul_ou = oUL_u; tul_ov = oUL_v; tul_pu = pUL_u; tul_pv = pUL_v;
      oUL_u = oL_u; oUL_v = oL_v; pUL_u = pL_u; pUL_v = pL_v;
    }
    // R0 = orig - Lorenzo(orig, prev) with zero padding outside the frame
    const int64_t R_u = o_u - (oU_u + tl_ou - tul_ou) - (pp_u - pU_u - tl_pu + tul_pu);
    const int64_t R_v = o_v - (oU_v + tl_ov - tul_ov) - (pp_v - pU_v - tl_pv + tul_pv);
    ovf |= colok && (R_u >= 2147483647LL || R_u <= -2147483647LL ||
                     R_v >= 2147483647LL || R_v <= -2147483647LL);
    sm.r0[0][r][lane] = (int32_t)R_u;
    sm.r0[1][r][lane] = (int32_t)R_v;
    oU_u = o_u; oU_v = o_v; pU_u = pp_u; pU_v = pp_v;
  }
  if (__any_sync(FULL, ovf) && lane == 0) atomicOr(overflow, 1);
  __syncwarp();

  // ---- MoP (mop.py:79-151) for frames t >= 1
  int mode = p.force_sl;
  if (p.mop) {
    const int nsx = (ncl + p.stride - 1) / p.stride;
    const int nsy = (nr + p.stride - 1) / p.stride;
    const int ns = 2 * nsx * nsy;
    for (int k = lane; k < ETB; k += 32) { sm.first[k] = 0x7fffffff; sm.cnt[k] = 0; }
    const int64_t tau = p.tau, two_tau = 2 * tau;
    const double inv = 1.0 / (double)two_tau;
    // Lorenzo trial: error form with uniform e = tau', block-local errors
    {
      int64_t eL[2] = {0, 0}, eUp[2] = {0, 0}, eLast[2] = {0, 0};
      const int i = lane;   // lane = row of the block
      for (int s = 0; s < ncl + 31; s++) {
        const int jj = s - lane;
        int64_t eU[2];
#pragma unroll
        for (int comp = 0; comp < 2; comp++) {
          const int64_t x = __shfl_up_sync(FULL, eLast[comp], 1);
          eU[comp] = lane == 0 ? 0 : x;
        }
        const bool act = i < nr && jj >= 0 && jj < ncl;
        if (act) {
          const bool smp = (i % p.stride == 0) && (jj % p.stride == 0);
#pragma unroll
          for (int comp = 0; comp < 2; comp++) {
            const int64_t d = (i > 0 ? eU[comp] : 0) + (jj > 0 ? eL[comp] : 0) -
                              ((i > 0 && jj > 0) ? eUp[comp] : 0);
            const int64_t x = (int64_t)sm.r0[comp][i][jj] - d;
            const int64_t q = quant_rha(x, tau, inv);
            const bool ok = q > -p.radius && q < p.radius;
            const int64_t err = ok ? q * two_tau - x : 0;
            eL[comp] = err;
            eLast[comp] = err;
            if (smp)
              sm.samp[2 * ((i / p.stride) * nsx + jj / p.stride) + comp] =
                  ok ? (int32_t)(q < 0 ? -q : q) : -1;
          }
        }
#pragma unroll
        for (int comp = 0; comp < 2; comp++) eUp[comp] = eU[comp];
      }
    }
    __syncwarp();
    const double r_lor = block_rate(sm.samp, ns, sm.first, sm.cnt, log2tab,
                                    p.lam, p.rmeta, lane);
    // SL trial at the stride samples
    for (int sidx = lane; sidx < nsx * nsy; sidx += 32) {
      const int si = sidx / nsx, sj = sidx - si * nsx;
      const int i = r0 + si * p.stride, jj = c0 + sj * p.stride;
      int64_t pr_u, pr_v;
      sl_predict2(su, sv, H, W, i, jj, p.cfl_x, p.cfl_y, p.d_max, p.n_max,
                  &pr_u, &pr_v);
      const int64_t ru = (int64_t)load_fixed(uo, (int64_t)i * W + jj, p.S) - pr_u;
      const int64_t rv = (int64_t)load_fixed(vo, (int64_t)i * W + jj, p.S) - pr_v;
      const int64_t qu = quant_rha(ru, tau, inv), qv = quant_rha(rv, tau, inv);
      sm.samp[2 * sidx] = (qu > -p.radius && qu < p.radius) ? (int32_t)(qu < 0 ? -qu : qu) : -1;
      sm.samp[2 * sidx + 1] = (qv > -p.radius && qv < p.radius) ? (int32_t)(qv < 0 ? -qv : qv) : -1;
    }
    __syncwarp();
    const double r_sl = block_rate(sm.samp, ns, sm.first, sm.cnt, log2tab,
                                   p.lam, p.rmeta, lane);
    mode = (r_lor > 0.0 && __ddiv_rn(__dsub_rn(r_lor, r_sl), r_lor) > p.theta) ? 1 : 0;
  }
  if (modes_t && lane == 0) modes_t[blk] = (uint8_t)mode;

  // ---- per-pixel outputs (lane = column)
  const int nchunks = p.nchunks;
  int ll_cnt_dummy = 0;
  (void)ll_cnt_dummy;
  for (int r = 0; r < nr; r++) {
    const int i = r0 + r;
    const int64_t row = (int64_t)p.t * H + i;
    const int cd = colok ? codes[(int64_t)p.t * HW + (int64_t)i * W + j] : CODE_LOSSLESS;
    const int64_t e = p.lad.e[cd];
    const bool nl = colok && e != 0;
    const unsigned bnl = __ballot_sync(FULL, nl);
    const bool sl = nl && mode == 1;
    int32_t val_u = 0, val_v = 0;
    bool pu = !nl, pv = !nl;     // lossless pixels are pinned (err 0)
    int nll = (colok && !nl) ? 2 : 0;
    if (sl) {
      int64_t pr_u, pr_v;
      sl_predict2(su, sv, H, W, i, j, p.cfl_x, p.cfl_y, p.d_max, p.n_max,
                  &pr_u, &pr_v);
      const int64_t two_e = 2 * e;
      const double inv = p.lad.inv2e[cd];
      const int64_t ou = load_fixed(uo, (int64_t)i * W + j, p.S);
      const int64_t ov = load_fixed(vo, (int64_t)i * W + j, p.S);
      const int64_t qu = quant_rha(ou - pr_u, e, inv), qv = quant_rha(ov - pr_v, e, inv);
      const bool oku = qu > -p.radius && qu < p.radius;
      const bool okv = qv > -p.radius && qv < p.radius;
      val_u = oku ? (int32_t)(pr_u + qu * two_e - ou) : 0;
      val_v = okv ? (int32_t)(pr_v + qv * two_e - ov) : 0;
      const uint32_t syu = oku ? (uint32_t)(qu + p.radius) : 0u;
      const uint32_t syv = okv ? (uint32_t)(qv + p.radius) : 0u;
      const int64_t pos = qd_row_off[row] +
                          2 * ((int64_t)pre_nl[row * nchunks + bj] + __popc(bnl & lt));
      *reinterpret_cast<uint32_t*>(qd + pos) = syu | (syv << 16);
      pu = pv = true;
      nll = (oku ? 0 : 1) + (okv ? 0 : 1);
    } else if (nl) {
      val_u = sm.r0[0][r][lane];
      val_v = sm.r0[1][r][lane];
    }
    const unsigned b_pu = __ballot_sync(FULL, colok && pu);
    const unsigned b_pv = __ballot_sync(FULL, colok && pv);
    const unsigned b_sw = __ballot_sync(FULL, nl && !sl);
    int tot = nll;
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    const int64_t pr = (int64_t)i * Wp + j;
    if (colok) { a0[pr] = val_u; a1[pr] = val_v; }
    codes_p[pr] = (uint8_t)cd;
    if (lane == 0) {
      const int64_t pb = (int64_t)i * nchunks + bj;
      pin_u[pb] = b_pu;
      pin_v[pb] = b_pv;
      nlw[pb] = bnl;
      symw[pb] = b_sw;
      if (tot) atomicAdd(row_ll + row, tot);
    }
  }
}

// ---------------------------------------------------------- decoder prep
template <typename SYM>
__global__ void __launch_bounds__(128)
dec_prep_kernel(const uint8_t* __restrict__ codes, const SYM* __restrict__ qd,
                const int64_t* __restrict__ ll,
                const uint8_t* __restrict__ modes_t,
                const int32_t* __restrict__ rec_prev_u,
                const int32_t* __restrict__ rec_prev_v,
                const int64_t* __restrict__ qd_row_off,
                const int64_t* __restrict__ ll_row_off,
                const int32_t* __restrict__ pre_nl,
                const int32_t* __restrict__ pre_ll, PrepParams p,
                int32_t* __restrict__ a0, int32_t* __restrict__ a1,
                uint32_t* __restrict__ pin_u, uint32_t* __restrict__ pin_v) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int blk = blockIdx.x * 4 + wid;
  if (blk >= p.nbx * p.nby) return;
  const int bi = blk / p.nbx, bj = blk - bi * p.nbx;
  const int H = p.H, W = p.W, Wp = p.Wp;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const int j = c0 + lane;
  const bool colok = lane < ncl;
  const int64_t HW = (int64_t)H * W;
  const bool has_prev = p.t > 0;
  const DecPrev su{rec_prev_u, Wp}, sv{rec_prev_v, Wp};
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  const bool sl_blk = has_prev && modes_t && modes_t[blk] == 1;
  auto prevv = [&](const DecPrev& s, int i, int jj) -> uint32_t {
    return (has_prev && i >= 0 && jj >= 0) ? (uint32_t)s.ival(i, jj) : 0u;
  };
  uint32_t pU_u = 0, pU_v = 0, pUL_u = 0, pUL_v = 0;
  if (colok && r0 > 0) { pU_u = prevv(su, r0 - 1, j); pU_v = prevv(sv, r0 - 1, j); }
  if (lane == 0 && r0 > 0 && c0 > 0) {
    pUL_u = prevv(su, r0 - 1, c0 - 1);
    pUL_v = prevv(sv, r0 - 1, c0 - 1);
  }
  const int nchunks = p.nchunks;
  for (int r = 0; r < nr; r++) {
    const int i = r0 + r;
    const int64_t row = (int64_t)p.t * H + i;
    uint32_t pp_u = 0, pp_v = 0, pL_u = 0, pL_v = 0;
    if (colok) { pp_u = prevv(su, i, j); pp_v = prevv(sv, i, j); }
    if (lane == 0 && c0 > 0) { pL_u = prevv(su, i, c0 - 1); pL_v = prevv(sv, i, c0 - 1); }
    uint32_t tl_u = __shfl_up_sync(FULL, pp_u, 1), tl_v = __shfl_up_sync(FULL, pp_v, 1);
    uint32_t tul_u = __shfl_up_sync(FULL, pU_u, 1), tul_v = __shfl_up_sync(FULL, pU_v, 1);
    if (lane == 0) {
      tl_u = pL_u; tl_v = pL_v; tul_u = pUL_u; tul_v = pUL_v;
      pUL_u = pL_u; pUL_v = pL_v;
    }
    const int cd = colok ? codes[(int64_t)p.t * HW + (int64_t)i * W + j] : CODE_LOSSLESS;
    const int64_t e = p.lad.e[cd];
    const bool nl = colok && e != 0;
    const unsigned bnl = __ballot_sync(FULL, nl);
    int64_t syu = 0, syv = 0;
    if (nl) {
      const int64_t q = qd_row_off[row] +
                        2 * ((int64_t)pre_nl[row * nchunks + bj] + __popc(bnl & lt));
      syu = qd[q];
      syv = qd[q + 1];
    }
    const bool eu = (colok && !nl) || (nl && syu == 0);
    const bool ev = (colok && !nl) || (nl && syv == 0);
    const unsigned b_eu = __ballot_sync(FULL, eu);
    const unsigned b_ev = __ballot_sync(FULL, ev);
    int64_t lidx = ll_row_off[row] + pre_ll[row * nchunks + bj] +
                   __popc(b_eu & lt) + __popc(b_ev & lt);
    const int64_t two_e = 2 * e;
    const int64_t qu = syu - p.radius, qv = syv - p.radius;
    uint32_t val_u = (pp_u - pU_u - tl_u + tul_u) + (uint32_t)(qu * two_e);
    uint32_t val_v = (pp_v - pU_v - tl_v + tul_v) + (uint32_t)(qv * two_e);
    const bool sl = nl && sl_blk;
    if (sl) {
      int64_t pr_u, pr_v;
      sl_predict2(su, sv, H, W, i, j, p.cfl_x, p.cfl_y, p.d_max, p.n_max,
                  &pr_u, &pr_v);
      val_u = (uint32_t)(pr_u + qu * two_e);
      val_v = (uint32_t)(pr_v + qv * two_e);
    }
    if (eu) { val_u = (uint32_t)ll[lidx]; lidx++; }
    if (ev) val_v = (uint32_t)ll[lidx];
    const unsigned b_pu = __ballot_sync(FULL, colok && (eu || sl));
    const unsigned b_pv = __ballot_sync(FULL, colok && (ev || sl));
    const int64_t pr = (int64_t)i * Wp + j;
    if (colok) { a0[pr] = (int32_t)val_u; a1[pr] = (int32_t)val_v; }
    if (lane == 0) {
      const int64_t pb = (int64_t)i * nchunks + bj;
      pin_u[pb] = b_pu;
      pin_v[pb] = b_pv;
    }
    pU_u = pp_u; pU_v = pp_v;
  }
}

// ------------------------------------------------------------ launchers
template <typename SYM>
cudaError_t launch_chunk_prefix(const uint8_t* codes, const SYM* qd,
                                const int64_t* qd_row_off, int64_t nrows,
                                int W, int nchunks, int64_t tau,
                                int32_t* pre_nl, int32_t* pre_ll,
                                cudaStream_t st) {
  chunk_prefix_kernel<SYM><<<(unsigned)((nrows + 7) / 8), 256, 0, st>>>(
      codes, qd, qd_row_off, nrows, W, nchunks, tau, pre_nl, pre_ll);
  return cudaGetLastError();
}

template <typename F>
cudaError_t launch_enc_prep(const F* u, const F* v, const uint8_t* codes,
                            const int32_t* eu, const int32_t* ev,
                            const int64_t* qd_row_off, const int32_t* pre_nl,
                            const PrepParams& p, const double* log2tab,
                            uint8_t* modes_t, int32_t* a0, int32_t* a1,
                            uint32_t* pin_u, uint32_t* pin_v, uint32_t* nlw,
                            uint32_t* symw, uint16_t* qd, int32_t* row_ll,
                            int* overflow, uint8_t* codes_p, cudaStream_t st) {
  const int nblk = p.nbx * p.nby;
  const size_t smem = 4 * sizeof(EncPrepSmem);
  cudaError_t ce = cudaFuncSetAttribute(
      enc_prep_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)smem);
  if (ce != cudaSuccess) return ce;
  enc_prep_kernel<F><<<(nblk + 3) / 4, 128, smem, st>>>(
      u, v, codes, eu, ev, qd_row_off, pre_nl, p, log2tab, modes_t, a0, a1,
      pin_u, pin_v, nlw, symw, qd, row_ll, overflow, codes_p);
  return cudaGetLastError();
}

template <typename SYM>
cudaError_t launch_dec_prep(const uint8_t* codes, const SYM* qd,
                            const int64_t* ll, const uint8_t* modes_t,
                            const int32_t* ru, const int32_t* rv,
                            const int64_t* qd_row_off,
                            const int64_t* ll_row_off, const int32_t* pre_nl,
                            const int32_t* pre_ll, const PrepParams& p,
                            int32_t* a0, int32_t* a1, uint32_t* pin_u,
                            uint32_t* pin_v, cudaStream_t st) {
  const int nblk = p.nbx * p.nby;
  dec_prep_kernel<SYM><<<(nblk + 3) / 4, 128, 0, st>>>(
      codes, qd, ll, modes_t, ru, rv, qd_row_off, ll_row_off, pre_nl, pre_ll,
      p, a0, a1, pin_u, pin_v);
  return cudaGetLastError();
}

__global__ void widen_frame_kernel(const int32_t* __restrict__ ru,
                                   const int32_t* __restrict__ rv, int H,
                                   int W, int Wp, int64_t* __restrict__ fu,
                                   int64_t* __restrict__ fv) {
  const int64_t n = (int64_t)H * W;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / W, j = k - i * W;
    fu[k] = ru[i * Wp + j];
    fv[k] = rv[i * Wp + j];
  }
}

cudaError_t launch_widen_frame(const int32_t* ru, const int32_t* rv, int H,
                               int W, int Wp, int64_t* fu, int64_t* fv,
                               cudaStream_t st) {
  widen_frame_kernel<<<1184, 256, 0, st>>>(ru, rv, H, W, Wp, fu, fv);
  return cudaGetLastError();
}

template <bool ENC>
cudaError_t launch_chain(const ChainIO& io, int nsm, cudaStream_t st) {
  const size_t smem = sizeof(ChainSmem<ENC>);
  cudaError_t e = cudaFuncSetAttribute(
      chain_kernel<ENC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = 64 * chain_pairs(ENC);
  int occ = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chain_kernel<ENC>,
                                                    threads, smem);
  if (e != cudaSuccess) return e;
  const int ntask = chain_ntask(ENC, io.H);
  chain_kernel<ENC><<<min(max(occ, 1) * nsm, ntask), threads, smem, st>>>(io);
  return cudaGetLastError();
}

template cudaError_t launch_chunk_prefix<uint16_t>(const uint8_t*,
                                                   const uint16_t*,
                                                   const int64_t*, int64_t,
                                                   int, int, int64_t,
                                                   int32_t*, int32_t*,
                                                   cudaStream_t);
template cudaError_t launch_enc_prep<float>(
    const float*, const float*, const uint8_t*, const int32_t*,
    const int32_t*, const int64_t*, const int32_t*, const PrepParams&,
    const double*, uint8_t*, int32_t*, int32_t*, uint32_t*, uint32_t*,
    uint32_t*, uint32_t*, uint16_t*, int32_t*, int*, uint8_t*, cudaStream_t);
template cudaError_t launch_enc_prep<double>(
    const double*, const double*, const uint8_t*, const int32_t*,
    const int32_t*, const int64_t*, const int32_t*, const PrepParams&,
    const double*, uint8_t*, int32_t*, int32_t*, uint32_t*, uint32_t*,
    uint32_t*, uint32_t*, uint16_t*, int32_t*, int*, uint8_t*, cudaStream_t);
template cudaError_t launch_dec_prep<uint16_t>(
    const uint8_t*, const uint16_t*, const int64_t*, const uint8_t*,
    const int32_t*, const int32_t*, const int64_t*, const int64_t*,
    const int32_t*, const int32_t*, const PrepParams&, int32_t*, int32_t*,
    uint32_t*, uint32_t*, cudaStream_t);
template cudaError_t launch_chain<true>(const ChainIO&, int, cudaStream_t);
template cudaError_t launch_chain<false>(const ChainIO&, int, cudaStream_t);

}  // namespace vfcp
