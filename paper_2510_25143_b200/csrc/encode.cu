// Prediction, mode selection and quantisation (compress), frame by frame.
//
//   mop_kernel      <- mop.py:68-151 _score_frame / select_modes
//   encode_kernel   <- codec.py:118-164 _encode_frame
//   ll_write_kernel <- the ll appends of codec.py:129-131,155-158
//
// encode_kernel keeps the reference's raster-order Lorenzo recurrence exactly
// by an anti-diagonal wavefront: one warp owns a 32-row strip (lane = row)
// and sweeps the columns skewed by one column per lane, so at every step a
// lane's up / left / up-left neighbours are final.  Strips are chained in
// row order through a boundary row in global memory plus a progress counter;
// strips are handed out by an atomic ticket so a strip only ever waits on a
// strip that is already resident.
#include "common.cuh"

namespace vfcp {


// -------------------------------------------------------------- MoP
// One warp per block.  smem per warp: nsamp int32 sample values (|idx| or
// -1 for an overflow sample) + TB-entry first-touch/count tables + one
// row of trial errors for blocks taller than 32.
constexpr int TB = 1024;

template <typename F, typename I>
__global__ void mop_kernel(const F* __restrict__ u, const F* __restrict__ v,
                           const I* __restrict__ up, const I* __restrict__ vp,
                           FrameParams p, const double* __restrict__ log2tab,
                           uint8_t* __restrict__ modes,
                           double* __restrict__ scores, int warps_per_cta,
                           int nsamp_max) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x * warps_per_cta + warp;
  const int nblk = p.nbx * p.nby;
  size_t per_warp = (size_t)nsamp_max * 4 + TB * 8 + (size_t)p.bx * 16;
  unsigned char* base = smem_raw + per_warp * warp;
  int32_t* samp = (int32_t*)base;
  int32_t* first = (int32_t*)(base + (size_t)nsamp_max * 4);
  int32_t* cnt = first + TB;
  int64_t* lastrow = (int64_t*)(cnt + TB);   // [bx][2]
  if (blk >= nblk) return;

  const int bi = blk / p.nbx, bj = blk - bi * p.nbx;
  const int r0 = bi * p.by, r1 = min(r0 + p.by, p.H);
  const int c0 = bj * p.bx, c1 = min(c0 + p.bx, p.W);
  const int W = p.W, H = p.H;
  const int64_t fb = (int64_t)p.t * H * W;
  const int64_t tau = p.tau, two_tau = 2 * tau;
  const double inv = 1.0 / (double)two_tau;
  const int nsx = (c1 - c0 + p.stride - 1) / p.stride;
  const int nsy = (r1 - r0 + p.stride - 1) / p.stride;
  const int ns = 2 * nsx * nsy;
  for (int k = lane; k < TB; k += 32) { first[k] = 0x7fffffff; cnt[k] = 0; }

  auto orig_at = [&](int i, int j, int comp) -> int64_t {
    return comp ? (int64_t)load_fixed(v, fb + (int64_t)i * W + j, p.S)
                : (int64_t)load_fixed(u, fb + (int64_t)i * W + j, p.S);
  };

  double rate[2];
  for (int mode = 0; mode < 2; mode++) {
    if (mode == 0) {
      // Lorenzo trial on the candidate (block-local write-back), raster order
      for (int g = r0; g < r1; g += 32) {
        const int i = g + lane;
        const bool rowok = i < r1;
        int64_t eL[2] = {0, 0}, eU_prev[2] = {0, 0}, eLast[2] = {0, 0};
        const int nsteps = (c1 - c0) + 31;
        for (int s = 0; s < nsteps; s++) {
          const int j = c0 + s - lane;
          // neighbour errors (block-local; zero outside the block)
          int64_t eU[2];
#pragma unroll
          for (int comp = 0; comp < 2; comp++) {
            int64_t fromup = __shfl_up_sync(0xffffffffu, eLast[comp], 1);
            if (lane == 0)
              fromup = (g > r0 && j >= c0 && j < c1)
                           ? lastrow[(j - c0) * 2 + comp] : 0;
            eU[comp] = fromup;
          }
          const bool act = rowok && j >= c0 && j < c1;
          if (act) {
            const int64_t k = (int64_t)i * W + j;
            bool samp_here = ((i - r0) % p.stride == 0) &&
                             ((j - c0) % p.stride == 0);
#pragma unroll
            for (int comp = 0; comp < 2; comp++) {
              const I* prv = comp ? vp : up;
              int64_t o = orig_at(i, j, comp);
              int64_t pred = (int64_t)prv[k];
              if (i > 0) pred += orig_at(i - 1, j, comp) - (int64_t)prv[k - W];
              if (j > 0) pred += orig_at(i, j - 1, comp) - (int64_t)prv[k - 1];
              if (i > 0 && j > 0)
                pred += (int64_t)prv[k - W - 1] - orig_at(i - 1, j - 1, comp);
              int64_t dU = (i > r0) ? eU[comp] : 0;
              int64_t dL = (j > c0) ? eL[comp] : 0;
              int64_t dUL = (i > r0 && j > c0) ? eU_prev[comp] : 0;
              pred += dU + dL - dUL;
              int64_t r = o - pred;
              int64_t q = quant_rha(r, tau, inv);
              bool ok = q > -p.radius && q < p.radius;
              int64_t err = ok ? q * two_tau - r : 0;
              eL[comp] = err;
              eLast[comp] = err;
              if (samp_here) {
                int sp = 2 * (((i - r0) / p.stride) * nsx + (j - c0) / p.stride) + comp;
                samp[sp] = ok ? (int32_t)(q < 0 ? -q : q) : -1;
              }
            }
          }
#pragma unroll
          for (int comp = 0; comp < 2; comp++) eU_prev[comp] = eU[comp];
          if (lane == 31 && act) {
            lastrow[(j - c0) * 2 + 0] = eLast[0];
            lastrow[(j - c0) * 2 + 1] = eLast[1];
          }
          __syncwarp();
        }
      }
    } else {
      // SL trial: only the stride-sampled pixels reach the histogram
      for (int sidx = lane; sidx < nsx * nsy; sidx += 32) {
        int si = sidx / nsx, sj = sidx - si * nsx;
        int i = r0 + si * p.stride, j = c0 + sj * p.stride;
        double fi, fj;
        sl_departure(up, vp, H, W, i, j, p.cfl_x, p.cfl_y, p.d_max, p.n_max,
                     &fi, &fj);
        BilinearTap tp = bilinear_tap(H, W, fi, fj);
#pragma unroll
        for (int comp = 0; comp < 2; comp++) {
          int64_t pred = bilinear_apply(tp, comp ? vp : up);
          int64_t r = orig_at(i, j, comp) - pred;
          int64_t q = quant_rha(r, tau, inv);
          bool ok = q > -p.radius && q < p.radius;
          samp[2 * sidx + comp] = ok ? (int32_t)(q < 0 ? -q : q) : -1;
        }
      }
    }
    __syncwarp();
    // ---- first-touch histogram and entropy (mop.py:118-138)
    int n_ok = 0, lp = 0;
    bool big = false;
    for (int sp = lane; sp < ns; sp += 32) {
      int a = samp[sp];
      if (a < 0) { lp++; continue; }
      n_ok++;
      if (a < TB) { atomicMin(first + a, sp); atomicAdd(cnt + a, 1); }
      else big = true;
    }
    for (int o = 16; o; o >>= 1) {
      n_ok += __shfl_xor_sync(0xffffffffu, n_ok, o);
      lp += __shfl_xor_sync(0xffffffffu, lp, o);
    }
    big = __any_sync(0xffffffffu, big);
    __syncwarp();
    double acc = 0.0;
    for (int c = 0; c < ns; c += 32) {
      int sp = c + lane;
      bool ft = false;
      int h = 0;
      if (sp < ns) {
        int a = samp[sp];
        if (a >= 0 && a < TB) {
          ft = first[a] == sp;
          h = cnt[a];
        } else if (a >= TB) {
          // rare large index: exact scans
          ft = true;
          for (int q = 0; q < sp; q++)
            if (samp[q] == a) { ft = false; break; }
          if (ft)
            for (int q = 0; q < ns; q++) h += samp[q] == a;
        }
      }
      double term = ft ? __dmul_rn((double)h, log2tab[h]) : 0.0;
      unsigned bal = __ballot_sync(0xffffffffu, ft);
      while (bal) {
        int b = __ffs(bal) - 1;
        bal &= bal - 1;
        acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, term, b));
      }
    }
    (void)big;
    __syncwarp();
    for (int sp = lane; sp < ns; sp += 32) {
      int a = samp[sp];
      if (a >= 0 && a < TB) { first[a] = 0x7fffffff; cnt[a] = 0; }
    }
    __syncwarp();
    double h0 = 0.0;
    if (n_ok > 0)
      h0 = __dsub_rn(log2tab[n_ok], __ddiv_rn(acc, (double)n_ok));
    double r;
    if (n_ok + lp > 0)
      r = __dadd_rn(__dadd_rn(h0, __ddiv_rn(__dmul_rn(p.lam, (double)lp),
                                           (double)(n_ok + lp))),
                    p.rmeta);
    else
      r = p.rmeta;
    rate[mode] = r;
  }
  if (lane == 0) {
    int64_t mb = (int64_t)(p.t - 1) * nblk + blk;
    bool sl = rate[0] > 0.0 &&
              __ddiv_rn(__dsub_rn(rate[0], rate[1]), rate[0]) > p.theta;
    modes[mb] = sl ? 1 : 0;
    if (scores) {
      scores[2 * mb] = rate[0];
      scores[2 * mb + 1] = rate[1];
    }
  }
}

// -------------------------------------------------------------- encode
template <typename F, typename I, typename SYM>
__global__ void __launch_bounds__(32)
encode_kernel(const F* __restrict__ u, const F* __restrict__ v,
              const uint8_t* __restrict__ codes, const I* __restrict__ up,
              const I* __restrict__ vp, I* __restrict__ cu, I* __restrict__ cv,
              const uint8_t* __restrict__ modes_t, FrameParams p, Ladder lad,
              const int64_t* __restrict__ qd_row_off, SYM* __restrict__ qd,
              int32_t* __restrict__ row_ll, I* bnd, int* progress,
              int* ticket) {
  const int lane = threadIdx.x;
  int strip = 0;
  if (lane == 0) strip = atomicAdd(ticket, 1);
  strip = __shfl_sync(0xffffffffu, strip, 0);
  const int H = p.H, W = p.W;
  const int i = strip * 32 + lane;
  const bool rowok = i < H;
  const int64_t fb = (int64_t)p.t * H * W;
  const int64_t row = (int64_t)p.t * H + i;
  int64_t pos = rowok ? qd_row_off[row] : 0;
  int nll = 0;
  int64_t rL[2] = {0, 0}, rLast[2] = {0, 0}, rUprev[2] = {0, 0};
  const int nsteps = W + 31;
  const int nstrips = (H + 31) / 32;
  I* my_bnd = bnd + (size_t)strip * W * 2;
  const I* up_bnd = bnd + (size_t)(strip - 1) * W * 2;
  for (int s0 = 0; s0 < nsteps; s0 += 32) {
    // wait until the strip above has finished the columns lane 0 needs
    if (strip > 0) {
      int need = min(W, s0 + 32);
      if (lane == 0) {
        volatile int* pr = progress + strip - 1;
        while (*pr < need) __nanosleep(64);
      }
      __syncwarp();
      __threadfence();
    }
    for (int s = s0; s < min(s0 + 32, nsteps); s++) {
      const int j = s - lane;
      int64_t rU[2];
#pragma unroll
      for (int comp = 0; comp < 2; comp++) {
        int64_t x = __shfl_up_sync(0xffffffffu, rLast[comp], 1);
        if (lane == 0)
          x = (strip > 0 && j >= 0 && j < W)
                  ? (int64_t)__ldcg(up_bnd + 2 * (size_t)j + comp) : 0;
        rU[comp] = x;
      }
      const bool act = rowok && j >= 0 && j < W;
      if (act) {
        const int64_t k = (int64_t)i * W + j;
        const int code = codes[fb + k];
        const int64_t e = lad.e[code];
        int64_t o[2] = {(int64_t)load_fixed(u, fb + k, p.S),
                        (int64_t)load_fixed(v, fb + k, p.S)};
        int64_t rec[2];
        if (e == 0) {
          rec[0] = o[0]; rec[1] = o[1];
          nll += 2;
        } else {
          const int64_t two_e = 2 * e;
          const double inv = lad.inv2e[code];
          bool sl = p.use_modes &&
                    modes_t[(i / p.by) * p.nbx + j / p.bx] == 1;
          int64_t pred[2];
          if (sl) {
            double fi, fj;
            sl_departure(up, vp, H, W, i, j, p.cfl_x, p.cfl_y, p.d_max,
                         p.n_max, &fi, &fj);
            BilinearTap tp = bilinear_tap(H, W, fi, fj);
            pred[0] = bilinear_apply(tp, up);
            pred[1] = bilinear_apply(tp, vp);
          } else {
#pragma unroll
            for (int comp = 0; comp < 2; comp++) {
              const I* prv = comp ? vp : up;
              int64_t pr = (int64_t)prv[k];
              if (i > 0) pr += rU[comp] - (int64_t)prv[k - W];
              if (j > 0) pr += rL[comp] - (int64_t)prv[k - 1];
              if (i > 0 && j > 0) pr += (int64_t)prv[k - W - 1] - rUprev[comp];
              pred[comp] = pr;
            }
          }
          SYM sym[2];
#pragma unroll
          for (int comp = 0; comp < 2; comp++) {
            int64_t r = o[comp] - pred[comp];
            int64_t q = quant_rha(r, e, inv);
            if (q > -p.radius && q < p.radius) {
              sym[comp] = (SYM)(q + p.radius);
              rec[comp] = pred[comp] + q * two_e;
            } else {
              sym[comp] = 0;
              rec[comp] = o[comp];
              nll += 1;
            }
          }
          qd[pos] = sym[0];
          qd[pos + 1] = sym[1];
          pos += 2;
        }
        cu[k] = (I)rec[0];
        cv[k] = (I)rec[1];
        rL[0] = rec[0]; rL[1] = rec[1];
        rLast[0] = rec[0]; rLast[1] = rec[1];
        if (lane == 31) {
          my_bnd[2 * (size_t)j] = (I)rec[0];
          my_bnd[2 * (size_t)j + 1] = (I)rec[1];
        }
      }
      rUprev[0] = rU[0]; rUprev[1] = rU[1];
    }
    // publish: the last row of this strip has finished columns < done
    // (only full strips have a successor; lane 31 wrote the boundary row)
    if (strip + 1 < nstrips && lane == 31) {
      int done = min(W, s0 + 1);
      __threadfence();
      atomicMax(progress + strip, done);
    }
    __syncwarp();
  }
  if (rowok) row_ll[row] = nll;
}

// -------------------------------------------------------------- ll stream
// One warp per frame row; rows without ll entries exit immediately.
template <typename F, typename SYM>
__global__ void ll_write_kernel(const F* __restrict__ u,
                                const F* __restrict__ v,
                                const uint8_t* __restrict__ codes,
                                const SYM* __restrict__ qd,
                                const int64_t* __restrict__ qd_row_off,
                                const int32_t* __restrict__ row_ll,
                                const int64_t* __restrict__ ll_row_off,
                                int64_t nrows, int H, int W, double S,
                                int64_t* __restrict__ ll) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows || row_ll[row] == 0) return;
  const int64_t rb = row * W;   // vid of (t, i, 0): rows are frame-major
  int64_t qpos = qd_row_off[row];
  int64_t lpos = ll_row_off[row];
  for (int c0 = 0; c0 < W; c0 += 32) {
    int j = c0 + lane;
    bool inb = j < W;
    int code = inb ? codes[rb + j] : 31;
    bool nl = inb && code != 31;
    unsigned bnl = __ballot_sync(0xffffffffu, nl);
    int64_t my_q = qpos + 2 * __popc(bnl & ((1u << lane) - 1));
    int nll = 0;
    bool eu = false, ev = false;
    if (inb) {
      if (!nl) { nll = 2; eu = ev = true; }
      else {
        eu = qd[my_q] == 0;
        ev = qd[my_q + 1] == 0;
        nll = (int)eu + (int)ev;
      }
    }
    int incl = nll;
    for (int o = 1; o < 32; o <<= 1) {
      int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    int64_t my_l = lpos + incl - nll;
    if (eu) ll[my_l++] = load_fixed(u, rb + j, S);
    if (ev) ll[my_l++] = load_fixed(v, rb + j, S);
    qpos += 2 * __popc(bnl);
    lpos += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ------------------------------------------------------------ launchers
template <typename F, typename I>
cudaError_t launch_mop(const F* u, const F* v, const I* up, const I* vp,
                       const FrameParams& p, const double* log2tab,
                       uint8_t* modes, double* scores, cudaStream_t st) {
  int nsx = (p.bx + p.stride - 1) / p.stride;
  int nsy = (p.by + p.stride - 1) / p.stride;
  int nsamp = 2 * nsx * nsy;
  size_t per_warp = (size_t)nsamp * 4 + TB * 8 + (size_t)p.bx * 16;
  int wpc = (int)max((size_t)1, min((size_t)4, (size_t)(200 * 1024) / per_warp));
  size_t smem = per_warp * wpc;
  cudaError_t e = cudaFuncSetAttribute(
      mop_kernel<F, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int nblk = p.nbx * p.nby;
  mop_kernel<F, I><<<(nblk + wpc - 1) / wpc, 32 * wpc, smem, st>>>(
      u, v, up, vp, p, log2tab, modes, scores, wpc, nsamp);
  return cudaGetLastError();
}

template <typename F, typename I, typename SYM>
cudaError_t launch_encode(const F* u, const F* v, const uint8_t* codes,
                          const I* up, const I* vp, I* cu, I* cv,
                          const uint8_t* modes_t, const FrameParams& p,
                          const Ladder& lad, const int64_t* qd_row_off,
                          SYM* qd, int32_t* row_ll, I* bnd, int* progress,
                          int* ticket, cudaStream_t st) {
  int nstrips = (p.H + 31) / 32;
  cudaMemsetAsync(progress, 0, sizeof(int) * (nstrips + 1), st);
  cudaMemsetAsync(ticket, 0, sizeof(int), st);
  encode_kernel<F, I, SYM><<<nstrips, 32, 0, st>>>(
      u, v, codes, up, vp, cu, cv, modes_t, p, lad, qd_row_off, qd, row_ll,
      bnd, progress, ticket);
  return cudaGetLastError();
}

template <typename F, typename SYM>
cudaError_t launch_ll_write(const F* u, const F* v, const uint8_t* codes,
                            const SYM* qd, const int64_t* qd_row_off,
                            const int32_t* row_ll, const int64_t* ll_row_off,
                            int64_t nrows, int H, int W, double S, int64_t* ll,
                            cudaStream_t st) {
  int64_t blocks = (nrows + 7) / 8;
  ll_write_kernel<F, SYM><<<(unsigned)blocks, 256, 0, st>>>(
      u, v, codes, qd, qd_row_off, row_ll, ll_row_off, nrows, H, W, S, ll);
  return cudaGetLastError();
}

#define VFCP_INST_ENC(F, I, SYM)                                              \
  template cudaError_t launch_encode<F, I, SYM>(                              \
      const F*, const F*, const uint8_t*, const I*, const I*, I*, I*,         \
      const uint8_t*, const FrameParams&, const Ladder&, const int64_t*,      \
      SYM*, int32_t*, I*, int*, int*, cudaStream_t);
#define VFCP_INST_MOP(F, I)                                                   \
  template cudaError_t launch_mop<F, I>(const F*, const F*, const I*,         \
                                        const I*, const FrameParams&,         \
                                        const double*, uint8_t*, double*,     \
                                        cudaStream_t);
#define VFCP_INST_LL(F, SYM)                                                  \
  template cudaError_t launch_ll_write<F, SYM>(                               \
      const F*, const F*, const uint8_t*, const SYM*, const int64_t*,         \
      const int32_t*, const int64_t*, int64_t, int, int, double, int64_t*,    \
      cudaStream_t);

VFCP_INST_MOP(float, int32_t)
VFCP_INST_MOP(float, int64_t)
VFCP_INST_MOP(double, int32_t)
VFCP_INST_MOP(double, int64_t)
VFCP_INST_ENC(float, int32_t, uint16_t)
VFCP_INST_ENC(float, int64_t, uint16_t)
VFCP_INST_ENC(double, int32_t, uint16_t)
VFCP_INST_ENC(double, int64_t, uint16_t)
VFCP_INST_ENC(float, int32_t, uint32_t)
VFCP_INST_ENC(float, int64_t, uint32_t)
VFCP_INST_ENC(double, int32_t, uint32_t)
VFCP_INST_ENC(double, int64_t, uint32_t)
VFCP_INST_LL(float, uint16_t)
VFCP_INST_LL(double, uint16_t)
VFCP_INST_LL(float, uint32_t)
VFCP_INST_LL(double, uint32_t)

}  // namespace vfcp
