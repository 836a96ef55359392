// Decompression: stream offsets and the per-frame reconstruction.
//
//   decode_rows_kernel   codes per row -> non-lossless counts, plus the
//                        l_d / code consistency check of codec.py:411-413
//   decode_ll_kernel     escapes per row (symbol 0) -> ll counts
//   decode_kernel        codec.py:167-206 _decode_frame, plus the float64
//                        output of codec.py:443-444 (recon * (1/S), exact)
//
// decode_kernel uses the same strip wavefront as the encoder: a lane owns a
// row, lanes are skewed by one column, strips chain through a boundary row.
#include "common.cuh"

namespace vfcp {


// One warp per frame row.
__global__ void decode_rows_kernel(const uint8_t* __restrict__ codes,
                                   const uint8_t* __restrict__ ld,
                                   int64_t nrows, int W, int64_t tau,
                                   int32_t* __restrict__ row_n31,
                                   int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int64_t rb = row * W;
  int n31 = 0;
  bool mismatch = false;
  for (int c0 = 0; c0 < W; c0 += 32) {
    int j = c0 + lane;
    if (j < W) {
      // eq == 0 (codec.py:408-410): code 31, or a code past tau's bit length
      int c = codes[rb + j];
      bool l = c >= CODE_LOSSLESS || tau <= 0 || (tau >> c) == 0;
      n31 += l;
      if (ld && (get_packbit(ld, rb + j) != (int)l)) mismatch = true;
    }
  }
  for (int o = 16; o; o >>= 1) n31 += __shfl_xor_sync(0xffffffffu, n31, o);
  if (__any_sync(0xffffffffu, mismatch) && lane == 0) atomicOr(bad, 1);
  if (lane == 0) row_n31[row] = n31;
}

template <typename SYM>
__global__ void decode_ll_kernel(const SYM* __restrict__ qd,
                                 const int64_t* __restrict__ qd_row_off,
                                 const int32_t* __restrict__ row_n31,
                                 int64_t nrows, int32_t* __restrict__ row_ll) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  int64_t a = qd_row_off[row], b = qd_row_off[row + 1];
  int z = 0;
  for (int64_t q = a + lane; q < b; q += 32) z += qd[q] == 0;
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) row_ll[row] = z + 2 * row_n31[row];
}

template <typename I, typename SYM>
__global__ void __launch_bounds__(32)
decode_kernel(const uint8_t* __restrict__ codes, const SYM* __restrict__ qd,
              const int64_t* __restrict__ ll, const uint8_t* __restrict__ modes_t,
              const I* __restrict__ up, const I* __restrict__ vp,
              I* __restrict__ cu, I* __restrict__ cv, DecodeParams p,
              Ladder lad, const int64_t* __restrict__ qd_row_off,
              const int64_t* __restrict__ ll_row_off,
              double* __restrict__ out_u, double* __restrict__ out_v,
              int64_t* __restrict__ fix_u, int64_t* __restrict__ fix_v,
              I* bnd, int* progress, int* ticket) {
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
  int64_t lpos = rowok ? ll_row_off[row] : 0;
  int64_t rL[2] = {0, 0}, rLast[2] = {0, 0}, rUprev[2] = {0, 0};
  const int nsteps = W + 31;
  const int nstrips = (H + 31) / 32;
  I* my_bnd = bnd + (size_t)strip * W * 2;
  const I* up_bnd = bnd + (size_t)(strip - 1) * W * 2;
  for (int s0 = 0; s0 < nsteps; s0 += 32) {
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
        int64_t rec[2];
        if (e == 0) {
          rec[0] = ll[lpos];
          rec[1] = ll[lpos + 1];
          lpos += 2;
        } else {
          const int64_t two_e = 2 * e;
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
#pragma unroll
          for (int comp = 0; comp < 2; comp++) {
            int64_t sym = (int64_t)qd[pos + comp];
            if (sym == 0) rec[comp] = ll[lpos++];
            else rec[comp] = pred[comp] + (sym - p.radius) * two_e;
          }
          pos += 2;
        }
        cu[k] = (I)rec[0];
        cv[k] = (I)rec[1];
        out_u[fb + k] = __dmul_rn((double)rec[0], p.inv_S);
        out_v[fb + k] = __dmul_rn((double)rec[1], p.inv_S);
        if (fix_u) { fix_u[fb + k] = rec[0]; fix_v[fb + k] = rec[1]; }
        rL[0] = rec[0]; rL[1] = rec[1];
        rLast[0] = rec[0]; rLast[1] = rec[1];
        if (lane == 31) {
          my_bnd[2 * (size_t)j] = (I)rec[0];
          my_bnd[2 * (size_t)j + 1] = (I)rec[1];
        }
      }
      rUprev[0] = rU[0]; rUprev[1] = rU[1];
    }
    if (strip + 1 < nstrips && lane == 31) {
      int done = min(W, s0 + 1);
      __threadfence();
      atomicMax(progress + strip, done);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ launchers
cudaError_t launch_decode_rows(const uint8_t* codes, const uint8_t* ld,
                               int64_t nrows, int W, int64_t tau,
                               int32_t* row_n31, int* bad, cudaStream_t st) {
  decode_rows_kernel<<<(unsigned)((nrows + 7) / 8), 256, 0, st>>>(
      codes, ld, nrows, W, tau, row_n31, bad);
  return cudaGetLastError();
}

template <typename SYM>
cudaError_t launch_decode_ll(const SYM* qd, const int64_t* qd_row_off,
                             const int32_t* row_n31, int64_t nrows,
                             int32_t* row_ll, cudaStream_t st) {
  decode_ll_kernel<SYM><<<(unsigned)((nrows + 7) / 8), 256, 0, st>>>(
      qd, qd_row_off, row_n31, nrows, row_ll);
  return cudaGetLastError();
}

template <typename I, typename SYM>
cudaError_t launch_decode(const uint8_t* codes, const SYM* qd,
                          const int64_t* ll, const uint8_t* modes_t,
                          const I* up, const I* vp, I* cu, I* cv,
                          const DecodeParams& p, const Ladder& lad,
                          const int64_t* qd_row_off,
                          const int64_t* ll_row_off, double* out_u,
                          double* out_v, int64_t* fix_u, int64_t* fix_v,
                          I* bnd, int* progress, int* ticket,
                          cudaStream_t st) {
  int nstrips = (p.H + 31) / 32;
  cudaMemsetAsync(progress, 0, sizeof(int) * (nstrips + 1), st);
  cudaMemsetAsync(ticket, 0, sizeof(int), st);
  decode_kernel<I, SYM><<<nstrips, 32, 0, st>>>(
      codes, qd, ll, modes_t, up, vp, cu, cv, p, lad, qd_row_off, ll_row_off,
      out_u, out_v, fix_u, fix_v, bnd, progress, ticket);
  return cudaGetLastError();
}

#define VFCP_INST_DEC(I, SYM)                                                 \
  template cudaError_t launch_decode<I, SYM>(                                 \
      const uint8_t*, const SYM*, const int64_t*, const uint8_t*, const I*,   \
      const I*, I*, I*, const DecodeParams&, const Ladder&, const int64_t*,   \
      const int64_t*, double*, double*, int64_t*, int64_t*, I*, int*, int*,   \
      cudaStream_t);
VFCP_INST_DEC(int32_t, uint16_t)
VFCP_INST_DEC(int64_t, uint16_t)
VFCP_INST_DEC(int32_t, uint32_t)
VFCP_INST_DEC(int64_t, uint32_t)
template cudaError_t launch_decode_ll<uint16_t>(const uint16_t*,
                                                const int64_t*, const int32_t*,
                                                int64_t, int32_t*,
                                                cudaStream_t);
template cudaError_t launch_decode_ll<uint32_t>(const uint32_t*,
                                                const int64_t*, const int32_t*,
                                                int64_t, int32_t*,
                                                cudaStream_t);

}  // namespace vfcp
