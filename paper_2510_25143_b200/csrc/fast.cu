// The per-(row, chunk) prefix counts that place any block's symbols and ll
// values in the streams (encoder and decoder block kernels, enc_block.cu /
// dec_block.cu, and the block scan, bscan.cuh).
#include "bscan.cuh"
#include "predict.cuh"

namespace vfcp {

// ----------------------------------------------------------- prefix counts
// Per frame row: for each 32-column chunk, the number of non-lossless
// pixels (and, for the decoder, ll entries: 2 per lossless pixel plus the
// escapes, symbol 0, among the chunk's symbols) before it in the row.
// One warp per row, lane = chunk; the row is taken in segments of 256
// chunks.  Within a segment every load is independent of the counts: the
// codes of all 256 chunks are read first, and the segment's symbol range
// (which follows from the row offset and the running count) is then
// streamed in 16-byte quads; a quad batch holding an escape attributes it
// to its chunk by a binary search over the chunk starts kept in shared
// memory (escapes are rare).
constexpr int CP_SEG = 256;
template <typename SYM>
__global__ void __launch_bounds__(256)
chunk_prefix_kernel(const uint8_t* __restrict__ codes,
                    const SYM* __restrict__ qd,
                    const int64_t* __restrict__ qd_row_off, int64_t nrows,
                    int W, int nchunks, int64_t tau,
                    int32_t* __restrict__ pre_nl, int32_t* __restrict__ pre_ll) {
  __shared__ int32_t s_start[8][CP_SEG + 1];   // segment-relative pair starts
  __shared__ int32_t s_esc[8][CP_SEG];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (row >= nrows) return;
  // code c quantises iff e = tau >> c > 0 (31 is lossless): the lossy codes
  // are c < cmax = min(31, bit length of tau), counted four bytes at a time
  int cmax = 0;
  for (int c = 0; c < CODE_LOSSLESS; c++)
    if (tau > 0 && (tau >> c) != 0) cmax = c + 1;
  const uint32_t cm4 = 0x01010101u * (uint32_t)cmax;
  const uint8_t* cr = codes + row * (int64_t)W;
  const bool vec = ((row * (int64_t)W) & 15) == 0 &&
                   ((uintptr_t)codes & 15) == 0;
  const int64_t q0 = qd ? qd_row_off[row] : 0;
  int32_t* st = s_start[wid];
  int32_t* es = s_esc[wid];
  int32_t nl_run = 0, ll_run = 0;
  for (int s0 = 0; s0 < nchunks; s0 += CP_SEG) {
    const int nseg = min(CP_SEG, nchunks - s0);
    int nl[8], ncl[8];
#pragma unroll
    for (int g = 0; g < 8; g++) {
      const int x = s0 + 32 * g + lane;
      nl[g] = 0;
      ncl[g] = 0;
      if (32 * g < nseg && x < nchunks) {
        const int jb = 32 * x;
        ncl[g] = min(32, W - jb);
        if (vec && ncl[g] == 32) {
          const uint4 a = __ldg(reinterpret_cast<const uint4*>(cr + jb));
          const uint4 b = __ldg(reinterpret_cast<const uint4*>(cr + jb + 16));
          nl[g] = (__popc(__vcmpltu4(a.x, cm4)) + __popc(__vcmpltu4(a.y, cm4)) +
                   __popc(__vcmpltu4(a.z, cm4)) + __popc(__vcmpltu4(a.w, cm4)) +
                   __popc(__vcmpltu4(b.x, cm4)) + __popc(__vcmpltu4(b.y, cm4)) +
                   __popc(__vcmpltu4(b.z, cm4)) + __popc(__vcmpltu4(b.w, cm4))) >> 3;
        } else {
          for (int k = 0; k < ncl[g]; k++) nl[g] += (int)cr[jb + k] < cmax;
        }
      }
    }
    int carry = 0;   // segment-relative
#pragma unroll
    for (int g = 0; g < 8; g++) {
      if (32 * g >= nseg) break;   // warp-uniform
      int incl = nl[g];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int c = 32 * g + lane;
      if (c < nseg) {
        pre_nl[row * nchunks + s0 + c] = nl_run + carry + incl - nl[g];
        st[c] = carry + incl - nl[g];
        es[c] = 0;
      }
      carry += __shfl_sync(FULL, incl, 31);
    }
    if (lane == 0) st[nseg] = carry;
    __syncwarp();
    if (pre_ll) {
      if (qd) {
        const int S = carry;   // the segment's symbol pairs
        const int64_t qs = q0 + 2 * (int64_t)nl_run;
        // the chunk holding pair k: the last start <= k
        auto attribute = [&](int zc, int k) {
          if (!zc) return;
          int lo = 0, hi = nseg - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (st[mid] <= k) lo = mid; else hi = mid - 1;
          }
          atomicAdd(es + lo, zc);
        };
        if constexpr (sizeof(SYM) == 2) {
          // aligned quads holding the range (a quad with one pair of the
          // range is mapped memory); pairs outside it are masked by k
          const uintptr_t bp = (uintptr_t)(qd + qs);
          const uint4* qa = reinterpret_cast<const uint4*>(bp & ~(uintptr_t)15);
          const int off = (int)((bp & 15) >> 2);
          const int nq = (S + off + 3) >> 2;
          constexpr int QU = 8;
          for (int g0 = 0; g0 < nq; g0 += 32 * QU) {
            uint4 w[QU];
#pragma unroll
            for (int u = 0; u < QU; u++) {
              const int g = g0 + 32 * u + lane;
              w[u] = g < nq ? __ldg(qa + g) : make_uint4(1u, 1u, 1u, 1u);
            }
            uint32_t z = 0;
#pragma unroll
            for (int u = 0; u < QU; u++)
              z |= __vcmpeq2(w[u].x, 0u) | __vcmpeq2(w[u].y, 0u) |
                   __vcmpeq2(w[u].z, 0u) | __vcmpeq2(w[u].w, 0u);
            if (z == 0u) continue;
#pragma unroll
            for (int u = 0; u < QU; u++) {
              const int kb = 4 * (g0 + 32 * u + lane) - off;
              const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const int k = kb + q;
                if (k >= 0 && k < S)
                  attribute(((ww[q] & 0xffffu) == 0u) + ((ww[q] >> 16) == 0u), k);
              }
            }
          }
        } else {
          for (int k = lane; k < S; k += 32)
            attribute((__ldg(qd + qs + 2 * k) == 0) + (__ldg(qd + qs + 2 * k + 1) == 0), k);
        }
        __syncwarp();
      }
      int lcarry = 0;
#pragma unroll
      for (int g = 0; g < 8; g++) {
        if (32 * g >= nseg) break;   // warp-uniform
        const int c = 32 * g + lane;
        const int ll = c < nseg ? 2 * (ncl[g] - nl[g]) + es[c] : 0;
        int lincl = ll;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, lincl, o);
          if (lane >= o) lincl += y;
        }
        if (c < nseg) pre_ll[row * nchunks + s0 + c] = ll_run + lcarry + lincl - ll;
        lcarry += __shfl_sync(FULL, lincl, 31);
      }
      ll_run += lcarry;
    }
    nl_run += carry;
    __syncwarp();   // st / es are rewritten by the next segment
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

template cudaError_t launch_chunk_prefix<uint16_t>(const uint8_t*,
                                                   const uint16_t*,
                                                   const int64_t*, int64_t,
                                                   int, int, int64_t,
                                                   int32_t*, int32_t*,
                                                   cudaStream_t);
}  // namespace vfcp
