// The raster-order Lorenzo recurrence of one frame as a 2D block scan.
//
// In: the prepared planes a (encoder: R0 = orig - Lorenzo(orig, prev), or
// the pinned err; decoder, run on Z = recon - prev: (sym - radius) * 2e, or
// the pinned Z), the per-(row, chunk) pin words and (encoder) the frame
// codes.  Out: the err / recon plane, (encoder) the Lorenzo symbols written
// into the interleaved symbol stream, (decoder) the float64 output -- bit for
// bit what the reference's raster loop (codec.py:118-164 _encode_frame,
// 167-206 _decode_frame) produces.
//
// Why a scan is exact.  Per component, with v the chain value (encoder: err
// = recon - orig; decoder: Z) and zero padding outside the frame,
//   decoder:  v = vU + vL - vUL + A                 (exact)
//   encoder:  v = q*2e - x,  x = R0 - (vU + vL - vUL),  q = rha(x / 2e)
// so in the encoder v == -R0 + vU + vL - vUL (mod 2e) whenever the pixel is
// quantised with the same step e (v in [-e, e] is the representative of
// that residue; a residue of exactly e is a tie whose sign follows x, which
// rounds away from zero).  Over a 32x32 block whose pixels all share one
// step, have no pins and cannot escape (|R0| < (2 radius - 4) e), every
// value is therefore a 2D prefix sum of the block plus its boundary:
//   v(i, j) = top(j) + left(i) - corner + sum_{a<=i, b<=j} X(a, b)
// with X = A (decoder, wrapping uint32 arithmetic is exact because the
// result fits int32) or X = -R0 mod 2e (encoder, then the representative).
// Blocks whose values are known without the recurrence (all pixels pinned:
// semi-Lagrangian blocks, lossless areas) pass their prepared values; any
// other block (mixed pins, mixed steps, possible escapes, a tie on its
// boundary) is swept exactly, pixel by pixel, given its exact boundary.
//
// Three phases per frame:
//   phase A  fully parallel, in the prepare kernels (enc_r0_kernel and
//            enc_pix_kernel; bs_local_kernel for the decoder): block class
//            and the bottom row / right column of the block-local prefix
//            sums (LB, LR), or the known edge values;
//   phase B  chain tasks of bs_chain_kernel, the only sequential part: block
//            boundaries travel down the block rows (one warp per block row
//            and component walks its row; 32 exact values per block are
//            handed to the warp below) -- the critical path is ~nby + nbx
//            cheap block steps instead of H + W pixel steps;
//   phase C  interior tasks of the same persistent kernel, handed out after
//            the chain tasks and started per 32-block segment once the chain
//            has published it, so they overlap the chain: the interior of
//            every block from its exact boundary (prefix sums in shared
//            memory, ties resolved in raster order, symbols).
#pragma once

#include "frame.cuh"

namespace vfcp {

enum : uint8_t { BS_SLOW = 0, BS_KNOWN = 1, BS_REG = 2, BS_DONE = 3 };

struct BScanIO {
  const int32_t* a[2];
  const uint8_t* codes;     // encoder: frame codes (pitch Wp)
  const uint32_t* pin[2];   // per (row, chunk)
  int32_t* out[2];          // encoder: err; decoder: recon (pitch Wp)
  // encoder, frame t: the interleaved symbol stream (u, v per non-lossless
  // vertex in raster order; positions from the per-row offsets and the
  // per-(row, chunk) prefix counts) and the per-row escape counts
  uint16_t* qd;
  const int64_t* qd_row_off;  // [H] (frame t)
  const int32_t* pre_nl;      // [H][nchunks] (frame t)
  const uint32_t* nlw;        // [H][nchunks] non-lossless bit words
  int32_t* row_ll;            // [H] (frame t)
  int32_t* lb;              // [2][nblk][32] block bottom row: local prefix
                            // (REG) or the known values (KNOWN)
  int32_t* lr;              // [2][nblk][32] block right column, likewise
  unsigned long long* stamps;  // optional [2][nby][3] ns: start, first top, end
  unsigned long long* prog;    // [2][nby]: frame tag << 32 | blocks finished
  uint32_t frame_tag;          // unique per frame of a call (t + 1)
  // decoder, frame t: the float64 output recon * inv_S (and optionally the
  // int64 fixed-point recon), pitch W -- written by the interior pass
  double* f64[2];
  int64_t* fix[2];
  double inv_S;
  // decoder: the chain runs on Z = recon - p (dec_prep_kernel); p is the
  // previous frame's recon (pitch Wp), nullptr for frame 0
  const int32_t* prev[2];
  int32_t* ebot;            // [2][nblk][32] exact block bottom rows (chain)
  int32_t* eright;          // [2][nblk][32] exact block right columns (chain)
  int32_t* cls;             // [2][nblk] class | code << 2
  uint64_t* bnd;            // tagged boundary slots [ntask][W]
  int* ticket;
  uint32_t tag_base;
  int H, W, Wp, nchunks, nbx, nby;
  int radius;
  int32_t e_tab[32];        // e per code (0: lossless)
  uint32_t mag_tab[32];     // floor(2^32 / 2e) per code (0: lossless)
};

constexpr int BS_NW = 8;        // block rows (warps) per chain CTA
constexpr int BS_HRING = 256;   // shared boundary ring (columns), power of 2
constexpr int BS_PF = 8;        // blocks of (class, LB, LR) staged ahead
constexpr int BS_SEG = 32;      // blocks per progress mark / interior task

__host__ __device__ inline int bs_ntask(int nby) {
  return 2 * ((nby + BS_NW - 1) / BS_NW);
}

// x mod m for any uint32 x, M = floor(2^32 / m), m >= 2: the estimate
// umulhi(x, M) is floor(x/m) or one less.
__device__ __forceinline__ uint32_t bs_umod(uint32_t x, uint32_t m, uint32_t M) {
  const uint32_t r = x - __umulhi(x, M) * m;
  return r >= m ? r - m : r;
}
__device__ __forceinline__ uint32_t bs_madd(uint32_t a, uint32_t b, uint32_t m) {
  const uint32_t s = a + b;
  return s >= m ? s - m : s;
}
__device__ __forceinline__ uint32_t bs_msub(uint32_t a, uint32_t b, uint32_t m) {
  return a >= b ? a - b : a + m - b;
}
// residue in [0, m) of any int32 (neighbouring values may come from blocks
// with other step sizes)
__device__ __forceinline__ uint32_t bs_res_any(int32_t v, uint32_t m, uint32_t M) {
  // branch-free: lanes of a warp hold values of both signs
  const uint32_t a = v < 0 ? (uint32_t)0 - (uint32_t)v : (uint32_t)v;
  const uint32_t r = bs_umod(a, m, M);
  return (v < 0 && r != 0u) ? m - r : r;
}
// residue of a neighbour's exact value: |v| < m unless the neighbour was
// quantised with a larger step
__device__ __forceinline__ uint32_t bs_res(int32_t v, uint32_t m, uint32_t M) {
  const uint32_t r = (uint32_t)v + (v < 0 ? m : 0u);
  if (r < m) return r;
  return bs_res_any(v, m, M);
}
// residue of -R0 (|R0| < 2^31 - 1 on this path)
__device__ __forceinline__ uint32_t bs_negres(int32_t r0, uint32_t m, uint32_t M) {
  return bs_res_any(-r0, m, M);
}
// representative in [-e, e] of a residue that is not the tie e
__device__ __forceinline__ int32_t bs_rep(uint32_t r, uint32_t e, uint32_t m) {
  return r < e ? (int32_t)r : (int32_t)r - (int32_t)m;
}

// Exact encoder step (codec.py:140-155): x = R0 - d, q = rha(x / 2e);
// escape -> err 0, symbol 0.
__device__ __forceinline__ int32_t bs_enc_exact(int32_t R0, int32_t d,
                                                int32_t e, int32_t radius,
                                                uint32_t* sym) {
  const int64_t m = 2 * (int64_t)e;
  const int64_t x = (int64_t)R0 - d;
  int64_t q = (int64_t)floor(__ddiv_rn((double)x, (double)m));
  int64_t r = x - q * m;
  if (r < 0) { q--; r += m; }
  else if (r >= m) { q++; r -= m; }
  if (2 * r > m || (2 * r == m && x > 0)) q++;
  if (q <= -radius || q >= radius) { *sym = 0u; return 0; }
  *sym = (uint32_t)(q + radius);
  return (int32_t)(q * m - x);
}

// ------------------------------------------------------------ phase A
// CTA = one block, warp = component (lane = column).
template <bool ENC>
__global__ void __launch_bounds__(64) bs_local_kernel(BScanIO io) {
  __shared__ uint32_t sx[2][32][33];
  __shared__ int32_t etab[32];
  __shared__ uint32_t mtab[32];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, comp = threadIdx.x >> 5;
  if (threadIdx.x < 32) { etab[lane] = io.e_tab[lane]; mtab[lane] = io.mag_tab[lane]; }
  const int bj = blockIdx.x, bi = blockIdx.y;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, io.H - r0), ncl = min(32, io.W - c0);
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int32_t* a = io.a[comp];
  const uint32_t vm = ncl >= 32 ? FULL : ((1u << ncl) - 1u);
  const uint32_t pw =
      lane < nr ? (io.pin[comp][(int64_t)(r0 + lane) * io.nchunks + bj] & vm) : 0u;
  const bool anypin = __any_sync(FULL, pw != 0u);
  const bool allpin = __all_sync(FULL, lane >= nr || pw == vm);
  __syncthreads();
  int32_t cls;
  if (allpin) {
    // known values: the chain passes the edges on
    cls = BS_KNOWN;
    io.lb[(comp * nblk + blk) * 32 + lane] =
        lane < ncl ? __ldg(a + (int64_t)(r0 + nr - 1) * io.Wp + c0 + lane) : 0;
    io.lr[(comp * nblk + blk) * 32 + lane] =
        lane < nr ? __ldg(a + (int64_t)(r0 + lane) * io.Wp + c0 + ncl - 1) : 0;
  } else if (anypin) {
    cls = BS_SLOW;
  } else {
    const bool colok = lane < ncl;
    int32_t xa[32];
#pragma unroll
    for (int r = 0; r < 32; r++)
      xa[r] = (r < nr && colok) ? __ldg(a + (int64_t)(r0 + r) * io.Wp + c0 + lane) : 0;
    bool ok = true;
    uint32_t m = 0, M = 0;
    int code = 0;
    if (ENC) {
      code = io.codes[(int64_t)r0 * io.Wp + c0];
      const int32_t e = etab[code & 31];
      m = 2u * (uint32_t)e;
      M = mtab[code & 31];
      const int64_t lim = (2 * (int64_t)io.radius - 4) * (int64_t)e;
      ok = e > 0 && lim > 0;
#pragma unroll
      for (int r = 0; r < 32; r++) {
        if (r < nr && colok) {
          const int cd = io.codes[(int64_t)(r0 + r) * io.Wp + c0 + lane];
          const int64_t ax = xa[r] < 0 ? -(int64_t)xa[r] : (int64_t)xa[r];
          ok &= (cd == code) && ax < lim;
        }
      }
      ok = __all_sync(FULL, ok);
    }
    if (!ok) {
      cls = BS_SLOW;
    } else {
      cls = BS_REG | (code << 2);
#pragma unroll
      for (int r = 0; r < 32; r++)
        sx[comp][r][lane] = ENC ? bs_negres(xa[r], m, M) : (uint32_t)xa[r];
      __syncwarp();
      // column sum (lane = column) and row sum (lane = row)
      uint64_t cs = 0, rs = 0;
#pragma unroll
      for (int k = 0; k < 32; k++) {
        cs += sx[comp][k][lane];
        rs += sx[comp][lane][k];
      }
      uint32_t c32, r32;
      if (ENC) { c32 = (uint32_t)(cs % m); r32 = (uint32_t)(rs % m); }
      else { c32 = (uint32_t)cs; r32 = (uint32_t)rs; }
      // inclusive scans over lanes: LB(j) = sum_{b<=j} colsum(b),
      // LR(i) = sum_{a<=i} rowsum(a)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t pc = __shfl_up_sync(FULL, c32, o);
        const uint32_t pr = __shfl_up_sync(FULL, r32, o);
        if (lane >= o) {
          c32 = ENC ? bs_madd(c32, pc, m) : c32 + pc;
          r32 = ENC ? bs_madd(r32, pr, m) : r32 + pr;
        }
      }
      io.lb[(comp * nblk + blk) * 32 + lane] = (int32_t)c32;
      io.lr[(comp * nblk + blk) * 32 + lane] = (int32_t)r32;
    }
  }
  if (lane == 0) io.cls[comp * nblk + blk] = cls;
}

// ------------------------------------------------------------ phase B
// Shared memory of the fused chain / interior kernel.  The interior tiles
// (tasks after the chain tasks) overlay the chain-only region.
struct BSFinTiles {
  uint32_t x[BS_NW][32][33];
  int32_t v[BS_NW][33][33];
};
struct BSChainSmem {
  int32_t etab[32];
  uint32_t mtab[32];
  int task;
  int done[BS_NW];                     // blocks warp w has consumed
  alignas(16) int32_t pf[BS_NW][BS_PF][64];   // LB (0..31), LR (32..63)
  alignas(16) int32_t pfd[BS_NW][32][4];      // per-lane sink of idle copies
  int32_t pfc[BS_NW][BS_PF];           // class word per block
  union {
    struct {
      uint64_t hin[BS_NW + 1][BS_HRING];   // tagged (column + 1) << 32 | value
      // slow path tiles, [row][col] unpadded: the skewed sweep reads column
      // s - lane in row lane, distinct banks across lanes
      int32_t tv[BS_NW][32][32];           // slow path: values
      uint16_t ts[BS_NW][32][32];          // slow path: symbols (encoder)
      int64_t tq[BS_NW][32];               // slow path: row stream offsets
      uint8_t tc[BS_NW][32][32];           // slow path: codes (encoder)
    };
    BSFinTiles fin;
  };
};

template <bool ENC>
__device__ __forceinline__ void bs_slow_block(
    const BScanIO& io, BSChainSmem& sm, int w, int comp, int bi, int bj,
    int nr, int ncl, int32_t top, int32_t left, int32_t corner, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const bool colok = lane < ncl;
  const int32_t* a = io.a[comp];
  int32_t(*tv)[32] = sm.tv[w];
  for (int r = 0; r < nr; r++) {
    const int64_t k = (int64_t)(r0 + r) * io.Wp + c0 + lane;
    tv[r][lane] = colok ? __ldcg(a + k) : 0;
    if (ENC) sm.tc[w][r][lane] = colok ? io.codes[k] : (uint8_t)CODE_LOSSLESS;
  }
  const uint32_t pw = lane < nr ? io.pin[comp][(int64_t)(r0 + lane) * io.nchunks + bj] : 0u;
  __syncwarp();
  int32_t l = left;
  int32_t ul = __shfl_up_sync(FULL, left, 1);
  if (lane == 0) ul = corner;
  const int32_t radius = io.radius;
  for (int s = 0; s < 63; s++) {
    const int jj = s - lane;
    const bool act = lane < nr && jj >= 0 && jj < ncl;
    const int32_t bb = __shfl_sync(FULL, top, s & 31);
    const int32_t up = __shfl_up_sync(FULL, l, 1);
    const int32_t nu = lane == 0 ? bb : up;
    if (act) {
      const int32_t x = tv[lane][jj];
      int32_t v;
      uint32_t sy = 0;
      if ((pw >> jj) & 1u) {
        v = x;
      } else if (ENC) {
        const int32_t e = sm.etab[sm.tc[w][lane][jj] & 31];
        v = e > 0 ? bs_enc_exact(x, nu + l - ul, e, radius, &sy) : 0;
      } else {
        v = (int32_t)((uint32_t)nu + (uint32_t)l - (uint32_t)ul + (uint32_t)x);
      }
      tv[lane][jj] = v;
      if (ENC) sm.ts[w][lane][jj] = (uint16_t)sy;
      ul = nu;
      l = v;
    }
  }
  __syncwarp();
  int32_t* out = io.out[comp];
  for (int r = 0; r < nr; r++) {
    const int64_t k = (int64_t)(r0 + r) * io.Wp + c0 + lane;
    if (colok) out[k] = tv[r][lane];
  }
  if (ENC) {
    // symbols of the non-pinned (Lorenzo, non-lossless) pixels into the
    // stream; escapes (symbol 0) counted per row for the ll stream
    const int64_t pb = (int64_t)(r0 + (lane < nr ? lane : 0)) * io.nchunks + bj;
    const uint32_t nlr = lane < nr ? io.nlw[pb] : 0u;
    if (lane < nr)
      sm.tq[w][lane] = io.qd_row_off[r0 + lane] + 2 * (int64_t)io.pre_nl[pb];
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
    for (int r = 0; r < nr; r++) {
      const uint32_t pr_w = __shfl_sync(FULL, pw, r);
      const uint32_t nl_w = __shfl_sync(FULL, nlr, r);
      const bool put = colok && !((pr_w >> lane) & 1u);
      int esc = 0;
      if (put) {
        const uint16_t sy = sm.ts[w][r][lane];
        io.qd[sm.tq[w][r] + 2 * __popc(nl_w & lt) + comp] = sy;
        esc = sy == 0;
      }
      const int ne = __reduce_add_sync(FULL, esc);
      if (lane == 0 && ne) atomicAdd(io.row_ll + r0 + r, ne);
    }
  }
}

template <bool ENC>
__device__ __forceinline__ void bs_final_block(const BScanIO& io,
                                               uint32_t (*x)[33],
                                               int32_t (*v)[33],
                                               const int32_t* etab,
                                               const uint32_t* mtab, int bi,
                                               int bj, int comp, int lane);

template <bool ENC>
__global__ void __launch_bounds__(32 * BS_NW) bs_chain_kernel(BScanIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BSChainSmem& sm = *reinterpret_cast<BSChainSmem*>(smem_raw);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int H = io.H, W = io.W, nbx = io.nbx, nby = io.nby;
  const int64_t nblk = (int64_t)nbx * nby;
  const int ntask = bs_ntask(nby);
  if (threadIdx.x < 32) {
    sm.etab[threadIdx.x] = io.e_tab[threadIdx.x];
    sm.mtab[threadIdx.x] = io.mag_tab[threadIdx.x];
  }
  for (;;) {
    if (threadIdx.x == 0) sm.task = atomicAdd(io.ticket, 1);
    if (threadIdx.x < BS_NW) sm.done[threadIdx.x] = 0;
    for (int k = threadIdx.x; k < (BS_NW + 1) * BS_HRING; k += blockDim.x)
      (&sm.hin[0][0])[k] = 0;
    __syncthreads();
    const int task = sm.task;
    if (task >= ntask) {
      // ---- interior tasks: (segment of BS_SEG blocks, block row, comp) in
      // the order the chain finishes them (segment-major: segment s of row
      // bi is done at ~ bi * lag + (s + 1) * BS_SEG * step), each started
      // once the chain has finished the segment in its row and in the row
      // above
      const int nseg = (nbx + BS_SEG - 1) / BS_SEG;
      const int ft = task - ntask;
      if (ft >= 2 * nby * nseg) break;
      const int comp = ft & 1, rs = ft >> 1;
      const int sg = rs / nby, bi = rs - sg * nby;
      const int b0 = sg * BS_SEG, b1 = min(nbx, b0 + BS_SEG);
      if (threadIdx.x == 0) {
        const unsigned long long need = ((unsigned long long)io.frame_tag << 32) | (unsigned)b1;
        for (int r = bi; r >= bi - 1 && r >= 0; r--) {
          const volatile unsigned long long* pg = io.prog + (int64_t)comp * nby + r;
          long long spins = 0;
          while (*pg < need) {
            __nanosleep(128);
            if (++spins > (1ll << 28)) __trap();   // never: a hang guard
          }
        }
        __threadfence();
      }
      __syncthreads();
      for (int bj = b0 + w; bj < b1; bj += BS_NW)
        bs_final_block<ENC>(io, sm.fin.x[w], sm.fin.v[w], sm.etab, sm.mtab, bi,
                            bj, comp, lane);
      __syncthreads();
      continue;
    }
    const int g = task >> 1, comp = task & 1;
    const int bi = g * BS_NW + w;
    if (bi < nby) {
      const int r0 = 32 * bi;
      const int nr = min(32, H - r0);
      const bool has_next = bi + 1 < nby;
      const bool out_smem = has_next && w + 1 < BS_NW;
      const uint32_t tag_me = io.tag_base + (uint32_t)task + 1u;
      const uint32_t tag_up = io.tag_base + (uint32_t)task - 1u;   // task - 2
      uint64_t* my_gb = io.bnd + (int64_t)task * W;
      const uint64_t* up_gb = io.bnd + (int64_t)(task - 2) * W;
      const int32_t* clsp = io.cls + comp * nblk + (int64_t)bi * nbx;
      const int32_t* lbp = io.lb + (comp * nblk + (int64_t)bi * nbx) * 32;
      const int32_t* lrp = io.lr + (comp * nblk + (int64_t)bi * nbx) * 32;
      int32_t left = 0, corner = 0;
      // first warp of a CTA (row above in another CTA): the tagged slots of
      // the next two blocks are loaded ahead, so a block step does not pay
      // an L2 round trip whenever the CTA above is ahead
      const bool gtop = w == 0 && bi > 0;
      uint64_t g0 = 0, g1 = 0;
      if (gtop) {
        if (lane < W) g0 = ld_relaxed_u64(up_gb + lane);
        if (32 + lane < W) g1 = ld_relaxed_u64(up_gb + 32 + lane);
      }
      // (class, LB, LR) of the next BS_PF blocks in flight (cp.async ring):
      // they do not depend on the recurrence, so the block step never waits
      // on DRAM
      auto stage = [&](int b) {
        // branch-free: lanes 0-15 copy LB / LR (16 bytes each), lane 16 the
        // class word; the other lanes' copies are empty and land in a sink
        const bool vb = b < nbx;
        const int s = b % BS_PF, bb = vb ? b : 0;
        int32_t* d16 = lane < 16 ? &sm.pf[w][s][4 * lane] : &sm.pfd[w][lane][0];
        const int32_t* s16 = lane < 8 ? lbp + 32 * bb + 4 * lane
                                      : lrp + 32 * bb + 4 * ((lane - 8) & 7);
        cp_async<16>(d16, s16, vb && lane < 16);
        int32_t* d4 = lane == 16 ? &sm.pfc[w][s] : &sm.pfd[w][lane][0];
        cp_async<4>(d4, clsp + bb, vb && lane == 16);
        cp_async_commit();
      };
#pragma unroll 1
      for (int b = 0; b < BS_PF; b++) stage(b);
      auto stamp = [&](int k) {
        if (io.stamps && lane == 0) {
          unsigned long long tn;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
          io.stamps[((int64_t)comp * nby + bi) * 3 + k] = tn;
        }
      };
      stamp(0);
      for (int bj = 0; bj < nbx; bj++) {
        const int c0 = 32 * bj;
        const int ncl = min(32, W - c0);
        const int c = c0 + lane;
        const bool colok = lane < ncl;
        cp_async_wait_group<BS_PF - 1>();
        __syncwarp();
        const int slot = bj % BS_PF;
        const int32_t cls = sm.pfc[w][slot];
        const int32_t lbv = sm.pf[w][slot][lane], lrv = sm.pf[w][slot][32 + lane];
        __syncwarp();
        stage(bj + BS_PF);
        // ---- hand a bottom row to the block row below
        auto publish = [&](int32_t b) {
          if (!has_next) return;
          if (out_smem) {
            // ring slots of block bj - HRING/32 must have been read (the
            // reads fed the consumer's computation before it bumped its
            // counter)
            if (bj >= BS_HRING / 32 - 1)
              while (!__all_sync(FULL, *(volatile int*)&sm.done[w + 1] >=
                                           bj - (BS_HRING / 32 - 1))) {
              }
            if (colok)
              sm.hin[w + 1][c & (BS_HRING - 1)] = ((uint64_t)(c + 1) << 32) | (uint32_t)b;
          } else if (colok) {
            TaggedSlot<int32_t>::put(my_gb + c, tag_me, b);
          }
        };
        // ---- everything that does not need the row above, before waiting
        const int kind0 = cls & 3;
        const int32_t ll = __shfl_sync(FULL, left, nr - 1);
        uint32_t e = 0, m = 2, M = 0, pb = 0, pr = 0;
        if (kind0 == BS_REG) {
          if (ENC) {
            const int code = cls >> 2;
            e = (uint32_t)sm.etab[code];
            m = 2u * e;
            M = sm.mtab[code];
            const uint32_t rc = bs_res(corner, m, M);
            pb = bs_madd(bs_res(ll, m, M), bs_msub((uint32_t)lbv, rc, m), m);
            pr = bs_madd(bs_res(left, m, M), bs_msub((uint32_t)lrv, rc, m), m);
          } else {
            pb = (uint32_t)ll - (uint32_t)corner + (uint32_t)lbv;
            pr = (uint32_t)left - (uint32_t)corner + (uint32_t)lrv;
          }
        }
        // ---- the exact row above the block
        int32_t top = 0;
        if (bi > 0) {
          if (gtop) {
            uint64_t wv = colok ? g0 : 0;
            bool ok = !colok || (uint32_t)(wv >> 32) == tag_up;
            while (!__all_sync(FULL, ok)) {
              if (!ok) {
                wv = ld_relaxed_u64(up_gb + c);
                ok = (uint32_t)(wv >> 32) == tag_up;
              }
            }
            top = (int32_t)(uint32_t)wv;
            g0 = g1;
            g1 = c + 64 < W ? ld_relaxed_u64(up_gb + c + 64) : 0;
          } else {
            const volatile uint64_t* ep = &sm.hin[w][c & (BS_HRING - 1)];
            uint64_t v = colok ? *ep : 0;
            bool ok = !colok || (uint32_t)(v >> 32) == (uint32_t)(c + 1);
            while (!__all_sync(FULL, ok)) {
              if (!ok) {
                v = *ep;
                ok = (uint32_t)(v >> 32) == (uint32_t)(c + 1);
              }
            }
            top = colok ? (int32_t)(uint32_t)v : 0;
          }
          if (!colok) top = 0;
        }
        if (bj == 0) stamp(1);
        int kind = kind0;
        int32_t bot = 0, right = 0;
        bool published = false;
        if (kind == BS_REG) {
          if (ENC) {
            // the bottom row is exact unless one of its own residues is a
            // tie: hand it down first, the right column after
            const uint32_t rb = bs_madd(bs_res(top, m, M), pb, m);
            const bool btie = __any_sync(FULL, colok && rb == e);
            if (!btie) {
              bot = colok ? bs_rep(rb, e, m) : 0;
              publish(bot);
              published = true;
            }
            const int32_t tl = __shfl_sync(FULL, top, ncl - 1);
            const uint32_t rr = bs_madd(pr, bs_res(tl, m, M), m);
            const bool rtie = __any_sync(FULL, lane < nr && rr == e);
            if (btie || rtie) kind = BS_SLOW;
            else right = bs_rep(rr, e, m);
          } else {
            bot = colok ? (int32_t)((uint32_t)top + pb) : 0;
            publish(bot);
            published = true;
            const int32_t tl = __shfl_sync(FULL, top, ncl - 1);
            right = (int32_t)(pr + (uint32_t)tl);
          }
        } else if (kind == BS_KNOWN) {
          bot = lbv;
          right = lrv;
        }
        if (kind == BS_SLOW) {
          bs_slow_block<ENC>(io, sm, w, comp, bi, bj, nr, ncl, top, left, corner, lane);
          bot = sm.tv[w][nr - 1][lane];
          right = sm.tv[w][lane][ncl - 1];
          if (lane == 0) io.cls[comp * nblk + (int64_t)bi * nbx + bj] = BS_DONE;
          __syncwarp();
        }
        if (!colok) bot = 0;
        if (lane >= nr) right = 0;
        if (!published) publish(bot);
        // ---- the block's exact edges for the interior pass (coalesced)
        {
          const int64_t eo = (comp * nblk + (int64_t)bi * nbx + bj) * 32 + lane;
          io.ebot[eo] = bot;
          io.eright[eo] = right;
        }
        if (lane == 0) *(volatile int*)&sm.done[w] = bj + 1;
        // progress for the interior tasks: the block edges (and any swept
        // block) are visible GPU-wide before the mark
        if ((bj + 1) % BS_SEG == 0 || bj + 1 == nbx) {
          __threadfence();
          __syncwarp();
          if (lane == 0)
            *(volatile unsigned long long*)(io.prog + (int64_t)comp * nby + bi) =
                ((unsigned long long)io.frame_tag << 32) | (unsigned)(bj + 1);
        }
        corner = __shfl_sync(FULL, top, 31);
        left = right;
      }
      stamp(2);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ phase C
// CTA = one block, warp = component.
// The interior of block (bi, bj), component comp, by one warp (lane =
// column); x, v: the warp's shared tiles.
template <bool ENC>
__device__ __forceinline__ void bs_final_block(const BScanIO& io,
                                               uint32_t (*x)[33],
                                               int32_t (*v)[33],
                                               const int32_t* etab,
                                               const uint32_t* mtab, int bi,
                                               int bj, int comp, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, io.H - r0), ncl = min(32, io.W - c0);
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int32_t cls = __ldcg(io.cls + comp * nblk + blk);
  const int kind = cls & 3;
  const int Wp = io.Wp;
  const int32_t* a = io.a[comp];
  int32_t* out = io.out[comp];
  const bool colok = lane < ncl;
  // decoder: the finished recon = Z + p goes to the recon plane (the next
  // frame's p) and out as float64 (codec.py:425-426 recon * (1/S), exact),
  // optionally as int64
  const int32_t* pv = ENC ? nullptr : io.prev[comp];
  // p of the block's rows, loaded up front (all loads in flight before the
  // stores below, which the compiler cannot reorder them past)
  int32_t pp[ENC ? 1 : 32];
  if (!ENC) {
#pragma unroll
    for (int r = 0; r < 32; r++)
      pp[ENC ? 0 : r] = (pv && r < nr && colok) ? __ldg(pv + (int64_t)(r0 + r) * Wp + c0 + lane) : 0;
  }
  auto emit = [&](int r, int32_t z) {
    if (!ENC) {
      const int32_t val = (int32_t)((uint32_t)z + (uint32_t)pp[ENC ? 0 : r]);
      out[(int64_t)(r0 + r) * Wp + c0 + lane] = val;
      const int64_t k = (int64_t)(r0 + r) * io.W + c0 + lane;
      io.f64[comp][k] = __dmul_rn((double)val, io.inv_S);
      if (io.fix[comp]) io.fix[comp][k] = val;
    }
  };
  if (kind == BS_DONE || kind == BS_SLOW) {   // warp-uniform
    // swept by the chain kernel
    if (!ENC) {
      int32_t zz[32];
#pragma unroll
      for (int r = 0; r < 32; r++)
        zz[r] = (r < nr && colok) ? __ldcg(out + (int64_t)(r0 + r) * Wp + c0 + lane) : 0;
#pragma unroll
      for (int r = 0; r < 32; r++)
        if (r < nr && colok) emit(r, zz[r]);
    }
    return;
  }
  int32_t xa[32];
#pragma unroll
  for (int r = 0; r < 32; r++)
    xa[r] = (r < nr && colok) ? __ldg(a + (int64_t)(r0 + r) * Wp + c0 + lane) : 0;
  if (kind == BS_KNOWN) {
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (r < nr && colok) {
        if (ENC) out[(int64_t)(r0 + r) * Wp + c0 + lane] = xa[r];
        else emit(r, xa[r]);
      }
    }
    return;
  }
  // ---- exact boundary from phase B
  const int32_t* eb = io.ebot + comp * nblk * 32;
  const int32_t* er = io.eright + comp * nblk * 32;
  const int32_t top = (bi > 0 && colok) ? __ldcg(eb + (blk - io.nbx) * 32 + lane) : 0;
  const int32_t left = (bj > 0 && lane < nr) ? __ldcg(er + (blk - 1) * 32 + lane) : 0;
  const int32_t corner = (bi > 0 && bj > 0) ? __ldcg(eb + (blk - io.nbx - 1) * 32 + 31) : 0;
  uint32_t e = 0, m = 0, M = 0;
  if (ENC) {
    const int code = cls >> 2;
    e = (uint32_t)etab[code];
    m = 2u * e;
    M = mtab[code];
  }
#pragma unroll
  for (int r = 0; r < 32; r++) x[r][lane] = ENC ? bs_negres(xa[r], m, M) : (uint32_t)xa[r];
  v[0][lane + 1] = top;
  v[lane + 1][0] = left;
  if (lane == 0) v[0][0] = corner;
  __syncwarp();
  {  // row prefix (lane = row), then column prefix (lane = column)
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) {
      acc = ENC ? bs_madd(acc, x[lane][k], m) : acc + x[lane][k];
      x[lane][k] = acc;
    }
    __syncwarp();
    acc = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) {
      acc = ENC ? bs_madd(acc, x[k][lane], m) : acc + x[k][lane];
      x[k][lane] = acc;
    }
    __syncwarp();
  }
  if (!ENC) {
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (r < nr && colok) {
        const uint32_t val = (uint32_t)top + (uint32_t)v[r + 1][0] - (uint32_t)corner + x[r][lane];
        emit(r, (int32_t)val);
      }
    }
    return;
  }
  const uint32_t rt = bs_res(top, m, M), rc = bs_res(corner, m, M);
  const uint32_t base = bs_msub(rt, rc, m);
  const uint32_t rl = bs_res(left, m, M);   // lane r: row r's left residue
  // representatives; a tie (residue e) is marked and resolved below
  uint32_t tierows = 0;
#pragma unroll
  for (int r = 0; r < 32; r++) {
    const uint32_t s = bs_madd(bs_madd(base, __shfl_sync(FULL, rl, r), m), x[r][lane], m);
    const bool tie = s == e && r < nr && colok;
    tierows |= (__any_sync(FULL, tie) ? 1u : 0u) << r;
    v[r + 1][lane + 1] = tie ? INT32_MIN : bs_rep(s, e, m);
  }
  __syncwarp();
  if (tierows) {
    // raster order: a tie's sign follows x = R0 - (vU + vL - vUL), whose
    // neighbours may be earlier ties
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (!((tierows >> r) & 1u)) continue;   // warp-uniform
      uint32_t tm = __ballot_sync(FULL, colok && v[r + 1][lane + 1] == INT32_MIN);
      while (tm) {
        const int j = __ffs(tm) - 1;
        tm &= tm - 1u;
        if (lane == j) {
          const int64_t d = (int64_t)v[r][j + 1] + v[r + 1][j] - v[r][j];
          v[r + 1][j + 1] = ((int64_t)xa[r] - d) > 0 ? (int32_t)e : -(int32_t)e;
        }
        __syncwarp();
      }
    }
  }
  const int32_t radius = io.radius;
  // every pixel of a regular block is a non-lossless Lorenzo pixel: row r's
  // symbols are contiguous in the stream
  int64_t qb = 0;
  if (lane < nr)
    qb = io.qd_row_off[r0 + lane] +
         2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] + comp;
  int32_t* op = out + (int64_t)r0 * Wp + c0 + lane;
#pragma unroll
  for (int r = 0; r < 32; r++, op += Wp) {
    const int64_t qr = __shfl_sync(FULL, qb, r);
    if (r < nr && colok) {
      // x + err = q * 2e exactly; int32 is exact here (|R0| < 2^30 in a
      // regular block, |vU + vL - vUL - err| < 2^30)
      const int32_t err = v[r + 1][lane + 1];
      const int32_t d = v[r][lane + 1] + v[r + 1][lane] - v[r][lane];
      const int32_t n = xa[r] - d + err;
      const uint32_t an = (uint32_t)(n < 0 ? -n : n);
      uint32_t qa = __umulhi(an, M);
      if (qa * m != an) qa++;
      const int32_t q = n < 0 ? -(int32_t)qa : (int32_t)qa;
      *op = err;
      io.qd[qr + 2 * lane] = (uint16_t)(q + radius);
    }
  }
}

template <bool ENC>
cudaError_t launch_bs_local(const BScanIO& io, cudaStream_t st) {
  bs_local_kernel<ENC><<<dim3(io.nbx, io.nby), 64, 0, st>>>(io);
  return cudaGetLastError();
}

template <bool ENC>
cudaError_t launch_bs_chain(const BScanIO& io, int nsm, cudaStream_t st) {
  const size_t smem = sizeof(BSChainSmem);
  cudaError_t e = cudaFuncSetAttribute(
      bs_chain_kernel<ENC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bs_chain_kernel<ENC>,
                                                    32 * BS_NW, smem);
  if (e != cudaSuccess) return e;
  const int ntask = bs_ntask(io.nby) +
                    2 * io.nby * ((io.nbx + BS_SEG - 1) / BS_SEG);
  // persistent: every CTA is resident; tickets hand out the chain tasks
  // (block-row order) first, then the interior tasks
  bs_chain_kernel<ENC><<<min(max(occ, 1) * nsm, ntask), 32 * BS_NW, smem, st>>>(io);
  return cudaGetLastError();
}


}  // namespace vfcp
