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
#include <type_traits>

#include "common.cuh"
#include "wavefront.cuh"

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

// The same with 16 codes per lane and step (rows of a multiple of 16
// columns, 16-byte aligned): a code is lossless iff it is >= cmax (the bit
// length of tau; 0 when tau <= 0), compared four bytes at a time; the l_d bits
// of 16 pixels are two bytes, most significant bit first.
__global__ void decode_rows16_kernel(const uint8_t* __restrict__ codes,
                                     const uint8_t* __restrict__ ld,
                                     int64_t nrows, int W, int cmax,
                                     int32_t* __restrict__ row_n31,
                                     int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int64_t rb = row * W;
  const uint4* cr = reinterpret_cast<const uint4*>(codes + rb);
  const uint16_t* lr = ld ? reinterpret_cast<const uint16_t*>(ld + (rb >> 3)) : nullptr;
  const uint32_t cm4 = 0x01010101u * (uint32_t)cmax;
  int n31 = 0;
  bool mismatch = false;
  const int nq = W >> 4;
  for (int q = lane; q < nq; q += 32) {
    const uint4 c = __ldg(cr + q);
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    uint32_t bits = 0;   // pixel 0 in bit 15
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t ge = __vcmpgeu4(w[k], cm4) & 0x01010101u;
      n31 += __popc(ge);
      bits = (bits << 4) | ((ge * 0x08040201u) >> 24);
    }
    if (lr) {
      const uint32_t l2 = __ldg(lr + q);   // bytes k/8, k/8 + 1 (little endian)
      const uint32_t want = ((l2 & 0xffu) << 8) | (l2 >> 8);
      mismatch |= want != bits;
    }
  }
  for (int o = 16; o; o >>= 1) n31 += __shfl_xor_sync(0xffffffffu, n31, o);
  if (__any_sync(0xffffffffu, mismatch) && lane == 0) atomicOr(bad, 1);
  if (lane == 0) row_n31[row] = n31;
}

// Escapes (symbol 0) of a row's symbols, eight 16-bit symbols per lane and
// step where the row's range allows 16-byte loads.
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
  if (sizeof(SYM) == 2) {
    // head up to the first 16-byte boundary, 16-byte body, tail
    int64_t a8 = (a + 7) & ~(int64_t)7;
    if (a8 > b) a8 = b;
    const int64_t b8 = a8 + ((b - a8) & ~(int64_t)7);
    for (int64_t q = a + lane; q < a8; q += 32) z += qd[q] == 0;
    const uint4* body = reinterpret_cast<const uint4*>(qd + a8);
    const int64_t nv = (b8 - a8) >> 3;
    for (int64_t q = lane; q < nv; q += 32) {
      const uint4 x = __ldg(body + q);
      z += __popc(__vcmpeq2(x.x, 0u) & 0x00010001u) + __popc(__vcmpeq2(x.y, 0u) & 0x00010001u) +
           __popc(__vcmpeq2(x.z, 0u) & 0x00010001u) + __popc(__vcmpeq2(x.w, 0u) & 0x00010001u);
    }
    for (int64_t q = b8 + lane; q < b; q += 32) z += qd[q] == 0;
  } else {
    for (int64_t q = a + lane; q < b; q += 32) z += qd[q] == 0;
  }
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) row_ll[row] = z + 2 * row_n31[row];
}

// ---------------------------------------------------------------- decode
// Persistent, warp-specialised wavefront decoder (wavefront.cuh).
//
// A task (frame t, 32-row strip k) is run by a warp pair:
//   P (producer) stages one 32x32 chunk at a time with cp.async -- frame
//     t-1 (int recon frame, rows i0-1.., cols c0-1..), eb codes and the
//     chunk's compacted symbol words -- in ONE round trip, then computes per
//     pixel either a pin (lossless / escape / semi-Lagrangian pixels: value
//     known without neighbours) or the Lorenzo increment
//     A = Pd + (sym - radius) * 2e,  Pd = p - pU - pL + pUL  (frame t-1),
//     into a 3-chunk shared-memory ring; it also writes finished chunks out
//     (float64 recon * (1/S), codec.py:443-444, plus the int recon frame
//     the next frame reads) and publishes frame progress;
//   C (chain) runs the raster recurrence r = rU + rL - rUL + A
//     (codec.py:167-206 with predictors.py:62-73) as an anti-diagonal sweep,
//     lane = row, exchanging the strip's last row with the strip below
//     through tagged slots.
// Only C is on the wavefront's critical path; P runs a chunk ahead.
// Arithmetic is modulo 2^w (w = bits of IW): intermediate sums may wrap but
// every reconstruction fits IW.
constexpr int NC = 3;             // ring chunks per pair
constexpr int PROG_EVERY = 4;     // chunks between frame-progress releases

template <typename IW, typename SYM>
struct PairSmem {
  static constexpr int WPP = sizeof(SYM) / 2;   // 32-bit words per pixel
  // ring element (row, col) lives at [row][col ^ row]: conflict-free for
  // P's row-wise and write-out column-wise accesses, <= 2-way for C's
  // anti-diagonal sweep
  IW ring[NC][2][32][32];
  uint32_t pinw[NC][32][3];       // [slot][row][u pins, v pins, pad]
  IW stg_p[2][33][33];            // frame t-1: rows i0-1.., cols c0-1..
  uint32_t stg_sy[32][32 * WPP + 1];  // compacted symbol words of each row
  uint32_t stg_cd[32][9];         // eb codes, 4 per word
  int64_t etab[32];               // e per ladder code
  IW bnd[2][32];                  // C: row i0-1 for the current step block
  int task;                       // ticket of the current task, -1 = exit
  int full;                       // chunks precomputed (this task)
  int done;                       // step blocks chained (this task)
};

template <typename IW>
using UW = typename std::conditional<sizeof(IW) == 4, uint32_t, uint64_t>::type;

__device__ __forceinline__ void pair_bar(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ int vload(const int* p) {
  return *(volatile const int*)p;
}
__device__ __forceinline__ void vstore(int* p, int v) {
  *(volatile int*)p = v;
}
// warp-uniform spin on a shared-memory counter, then acquire
__device__ __forceinline__ void wait_smem_ge(const int* p, int need, int lane) {
  (void)lane;
  while (!__all_sync(0xffffffffu, vload(p) >= need)) __nanosleep(20);
  __threadfence_block();
}
__device__ __forceinline__ void signal_smem(int* p, int v, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    vstore(p, v);
  }
}
__device__ __forceinline__ int mod3(int x) { return x - 3 * ((x * 0xAAAB) >> 17); }

template <typename IW, typename SYM, int NP>
__global__ void __launch_bounds__(64 * NP, 1)
wf_decode_kernel(const uint8_t* __restrict__ codes, const SYM* __restrict__ qd,
                 const int64_t* __restrict__ ll,
                 const uint8_t* __restrict__ modes, DecodeParams p, Ladder lad,
                 const int64_t* __restrict__ qd_row_off,
                 const int64_t* __restrict__ ll_row_off, double* out_u,
                 double* out_v, int64_t* __restrict__ fix_u,
                 int64_t* __restrict__ fix_v, IW* rec, int Wp,
                 uint64_t* bnd_g, WaveSched ws, int reach_rows) {
  typedef UW<IW> U;
  typedef TaggedSlot<IW> TS;
  typedef PairSmem<IW, SYM> SM;
  constexpr int WPP = SM::WPP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pair = wid >> 1;
  const bool producer = (wid & 1) == 0;
  SM& sm = reinterpret_cast<SM*>(smem_raw)[pair];
  const int H = p.H, W = p.W, T = p.T, K = ws.K;
  const int64_t HW = (int64_t)H * W;
  const int64_t HWp = (int64_t)H * Wp;
  const int nchunks = (W + 31) / 32;
  const int nblocks = (W + 31 + 31) / 32;
  const unsigned FULL = 0xffffffffu;
  const int64_t nblk = (int64_t)p.nbx * ((H + p.by - 1) / p.by);
  const int bar_id = 1 + pair;
  const bool codes_vec = (W & 3) == 0;
  const uint32_t* qd32 = reinterpret_cast<const uint32_t*>(qd);
  const int64_t nqd_words = p.n_qd / 2;

  if (producer) sm.etab[lane] = lad.e[lane];
  int64_t qpos = 0, lpos = 0;   // P: stream cursors of row `lane`
  for (;;) {
    if (producer) {
      int tk = 0;
      if (lane == 0) tk = atomicAdd(ws.ticket, 1);
      tk = __shfl_sync(FULL, tk, 0);
      if (tk < T * K) {
        const int t = tk / K, k = tk - t * K;
        const int i = 32 * k + lane;
        if (i < H) {
          qpos = qd_row_off[(int64_t)t * H + i];
          lpos = ll_row_off[(int64_t)t * H + i];
        }
      }
      if (lane == 0) {
        sm.task = tk < T * K ? tk : -1;
        sm.full = 0;
        sm.done = 0;
      }
      __threadfence_block();
    }
    pair_bar(bar_id);
    const int tk = vload(&sm.task);
    if (tk < 0) break;
    const int t = tk / K, k = tk - t * K;
    const uint32_t tag = (uint32_t)tk + 1u;
    const int i0 = 32 * k;
    const int nrows = min(32, H - i0);
    const int64_t fb = (int64_t)t * HW;

    if (producer) {
      // ================================================== producer warp
      PhaseClock pc(ws.stats);
      const IW* rpu = rec + (2 * (int64_t)t - 2) * HWp;   // frame t-1
      const IW* rpv = rpu + HWp;
      IW* rcu = rec + 2 * (int64_t)t * HWp;              // frame t
      IW* rcv = rcu + HWp;
      const IntSrcCG<IW> su{rpu}, sv{rpv};
      const uint8_t* modes_t = t >= 1 ? modes + (int64_t)(t - 1) * nblk : nullptr;
      const bool sl_frame = p.use_modes && t >= 1;
      const int rr = sl_frame ? reach_rows : 0;
      const int klo = max(0, (i0 - 1 - rr) / 32);
      const int khi = min(K - 1, (i0 + 31 + rr) / 32);
      const int reach_c = sl_frame ? ws.reach_cols : 0;
      int next_pre = 0, next_out = 0;
      while (next_out < nchunks) {
        if (next_pre < nchunks && next_pre - next_out < NC) {
          const int m = next_pre;
          const int c0 = 32 * m;
          const int slot = mod3(m);
          if (t > 0) {
            const int need = min(W, c0 + 32 + reach_c);
            for (int kk = klo; kk <= khi; kk++)
              wait_ge(ws.prog + (t - 1) * K + kk, need, lane);
          }
          pc.lap(WP_WAITPREV, lane);
          // ---- stage the chunk (one round trip); lane = row r
          const int r = lane;
          const bool rv = r < nrows;
          {
            const int i = i0 + r;
            const int64_t o = (int64_t)(rv ? i : 0) * Wp;
            const int64_t oup = (int64_t)(i0 > 0 ? i0 - 1 : 0) * Wp;
#pragma unroll 3
            for (int q = 0; q < 33; q++) {
              const int c = c0 - 1 + q;
              const bool cv = t > 0 && c >= 0 && c < W;
              const int cc = cv ? c : 0;
              cp_async<sizeof(IW)>(&sm.stg_p[0][r + 1][q], rpu + o + cc, cv && rv);
              cp_async<sizeof(IW)>(&sm.stg_p[1][r + 1][q], rpv + o + cc, cv && rv);
              if (lane == 0) {
                cp_async<sizeof(IW)>(&sm.stg_p[0][0][q], rpu + oup + cc, cv && i0 > 0);
                cp_async<sizeof(IW)>(&sm.stg_p[1][0][q], rpv + oup + cc, cv && i0 > 0);
              }
            }
            const int64_t rowb = fb + (int64_t)(rv ? i : i0) * W + c0;
            if (codes_vec && c0 + 32 <= W) {
#pragma unroll
              for (int q = 0; q < 8; q++)
                cp_async<4>(&sm.stg_cd[r][q], codes + rowb + 4 * q, rv);
            } else if (rv) {
              for (int q = 0; q < 8; q++) {
                uint32_t wd = 0;
                for (int b = 0; b < 4; b++) {
                  const int c = c0 + 4 * q + b;
                  const uint32_t cd = c < W ? codes[rowb + 4 * q + b] : CODE_LOSSLESS;
                  wd |= cd << (8 * b);
                }
                sm.stg_cd[r][q] = wd;
              }
            }
            const int64_t qw = qpos / 2;
#pragma unroll 4
            for (int q = 0; q < 32 * WPP; q++) {
              const int64_t w = qw + q;
              cp_async<4>(&sm.stg_sy[r][q], qd32 + (w < nqd_words ? w : 0),
                          rv && w < nqd_words);
            }
          }
          // semi-Lagrangian block mask of row r over the chunk's columns
          uint32_t mmask = 0;
          if (sl_frame && rv) {
            const int64_t mrow = (int64_t)((i0 + r) / p.by) * p.nbx;
            const int cl = min(W, c0 + 32);
            for (int b = c0 / p.bx; b * p.bx < cl; b++) {
              if (modes_t[mrow + b]) {
                const int a0 = max(c0, b * p.bx) - c0;
                const int a1 = min(cl, (b + 1) * p.bx) - c0;   // exclusive
                const uint32_t hi = a1 >= 32 ? 0xffffffffu : ((1u << a1) - 1u);
                mmask |= hi & ~((1u << a0) - 1u);
              }
            }
          }
          cp_async_wait_all();
          __syncwarp();
          pc.lap(WP_X3, lane);
          // ---- per-pixel values: each lane scans its own row (no warp
          // collectives; stream cursors live in registers)
          uint32_t pins_u = 0, pins_v = 0;
          if (rv) {
            const int i = i0 + r;
            const int ncol = min(32, W - c0);
            const uint32_t colmask = ncol >= 32 ? 0xffffffffu : ((1u << ncol) - 1u);
            // pass 1: codes -> non-lossless mask (independent per pixel)
            uint32_t nlm = 0;
#pragma unroll
            for (int jc = 0; jc < 32; jc++) {
              const int cd = (sm.stg_cd[r][jc >> 2] >> (8 * (jc & 3))) & 31;
              nlm |= (sm.etab[cd] != 0 ? 1u : 0u) << jc;
            }
            nlm &= colmask;
            // pass 2: symbols by compacted index -> escape masks
            uint32_t eum = ~nlm & colmask, evm = ~nlm & colmask;
#pragma unroll
            for (int jc = 0; jc < 32; jc++) {
              const int wq = __popc(nlm & ((1u << jc) - 1u));
              const bool nl = (nlm >> jc) & 1u;
              uint32_t a, b;
              if (WPP == 1) {
                const uint32_t w2 = nl ? sm.stg_sy[r][wq] : 1u;
                a = w2 & 0xffffu; b = w2 >> 16;
              } else {
                a = nl ? sm.stg_sy[r][2 * wq] : 1u;
                b = nl ? sm.stg_sy[r][2 * wq + 1] : 1u;
              }
              eum |= (nl && a == 0) ? (1u << jc) : 0u;
              evm |= (nl && b == 0) ? (1u << jc) : 0u;
            }
            // pass 3: values (independent per pixel)
#pragma unroll 8
            for (int jc = 0; jc < 32; jc++) {
              if (jc >= ncol) break;
              const int j = c0 + jc;
              const uint32_t below = (1u << jc) - 1u;
              const bool nl = (nlm >> jc) & 1u;
              const bool eu = (eum >> jc) & 1u, ev = (evm >> jc) & 1u;
              const int64_t lu = lpos + __popc(eum & below) + __popc(evm & below);
              const int64_t lv = lu + (eu ? 1 : 0);
              VFCP_CHECK(!(eu || ev) || (lu >= 0 && lv + (ev ? 1 : 0) <= p.n_ll), "ll index");
              const int wq = __popc(nlm & below);
              int64_t syu = 0, syv = 0;
              if (nl) {
                if (WPP == 1) {
                  const uint32_t w2 = sm.stg_sy[r][wq];
                  syu = w2 & 0xffffu; syv = w2 >> 16;
                } else {
                  syu = sm.stg_sy[r][2 * wq]; syv = sm.stg_sy[r][2 * wq + 1];
                }
              }
              const int cd = (sm.stg_cd[r][jc >> 2] >> (8 * (jc & 3))) & 31;
              const int64_t e = sm.etab[cd];
              const bool sl_px = nl && ((mmask >> jc) & 1u);
              const int64_t two_e = 2 * e;
              const int64_t qu = syu - p.radius;
              const int64_t qv = syv - p.radius;
              U val_u = (U)sm.stg_p[0][r + 1][jc + 1] - (U)sm.stg_p[0][r][jc + 1] -
                        (U)sm.stg_p[0][r + 1][jc] + (U)sm.stg_p[0][r][jc] + (U)(qu * two_e);
              U val_v = (U)sm.stg_p[1][r + 1][jc + 1] - (U)sm.stg_p[1][r][jc + 1] -
                        (U)sm.stg_p[1][r + 1][jc] + (U)sm.stg_p[1][r][jc] + (U)(qv * two_e);
              if (sl_px) {
                double fi, fj;
                sl_departure_src(su, sv, H, W, i, j, p.cfl_x, p.cfl_y,
                                 p.d_max, p.n_max, &fi, &fj, Wp);
                BilinearTap tp = bilinear_tap(H, W, fi, fj, Wp);
                val_u = (U)(bilinear_src(tp, su) + qu * two_e);
                val_v = (U)(bilinear_src(tp, sv) + qv * two_e);
              }
              if (eu) val_u = (U)ll[lu];
              if (ev) val_v = (U)ll[lv];
              sm.ring[slot][0][r][jc ^ r] = (IW)val_u;
              sm.ring[slot][1][r][jc ^ r] = (IW)val_v;
            }
            pins_u = eum | (nlm & mmask);
            pins_v = evm | (nlm & mmask);
            qpos += 2 * __popc(nlm);
            lpos += __popc(eum) + __popc(evm);
            sm.pinw[slot][r][0] = pins_u;
            sm.pinw[slot][r][1] = pins_v;
          }
          signal_smem(&sm.full, m + 1, lane);
          next_pre++;
          pc.lap(WP_PRE, lane);
        } else {
          // write out chunk next_out once C has swept past it
          const int x = next_out;
          wait_smem_ge(&sm.done, min(x + 2, nblocks), lane);
          pc.lap(WP_WAITBND, lane);
          const int slot = mod3(x);
          const int j = 32 * x + lane;
          if (j < W) {
#pragma unroll 8
            for (int r = 0; r < 32; r++) {
              if (r >= nrows) break;
              const int64_t n = fb + (int64_t)(i0 + r) * W + j;
              const int64_t nr = (int64_t)(i0 + r) * Wp + j;
              const IW ru = sm.ring[slot][0][r][lane ^ r];
              const IW rv = sm.ring[slot][1][r][lane ^ r];
              out_u[n] = __dmul_rn((double)ru, p.inv_S);
              out_v[n] = __dmul_rn((double)rv, p.inv_S);
              rcu[nr] = ru;
              rcv[nr] = rv;
              if (fix_u) { fix_u[n] = ru; fix_v[n] = rv; }
            }
          }
          next_out++;
          if ((next_out % PROG_EVERY) == 0 || next_out == nchunks) {
            __syncwarp();
            if (lane == 0) publish(ws.prog + t * K + k, min(W, 32 * next_out));
          }
          pc.lap(WP_WRITE, lane);
        }
      }
    } else {
      // ================================================== chain warp
      PhaseClock pc(ws.stats);
      const int my_i = i0 + lane;
      const bool rowok = my_i < H;
      uint64_t* my_bnd = bnd_g + (int64_t)tk * 2 * W * TS::SLOTS;
      const uint64_t* up_bnd = bnd_g + (int64_t)(tk - 1) * 2 * W * TS::SLOTS;
      U rl_u = 0, rl_v = 0, rul_u = 0, rul_v = 0, rlast_u = 0, rlast_v = 0;
      for (int m = 0; m < nblocks; m++) {
        const int c0 = 32 * m;
        wait_smem_ge(&sm.full, min(m + 1, nchunks), lane);
        if (k > 0 && c0 < W) {
          const int c = c0 + lane;
          const bool v = c < W;
          const int cc = v ? c : 0;
          sm.bnd[0][lane] = TS::get(up_bnd + (int64_t)cc * TS::SLOTS, tag - 1, v);
          sm.bnd[1][lane] = TS::get(up_bnd + (int64_t)(W + cc) * TS::SLOTS, tag - 1, v);
        }
        __syncwarp();
        pc.lap(WP_WAITBND, lane);
        // This lane's 32 columns of the block, c = c0 - lane + jj, span at
        // most two chunks: pull values and pin bits into registers so the
        // dependent path per step is only shfl -> add -> select.
        const int cbase = c0 - lane;
        U av_u[32], av_v[32];
        uint32_t pin_u_lo = 0, pin_v_lo = 0, pin_u_hi = 0, pin_v_hi = 0;
        int s_lo = 0, s_hi = 0;
        {
          const int x_lo = cbase >= 0 ? (cbase >> 5) : -1;   // chunk of jj = 0
          s_lo = x_lo >= 0 ? mod3(x_lo) : 0;
          s_hi = mod3(x_lo + 1);
          if (rowok) {
            if (x_lo >= 0) {
              pin_u_lo = sm.pinw[s_lo][lane][0];
              pin_v_lo = sm.pinw[s_lo][lane][1];
            }
            if (32 * (x_lo + 1) < W) {
              pin_u_hi = sm.pinw[s_hi][lane][0];
              pin_v_hi = sm.pinw[s_hi][lane][1];
            }
          }
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            const int c = cbase + jj;
            const int sl = jj < 32 - (cbase & 31) ? s_lo : s_hi;
            const bool ok = rowok && c >= 0 && c < W;
            av_u[jj] = ok ? (U)sm.ring[sl][0][lane][(c & 31) ^ lane] : 0;
            av_v[jj] = ok ? (U)sm.ring[sl][1][lane][(c & 31) ^ lane] : 0;
          }
        }
        pc.lap(WP_X1, lane);
        // boundary row: lane l holds column c0 + l; lane 0 gathers it per step
        const U bu = (U)sm.bnd[0][lane], bv = (U)sm.bnd[1][lane];
        const uint32_t split = 32 - (cbase & 31);   // jj where the chunk changes
        const bool top = k > 0;
        // the warp must be converged here, or every shuffle of the sweep
        // takes the divergent (WARPSYNC.COLLECTIVE) path
        __syncwarp();
        // branch-free sweep: every lane runs the same instruction stream
#pragma unroll
        for (int jj = 0; jj < 32; jj++) {
          const int c = cbase + jj;
          const U b_u = __shfl_sync(FULL, bu, jj);
          const U b_v = __shfl_sync(FULL, bv, jj);
          const U up_u = __shfl_up_sync(FULL, rlast_u, 1);
          const U up_v = __shfl_up_sync(FULL, rlast_v, 1);
          const bool inb = c < W;
          const U ru_u = lane == 0 ? ((top && inb) ? b_u : 0) : up_u;
          const U ru_v = lane == 0 ? ((top && inb) ? b_v : 0) : up_v;
          const bool act = rowok && c >= 0 && inb;
          const bool lo = (uint32_t)jj < split;
          const uint32_t bit = 1u << (c & 31);
          const bool pu_ = ((lo ? pin_u_lo : pin_u_hi) & bit) != 0;
          const bool pv_ = ((lo ? pin_v_lo : pin_v_hi) & bit) != 0;
          const bool first = c == 0;
          const U rl0_u = first ? 0 : rl_u, rl0_v = first ? 0 : rl_v;
          const U rul0_u = first ? 0 : rul_u, rul0_v = first ? 0 : rul_v;
          const U r_u = pu_ ? av_u[jj] : ru_u + (rl0_u + (av_u[jj] - rul0_u));
          const U r_v = pv_ ? av_v[jj] : ru_v + (rl0_v + (av_v[jj] - rul0_v));
          av_u[jj] = act ? r_u : av_u[jj];
          av_v[jj] = act ? r_v : av_v[jj];
          rl_u = act ? r_u : rl_u;
          rl_v = act ? r_v : rl_v;
          rlast_u = rl_u;
          rlast_v = rl_v;
          rul_u = ru_u;
          rul_v = ru_v;
        }
        pc.lap(WP_X2, lane);
        // results back to the ring for the producer's write-out
#pragma unroll
        for (int jj = 0; jj < 32; jj++) {
          const int c = cbase + jj;
          if (rowok && c >= 0 && c < W) {
            const int sl = (uint32_t)jj < split ? s_lo : s_hi;
            sm.ring[sl][0][lane][(c & 31) ^ lane] = (IW)av_u[jj];
            sm.ring[sl][1][lane][(c & 31) ^ lane] = (IW)av_v[jj];
          }
        }
        // the strip's last row for the strip below: lane l publishes column
        // c0 - 31 + l of row 31 (written in this block), one tagged slot each
        if (k + 1 < K) {
          __syncwarp();
          const int c = c0 - 31 + lane;
          if (c >= 0 && c < W) {
            const int sl = mod3(c >> 5);
            TS::put(my_bnd + (int64_t)c * TS::SLOTS, tag,
                    sm.ring[sl][0][31][(c & 31) ^ 31]);
            TS::put(my_bnd + (int64_t)(W + c) * TS::SLOTS, tag,
                    sm.ring[sl][1][31][(c & 31) ^ 31]);
          }
        }
        signal_smem(&sm.done, m + 1, lane);
        pc.lap(WP_CHAIN, lane);
      }
    }
    if (producer && ws.stats && lane == 0) atomicAdd(ws.stats + WP_TASKS, 1ull);
    pair_bar(bar_id);   // both warps are done with this task's state
  }
}

// ------------------------------------------------------------ launchers
cudaError_t launch_decode_rows(const uint8_t* codes, const uint8_t* ld,
                               int64_t nrows, int W, int64_t tau,
                               int32_t* row_n31, int* bad, cudaStream_t st) {
  if ((W & 15) == 0 && ((uintptr_t)codes & 15) == 0 && ((uintptr_t)ld & 1) == 0) {
    int cmax = 0;   // codes below cmax quantise (e = tau >> code > 0)
    for (int c = 0; c < CODE_LOSSLESS; c++)
      if (tau > 0 && (tau >> c) != 0) cmax = c + 1;
    decode_rows16_kernel<<<(unsigned)((nrows + 7) / 8), 256, 0, st>>>(
        codes, ld, nrows, W, cmax, row_n31, bad);
    return cudaGetLastError();
  }
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

template <typename IW, typename SYM>
cudaError_t launch_decode(const uint8_t* codes, const SYM* qd,
                          const int64_t* ll, const uint8_t* modes,
                          const DecodeParams& p, const Ladder& lad,
                          const int64_t* qd_row_off,
                          const int64_t* ll_row_off, double* out_u,
                          double* out_v, int64_t* fix_u, int64_t* fix_v,
                          IW* rec, int Wp, uint64_t* bnd,
                          const WaveSched& ws, int reach_rows, int nsm,
                          cudaStream_t st) {
  constexpr int NP = sizeof(IW) == 4 ? 4 : 3;   // warp pairs per CTA
  size_t smem = sizeof(PairSmem<IW, SYM>) * NP;
  cudaError_t e = cudaFuncSetAttribute(
      wf_decode_kernel<IW, SYM, NP>,
      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int tasks = p.T * ws.K;
  int grid = min(nsm, (tasks + NP - 1) / NP);
  wf_decode_kernel<IW, SYM, NP><<<grid, 64 * NP, smem, st>>>(
      codes, qd, ll, modes, p, lad, qd_row_off, ll_row_off, out_u, out_v,
      fix_u, fix_v, rec, Wp, bnd, ws, reach_rows);
  return cudaGetLastError();
}

#define VFCP_INST_DEC(I, SYM)                                                 \
  template cudaError_t launch_decode<I, SYM>(                                 \
      const uint8_t*, const SYM*, const int64_t*, const uint8_t*,             \
      const DecodeParams&, const Ladder&, const int64_t*, const int64_t*,     \
      double*, double*, int64_t*, int64_t*, I*, int, uint64_t*,               \
      const WaveSched&, int, int,                                             \
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
