// The raster-order Lorenzo recurrence of one frame as a strip wavefront.
//
// Shared by the encoder (codec.py:118-164 _encode_frame) and the decoder
// (codec.py:167-206 _decode_frame).  Everything that does not depend on the
// current frame's reconstructed neighbours is computed beforehand, fully in
// parallel, by a prepare kernel; what is left is the recurrence through the
// up / left / up-left neighbours:
//
//   decoder (value form):  r = rU + rL - rUL + A,   A = Pd + (sym-radius)*2e
//   encoder (error form):  with err = recon - orig and
//     R0 = orig - Lorenzo(orig, prev)  (prepared),  D = errU + errL - errUL,
//     x = R0 - D,  q = rha(x / 2e),  err = q*2e - x  (0 on escape),
//     sym = q + radius  (0 on escape)
//
// The encoder never divides on the critical path: R0 is split once per
// pixel as R0 = Q0*2e + rho0, rho0 in [-e, e]; then y = rho0 - D lies in
// [-4e, 4e] and q = Q0 + g with g in {-2..2} found by four comparisons
// (ties -- y = +-e, +-3e -- round away from zero by the sign of x).
//
// A warp owns a 32-row strip (lane = row) and sweeps the columns with a
// one-column skew per lane, so the neighbours are final when read; a step
// is shfl -> a few integer ops -> select.  A CTA of CW warps owns CW
// consecutive strips and hands each strip's last row to the next warp
// through shared memory; CTAs (taken in row order by an atomic ticket, so a
// CTA only waits on an earlier, resident one) hand off through tagged
// global slots.  Inputs are staged per 32-column chunk with cp.async one
// chunk ahead of the sweep.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "wavefront.cuh"

namespace vfcp {

// Prepared planes (frame layout, row pitch Wp = 32 * nchunks):
//   a0, a1  int32 per component: decoder -- A or the pinned recon;
//           encoder -- R0 or the pinned err
//   pin_u, pin_v  uint32 per (row, chunk): bit j = pixel c0+j is pinned
//   nl      uint32 per (row, chunk): non-lossless (encoder: symbol slots)
//   symw    uint32 per (row, chunk): encoder: pixels whose symbols the chain
//           writes (non-lossless Lorenzo pixels)
struct ChainIO {
  const int32_t* a0;
  const int32_t* a1;
  const uint32_t* pin_u;
  const uint32_t* pin_v;
  const uint32_t* nl;
  const uint32_t* symw;
  const uint8_t* codes;      // frame t codes (pitch Wp), encoder
  int32_t* out_i0;           // decoder: recon; encoder: err (pitch Wp)
  int32_t* out_i1;
  double* out_f0;            // decoder: recon * inv_S (pitch W)
  double* out_f1;
  uint16_t* qd;              // encoder symbols
  const int64_t* qd_row_off; // per frame row
  const int32_t* chunk_nl;   // encoder: non-lossless count before each chunk
  int32_t* row_esc;          // encoder: escapes found by the chain, per row
  uint64_t* bnd;             // tagged last-row slots [ntask][2][W]
  unsigned long long* stats; // optional phase timers (WavePhase)
  int* ticket;
  uint32_t tag_base;          // tags unique across frames sharing `bnd`
  int H, W, Wp, nchunks;
  int radius;
  double inv_S;
  int32_t e_tab[32];         // e per code (encoder; requires tau' < 2^28)
  double inv2e_tab[32];
};

struct PrepParams {
  int H, W, Wp, nchunks, nbx, nby, t;
  double S, cfl_x, cfl_y, d_max, lam, theta, rmeta;
  int n_max, stride, radius;
  int64_t tau;
  int mop;          // run the MoP trial for this frame
  int force_sl;     // predictor 'sl' (and t >= 1, tau > 0)
  Ladder lad;
};

// warps (32-row strips) per chain CTA.  The per-frame chain is latency
// bound on its strip pipeline; one warp per CTA spreads the strips over all
// SMs (handoffs then go through the tagged global slots).
__host__ __device__ constexpr int chain_cw(bool enc) { return enc ? 1 : 1; }
constexpr int CNS = 3;   // chunk slots per warp: sweep uses m-1, m; m+1
                         // in flight; write-out reuses m-1 before m+2 lands
template <int CW>
struct ChainEncExtra {
  uint32_t sym[CW][CNS][32][32];      // symbol pair, ring layout
  uint32_t nl[CW][CNS][32];
  uint32_t symw[CW][CNS][32];
  uint32_t code[CW][CNS][32][8];      // [warp][slot][row][word] 4 codes/word
};
// decoder: never touched (the encoder branches are compiled but not run)
struct ChainNoExtra {
  uint32_t sym[1][1][1][1];
  uint32_t nl[1][1][1];
  uint32_t symw[1][1][1];
  uint32_t code[1][1][1][1];
};

template <int CW, bool ENC>
struct ChainSmem {
  int32_t ring[CW][CNS][2][32][32];   // [warp][slot][comp][row][col ^ row]
  uint32_t pin[CW][CNS][2][32];       // [warp][slot][comp][row]
  int32_t bnd[CW][4][2][32];          // [warp][chunk & 3][comp][col]: row 31
  int bdone[CW];                      // blocks whose row 31 is in bnd
  int bread[CW];                      // chunks of bnd[w-1] warp w consumed
  int task;
  typename std::conditional<ENC, ChainEncExtra<CW>, ChainNoExtra>::type x;
};

// exact rha(x / 2e) for integer x, e > 0, |x| < 2^31
__device__ __forceinline__ int32_t quant32(int32_t x, int32_t e, double inv2e) {
  const int32_t two_e = 2 * e;
  int32_t q = __double2int_rn(__dmul_rn((double)x, inv2e));
  int32_t rem = x - q * two_e;
  if (rem > e) { q += 1; rem -= two_e; }
  else if (rem < -e) { q -= 1; rem += two_e; }
  if (rem == e && x > 0) q += 1;
  else if (rem == -e && x < 0) q -= 1;
  return q;
}

// Encoder step in error form.  rho, q0: R0 = q0*2e + rho, rho in [-e, e];
// d = errU + errL - errUL.  With y = rho - d, x = q0*2e + y and
//   q = rha(x / 2e) = q0 + g,  g = floor((y+e)/2e)  (x >= 0)
//                              g = ceil((y-e)/2e)   (x <  0),
// err = g*2e - y (0 on escape).  Fast path: |y| < 4e (the neighbours share
// this pixel's step), g from four comparisons; otherwise the exact divisions.
__device__ __forceinline__ int32_t floordiv_p(int32_t a, int32_t d) {  // d > 0
  int32_t q = a / d;
  if ((a % d != 0) && (a < 0)) q--;
  return q;
}
__device__ __forceinline__ bool enc_in_fast_range(int32_t rho, int32_t e,
                                                  int32_t d) {
  const int32_t y = rho - d;
  return y < 4 * e && y > -4 * e;
}
template <bool FAST>
__device__ __forceinline__ int32_t enc_step(int32_t rho, int32_t q0,
                                            int32_t e, int32_t d,
                                            int32_t radius, uint32_t* sym) {
  const int32_t y = rho - d;
  const bool xneg = (int64_t)q0 * (2 * (int64_t)e) + y < 0;
  int32_t g;
  if (FAST) {
    const int32_t e3 = 3 * e;
    g = (y >= e) + (y >= e3) - (y < -e) - (y < -e3);
    const bool tie = (y == e) | (y == -e) | (y == e3) | (y == -e3);
    g -= (tie && xneg) ? 1 : 0;
  } else {
    g = xneg ? -floordiv_p(e - y, 2 * e) : floordiv_p(y + e, 2 * e);
  }
  const int64_t q = (int64_t)q0 + g;
  const bool esc = q <= -radius || q >= radius;
  *sym = esc ? 0u : (uint32_t)(q + radius);
  return esc ? 0 : g * 2 * e - y;
}

template <bool ENC, int CW>
__global__ void __launch_bounds__(32 * CW, 1)
chain_kernel(ChainIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChainSmem<CW, ENC>& sm = *reinterpret_cast<ChainSmem<CW, ENC>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const int H = io.H, W = io.W, Wp = io.Wp, nchunks = io.nchunks;
  const int nblocks = (W + 31 + 31) / 32;
  const int ntask = (H + 32 * CW - 1) / (32 * CW);

  for (;;) {
    if (threadIdx.x == 0) sm.task = atomicAdd(io.ticket, 1);
    if (threadIdx.x < CW) { sm.bdone[threadIdx.x] = 0; sm.bread[threadIdx.x] = 0; }
    __syncthreads();
    const int g = sm.task;
    if (g >= ntask) break;
    const int i0 = 32 * (CW * g + w);
    const bool wact = i0 < H;
    const int nrows = wact ? min(32, H - i0) : 0;
    const int my_i = i0 + lane;
    const bool rowok = my_i < H;
    const bool has_next = i0 + 32 < H;
    const bool next_in_cta = w + 1 < CW;
    const uint32_t tag = io.tag_base + (uint32_t)g + 1u;
    uint64_t* my_gb = io.bnd + (int64_t)g * 2 * W;
    const uint64_t* up_gb = io.bnd + (int64_t)(g - 1) * 2 * W;

    // coalesced staging of chunk m (lane = column; one row per iteration)
    auto stage = [&](int m) {
      const int s = m % CNS;
#pragma unroll 4
      for (int r = 0; r < 32; r++) {
        const bool rv = r < nrows;
        const int64_t rb = (int64_t)(i0 + (rv ? r : 0)) * Wp + 32 * m + lane;
        cp_async<4>(&sm.ring[w][s][0][r][lane ^ r], io.a0 + rb, rv);
        cp_async<4>(&sm.ring[w][s][1][r][lane ^ r], io.a1 + rb, rv);
      }
      const int64_t pb = (int64_t)(rowok ? my_i : i0) * nchunks + m;
      cp_async<4>(&sm.pin[w][s][0][lane], io.pin_u + pb, rowok);
      cp_async<4>(&sm.pin[w][s][1][lane], io.pin_v + pb, rowok);
      if (ENC) {
        cp_async<4>(&sm.x.nl[w][s][lane], io.nl + pb, rowok);
        cp_async<4>(&sm.x.symw[w][s][lane], io.symw + pb, rowok);
        // codes: 32 bytes per row, lanes (row r = lane >> 3 + 4 k, word lane & 7)
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int r = (lane >> 3) + 4 * k, q = lane & 7;
          const bool rv = r < nrows;
          cp_async<4>(&sm.x.code[w][s][r][q],
                      io.codes + (int64_t)(i0 + (rv ? r : 0)) * Wp + 32 * m + 4 * q,
                      rv);
        }
      }
    };
    // coalesced write-out of chunk x (complete) from its slot; escapes of
    // row r are added to esc_row of lane r
    int32_t esc_row = 0;
    auto write_out = [&](int x) {
      const int s = x % CNS;
      const int c = 32 * x + lane;
      const bool cv = c < W;
      uint32_t nl_r = 0, sw_r = 0;
      int32_t pre_r = 0;
      int64_t qrow_r = 0;
      if (ENC && rowok) {
        nl_r = sm.x.nl[w][s][lane];
        sw_r = sm.x.symw[w][s][lane];
        pre_r = io.chunk_nl[(int64_t)my_i * nchunks + x];
        qrow_r = io.qd_row_off[my_i];
      }
#pragma unroll 4
      for (int r = 0; r < 32; r++) {
        if (r >= nrows) break;
        const int32_t vu = sm.ring[w][s][0][r][lane ^ r];
        const int32_t vv = sm.ring[w][s][1][r][lane ^ r];
        if (cv) {
          const int64_t nr = (int64_t)(i0 + r) * Wp + c;
          io.out_i0[nr] = vu;
          io.out_i1[nr] = vv;
          if (!ENC) {
            const int64_t n = (int64_t)(i0 + r) * W + c;
            io.out_f0[n] = __dmul_rn((double)vu, io.inv_S);
            io.out_f1[n] = __dmul_rn((double)vv, io.inv_S);
          }
        }
        if (ENC) {
          const uint32_t nlw = __shfl_sync(FULL, nl_r, r);
          const uint32_t sww = __shfl_sync(FULL, sw_r, r);
          const int32_t pre = __shfl_sync(FULL, pre_r, r);
          const int64_t qrow = __shfl_sync(FULL, qrow_r, r);
          const uint32_t bit = 1u << lane;
          int ne = 0;
          if (cv && (sww & bit)) {
            const uint32_t sy = sm.x.sym[w][s][r][lane ^ r];
            const int64_t pos = qrow + 2 * ((int64_t)pre + __popc(nlw & (bit - 1u)));
            *reinterpret_cast<uint32_t*>(io.qd + pos) = sy;
            ne = ((sy & 0xffffu) == 0) + ((sy >> 16) == 0);
          }
          const int tot = __reduce_add_sync(FULL, ne);
          if (lane == r) esc_row += tot;
        }
      }
    };

    int32_t l_u = 0, l_v = 0, ul_u = 0, ul_v = 0, last_u = 0, last_v = 0;
    // one cp.async group per chunk (empty groups keep the count aligned):
    // at block m the newest group is chunk m+1, which may stay in flight
    if (wact) {
      stage(0);
      cp_async_commit();
      if (nchunks > 1) stage(1);
      cp_async_commit();
    }
    PhaseClock pc(io.stats);
    for (int m = 0; m < nblocks && wact; m++) {
      const int c0 = 32 * m;
      cp_async_wait_group<1>();   // chunks <= m have landed
      __syncwarp();
      pc.lap(WP_WAITPREV, lane);
      // ---- boundary row (row i0-1) for columns c0..c0+31
      int32_t bu = 0, bv = 0;
      if (i0 > 0 && c0 < W) {
        if (w > 0) {
          const int need = min(m + 2, nblocks);
          while (!__all_sync(FULL, ld_volatile(&sm.bdone[w - 1]) >= need))
            __nanosleep(20);
          __threadfence_block();
          bu = sm.bnd[w - 1][m & 3][0][lane];
          bv = sm.bnd[w - 1][m & 3][1][lane];
          __syncwarp();
          if (lane == 0) *(volatile int*)&sm.bread[w] = m + 1;
        } else {
          const int c = c0 + lane;
          const bool v = c < W;
          const int cc = v ? c : 0;
          bu = TaggedSlot<int32_t>::get(up_gb + cc, tag - 1, v);
          bv = TaggedSlot<int32_t>::get(up_gb + W + cc, tag - 1, v);
        }
      }
      // ---- this lane's 32 columns c = c0 - lane + jj (two chunks)
      pc.lap(WP_WAITBND, lane);
      const int cbase = c0 - lane;
      const int x_lo = cbase >> 5;   // -1 for the first block's lanes > 0
      const int s_lo = (x_lo + CNS) % CNS, s_hi = (x_lo + 1) % CNS;
      const uint32_t split = 32 - (cbase & 31);
      uint32_t pu_lo = 0, pv_lo = 0, pu_hi = 0, pv_hi = 0;
      if (rowok) {
        pu_lo = sm.pin[w][s_lo][0][lane]; pv_lo = sm.pin[w][s_lo][1][lane];
        pu_hi = sm.pin[w][s_hi][0][lane]; pv_hi = sm.pin[w][s_hi][1][lane];
      }
      const bool top = i0 > 0;
      if (!ENC) {
        int32_t av_u[32], av_v[32];
#pragma unroll
        for (int jj = 0; jj < 32; jj++) {
          const int c = cbase + jj;
          const int sl = (uint32_t)jj < split ? s_lo : s_hi;
          const int col = c & 31;
          av_u[jj] = sm.ring[w][sl][0][lane][col ^ lane];
          av_v[jj] = sm.ring[w][sl][1][lane][col ^ lane];
        }
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < 32; jj++) {
          const int c = cbase + jj;
          const int32_t b_u = __shfl_sync(FULL, bu, jj);
          const int32_t b_v = __shfl_sync(FULL, bv, jj);
          const int32_t up_u = __shfl_up_sync(FULL, last_u, 1);
          const int32_t up_v = __shfl_up_sync(FULL, last_v, 1);
          const bool inb = c < W;
          const int32_t nu_u = lane == 0 ? ((top && inb) ? b_u : 0) : up_u;
          const int32_t nu_v = lane == 0 ? ((top && inb) ? b_v : 0) : up_v;
          const bool act = rowok && c >= 0 && inb;
          const bool lo = (uint32_t)jj < split;
          const uint32_t bit = 1u << (c & 31);
          const bool pu_ = ((lo ? pu_lo : pu_hi) & bit) != 0;
          const bool pv_ = ((lo ? pv_lo : pv_hi) & bit) != 0;
          const bool first = c == 0;
          const int32_t l0_u = first ? 0 : l_u, l0_v = first ? 0 : l_v;
          const int32_t ul0_u = first ? 0 : ul_u, ul0_v = first ? 0 : ul_v;
          const int32_t r_u = pu_ ? av_u[jj]
              : (int32_t)((uint32_t)nu_u + ((uint32_t)l0_u +
                                            ((uint32_t)av_u[jj] - (uint32_t)ul0_u)));
          const int32_t r_v = pv_ ? av_v[jj]
              : (int32_t)((uint32_t)nu_v + ((uint32_t)l0_v +
                                            ((uint32_t)av_v[jj] - (uint32_t)ul0_v)));
          av_u[jj] = act ? r_u : av_u[jj];
          av_v[jj] = act ? r_v : av_v[jj];
          l_u = act ? r_u : l_u;
          l_v = act ? r_v : l_v;
          last_u = l_u;
          last_v = l_v;
          ul_u = nu_u;
          ul_v = nu_v;
        }
        if (rowok) {
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            const int c = cbase + jj;
            if (c >= 0 && c < W) {
              const int sl = (uint32_t)jj < split ? s_lo : s_hi;
              sm.ring[w][sl][0][lane][(c & 31) ^ lane] = av_u[jj];
              sm.ring[w][sl][1][lane][(c & 31) ^ lane] = av_v[jj];
            }
          }
        }
      } else {
        // encoder: per-step shared-memory operands (register budget); the
        // loads and the R0 split are independent of the chain and are
        // scheduled ahead by the unrolled loop
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < 32; jj++) {
          const int c = cbase + jj;
          const bool lo = (uint32_t)jj < split;
          const int sl = lo ? s_lo : s_hi;
          const int col = c & 31;
          const int32_t a_u = sm.ring[w][sl][0][lane][col ^ lane];
          const int32_t a_v = sm.ring[w][sl][1][lane][col ^ lane];
          const int cd = (sm.x.code[w][sl][lane][col >> 2] >> (8 * (col & 3))) & 31;
          const int32_t e = io.e_tab[cd];
          const double inv = io.inv2e_tab[cd];
          const uint32_t bit = 1u << col;
          const bool pu_ = ((lo ? pu_lo : pu_hi) & bit) != 0;
          const bool pv_ = ((lo ? pv_lo : pv_hi) & bit) != 0;
          const bool live = e != 0;
          const int32_t q0u = (!pu_ && live) ? quant32(a_u, e, inv) : 0;
          const int32_t q0v = (!pv_ && live) ? quant32(a_v, e, inv) : 0;
          const int32_t rho_u = a_u - q0u * 2 * e, rho_v = a_v - q0v * 2 * e;
          const int32_t b_u = __shfl_sync(FULL, bu, jj);
          const int32_t b_v = __shfl_sync(FULL, bv, jj);
          const int32_t up_u = __shfl_up_sync(FULL, last_u, 1);
          const int32_t up_v = __shfl_up_sync(FULL, last_v, 1);
          const bool inb = c < W;
          const int32_t nu_u = lane == 0 ? ((top && inb) ? b_u : 0) : up_u;
          const int32_t nu_v = lane == 0 ? ((top && inb) ? b_v : 0) : up_v;
          const bool act = rowok && c >= 0 && inb;
          const bool first = c == 0;
          const int32_t l0_u = first ? 0 : l_u, l0_v = first ? 0 : l_v;
          const int32_t ul0_u = first ? 0 : ul_u, ul0_v = first ? 0 : ul_v;
          uint32_t su, sv;
          const int32_t d_u = nu_u + l0_u - ul0_u, d_v = nu_v + l0_v - ul0_v;
          int32_t eu_ = enc_step<true>(rho_u, q0u, e, d_u, io.radius, &su);
          int32_t ev_ = enc_step<true>(rho_v, q0v, e, d_v, io.radius, &sv);
          const bool slow = live && !(enc_in_fast_range(rho_u, e, d_u) &&
                                      enc_in_fast_range(rho_v, e, d_v));
          if (__any_sync(FULL, slow)) {   // warp-uniform branch, rare
            uint32_t su2, sv2;
            const int32_t e1 = live ? e : 1;
            const int32_t eu2 = enc_step<false>(rho_u, q0u, e1, d_u, io.radius, &su2);
            const int32_t ev2 = enc_step<false>(rho_v, q0v, e1, d_v, io.radius, &sv2);
            if (slow) { eu_ = eu2; ev_ = ev2; su = su2; sv = sv2; }
          }
          const int32_t r_u = pu_ ? a_u : eu_;
          const int32_t r_v = pv_ ? a_v : ev_;
          if (act) {
            sm.ring[w][sl][0][lane][col ^ lane] = r_u;
            sm.ring[w][sl][1][lane][col ^ lane] = r_v;
            sm.x.sym[w][sl][lane][col ^ lane] =
                ((pu_ ? 0u : su) & 0xffffu) | ((pv_ ? 0u : sv) << 16);
          }
          l_u = act ? r_u : l_u;
          l_v = act ? r_v : l_v;
          last_u = l_u;
          last_v = l_v;
          ul_u = nu_u;
          ul_v = nu_v;
        }
      }
      __syncwarp();
      pc.lap(WP_CHAIN, lane);
      // ---- row 31 of this strip for the strip below (from the ring)
      if (has_next) {
        const int c = c0 - 31 + lane;        // the columns row 31 did now
        const bool cv = c >= 0 && c < W;
        const int sl = cv ? (c >> 5) % CNS : 0;
        const int32_t vu = cv ? sm.ring[w][sl][0][31][(c & 31) ^ 31] : 0;
        const int32_t vv = cv ? sm.ring[w][sl][1][31][(c & 31) ^ 31] : 0;
        if (next_in_cta) {
          // the consumer must be done with chunk m-3 (same slot as m+1)
          const int need = m - 3;
          while (!__all_sync(FULL, ld_volatile(&sm.bread[w + 1]) >= need))
            __nanosleep(20);
          if (cv) {
            sm.bnd[w][(c >> 5) & 3][0][c & 31] = vu;
            sm.bnd[w][(c >> 5) & 3][1][c & 31] = vv;
          }
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            *(volatile int*)&sm.bdone[w] = m + 1;
          }
          __syncwarp();
        } else if (cv) {
          TaggedSlot<int32_t>::put(my_gb + c, tag, vu);
          TaggedSlot<int32_t>::put(my_gb + W + c, tag, vv);
        }
      }
      // ---- chunk m-1 is complete: write it out, then reuse its slot for
      //      chunk m+2
      pc.lap(WP_X3, lane);
      if (m >= 1) write_out(m - 1);
      if (m == nblocks - 1 && 32 * m < W) write_out(m);
      __syncwarp();
      pc.lap(WP_WRITE, lane);
      if (m + 2 < nchunks) stage(m + 2);
      cp_async_commit();
      pc.lap(WP_PRE, lane);
    }
    if (ENC && rowok && esc_row) io.row_esc[my_i] += esc_row;
    cp_async_wait_all();
    __syncthreads();
  }
}

}  // namespace vfcp
