// The raster-order Lorenzo recurrence of one frame as a strip wavefront.
//
// Shared by the encoder (codec.py:118-164 _encode_frame) and the decoder
// (codec.py:167-206 _decode_frame).  Everything that does not depend on the
// current frame's reconstructed neighbours is computed beforehand, fully in
// parallel, by the prepare kernels (fast.cu); what is left is the
// recurrence through the up / left / up-left neighbours:
//
//   decoder (value form):  r = rU + rL - rUL + A,   A = Pd + (sym-radius)*2e
//   encoder (error form):  with err = recon - orig and
//     R0 = orig - Lorenzo(orig, prev)  (prepared),  D = errU + errL - errUL,
//     x = R0 - D,  q = rha(x / 2e),  err = q*2e - x  (0 on escape),
//     sym = q + radius  (0 on escape)
//
// The encoder never divides on the critical path: R0 is split once per
// pixel (prepare kernel) as R0 = Q0*2e + rho0, rho0 in [-e, e]; with
// y = rho0 - D, q = Q0 + g and, while |y| <= 4e, g follows from the signs
// of y -+ e, y -+ 3e (see enc_fast_g).  Blocks where some |y| > 4e (step
// sizes differ between neighbours) are redone with exact divisions.
//
// The two components are independent recurrences.  A task is one
// component of one 32-row strip, run by a warp PAIR:
//   C (chain warp): lane = row, sweeps the columns with a one-column skew
//     per lane so the three neighbours are final when read; a step is
//     shfl -> integer ops -> select on register operands.  It hands the
//     strip's last row to the strip below (shared memory inside the CTA,
//     tagged global slots across CTAs).
//   P (producer warp): stages 32-column chunks of the prepared planes with
//     coalesced cp.async into a 4-slot ring and writes finished chunks back
//     out coalesced (recon / err, symbol planes).
// A CTA holds NPAIR consecutive strips of one component; CTAs take tickets
// in (strip group, component) order, so a CTA only ever waits on an
// earlier, resident one.
#pragma once

#include "common.cuh"
#include "wavefront.cuh"

namespace vfcp {

// Prepared planes (frame layout, row pitch Wp = 32 * nchunks):
//   a0, a1    int32 per component: decoder -- A or the pinned recon;
//             encoder -- R0 or the pinned err
//   q0_0, q0_1  encoder: Q0 = rha(R0 / 2e) per component (0 where pinned)
//   codes     encoder: frame t codes (pitch Wp)
//   pin_u, pin_v  uint32 per (row, chunk): bit j = pixel c0+j is pinned
struct ChainIO {
  const int32_t* a0;
  const int32_t* a1;
  const int32_t* q0_0;
  const int32_t* q0_1;
  const uint8_t* codes;
  const uint32_t* pin_u;
  const uint32_t* pin_v;
  int32_t* out_i0;           // decoder: recon; encoder: err (pitch Wp)
  int32_t* out_i1;
  uint16_t* sym0;            // encoder: symbol planes (pitch Wp)
  uint16_t* sym1;
  uint64_t* bnd;             // tagged last-row slots [ntask][W]
  unsigned long long* stats; // optional phase timers (WavePhase)
  int stats_strip0;          // time only task 0, pair 0
  unsigned long long* tstamp; // optional per-task [start, first block, end] ns
  int* ticket;
  uint32_t tag_base;         // tags unique across frames sharing `bnd`
  int H, W, Wp, nchunks;
  int radius;
  int32_t e_tab[32];         // e per code (encoder; requires tau' < 2^28)
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

// Exact encoder step in error form.  rho, q0: R0 = q0*2e + rho; d = errU +
// errL - errUL.  With y = rho - d, x = q0*2e + y and
//   q = rha(x / 2e) = q0 + g,  g = floor((y+e)/2e)  (x >= 0)
//                              g = ceil((y-e)/2e)   (x <  0),
// err = g*2e - y (0 on escape).
__device__ __forceinline__ int32_t floordiv_p(int32_t a, int32_t d) {  // d > 0
  int32_t q = a / d;
  if ((a % d != 0) && (a < 0)) q--;
  return q;
}
__device__ __forceinline__ int32_t enc_step_exact(int32_t rho, int32_t q0,
                                                  int32_t e, int32_t d,
                                                  int32_t radius, uint32_t* sym) {
  const int32_t y = rho - d;
  const bool xneg = (int64_t)q0 * (2 * (int64_t)e) + y < 0;
  const int32_t g = xneg ? -floordiv_p(e - y, 2 * e) : floordiv_p(y + e, 2 * e);
  const int64_t q = (int64_t)q0 + g;
  const bool esc = q <= -radius || q >= radius;
  *sym = esc ? 0u : (uint32_t)(q + radius);
  return esc ? 0 : g * 2 * e - y;
}

// One encoder step without divisions, valid while |y| <= 4e (y = rho - d).
// With the breakpoints B = rho -+ e, rho -+ 3e (y = +-e, +-3e), g rounds
// ties downward in d* = d - [d < R0]: a tie rounds away from zero in
// x = R0 - d, i.e. toward the larger g iff x > 0, and g_up(d) = g_dn(d-1).
//   g = -2 - sum_k sign(d* - B_k)   (sign = arithmetic shift by 31)
// No overflow: |R0| < 2^31 is compared, never subtracted; |d| <= 3 * 2^28,
// |B_k| <= 4 * 2^28 (e < 2^28).  Returns the pixel's new err (0 on escape)
// and its symbol (0 on escape).
__device__ __forceinline__ int32_t enc_step_fast(int32_t R0, int32_t q0,
                                                 int32_t rho, int32_t e,
                                                 int32_t d, int32_t radius,
                                                 uint32_t* sym) {
  const int32_t ds = d - (d < R0 ? 1 : 0);
  const int32_t b1 = rho - 3 * e, b2 = rho - e, b3 = rho + e, b4 = rho + 3 * e;
  const int32_t g = -2 - (((ds - b1) >> 31) + ((ds - b2) >> 31)) -
                    (((ds - b3) >> 31) + ((ds - b4) >> 31));
  const int32_t q = q0 + g;
  const bool esc = (uint32_t)(q + radius - 1) >= (uint32_t)(2 * radius - 1);
  *sym = esc ? 0u : (uint32_t)(q + radius);
  return esc ? 0 : g * (2 * e) + (d - rho);
}

// strips (warp pairs) per CTA; tasks per frame
__host__ __device__ constexpr int chain_pairs(bool enc) { return enc ? 4 : 4; }
__host__ __device__ inline int chain_ntask(bool enc, int H) {
  return 2 * ((H + 32 * chain_pairs(enc) - 1) / (32 * chain_pairs(enc)));
}
constexpr int CNS = 4;   // chunk slots: the sweep of block m uses chunks m-1
                         // and m; P stages m+1, m+2 meanwhile

template <bool ENC>
struct PairRing {
  // [slot][row][col]: A -> recon; R0 -> err.  No swizzle: the chain warp
  // reads column c0 - lane + jj in row lane, distinct banks across lanes.
  int32_t v[CNS][32][32];
  uint32_t pin[CNS][32];
  int32_t q0[ENC ? CNS : 1][32][32];   // encoder: Q0, then the symbol
  uint32_t code[ENC ? CNS : 1][32][8]; // encoder: codes, 4 per word
};

constexpr int HRING = 128;   // boundary-row ring (columns), power of two

template <bool ENC>
struct ChainSmem {
  PairRing<ENC> r[chain_pairs(ENC)];
  // row i0-1 of strip p: (column + 1) << 32 | value, so the consumer spins
  // on the entry itself (no separate flag, no fence on the producer side)
  uint64_t hin[chain_pairs(ENC) + 1][HRING];
  int32_t etab[32];
  int full[chain_pairs(ENC)];        // chunks P_p has staged
  int done[chain_pairs(ENC)];        // blocks C_p has swept
  int task;
};

// Warp-uniform wait for a shared-memory counter.  The chain warps poll
// tightly (they are on the critical path); the producers back off so their
// polling does not take issue slots and shared-memory bandwidth from the
// chain warp on the same sub-partition.
// The counters use acquire loads / release stores at CTA scope instead of
// full fences: a fence would also wait for the warp's outstanding global
// loads (the prefetched boundary slots).
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}
template <int SLEEP_NS = 0>
__device__ __forceinline__ void spin_ge(const int* p, int need) {
  while (!__all_sync(0xffffffffu, ld_acquire_cta(p) >= need)) {
    if (SLEEP_NS) __nanosleep(SLEEP_NS);
  }
}
__device__ __forceinline__ void signal_set(int* p, int v, int lane) {
  __syncwarp();   // the warp's writes happen before lane 0's release
  if (lane == 0) st_release_cta(p, v);
  __syncwarp();
}

template <bool ENC>
__global__ void __launch_bounds__(64 * chain_pairs(ENC))
chain_kernel(ChainIO io) {
  constexpr int NPAIR = chain_pairs(ENC);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChainSmem<ENC>& sm = *reinterpret_cast<ChainSmem<ENC>*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // chain warps 0..NPAIR-1, producers NPAIR..2*NPAIR-1: with NPAIR = 4 every
  // SM sub-partition (warp % 4) holds one chain and one producer warp
  const int pr = wid % NPAIR;
  const bool producer = wid >= NPAIR;
  PairRing<ENC>& R = sm.r[pr];
  const unsigned FULL = 0xffffffffu;
  const int H = io.H, W = io.W, Wp = io.Wp, nchunks = io.nchunks;
  const int nblocks = (W + 31 + 31) / 32;
  const int ntask = chain_ntask(ENC, H);
  if (threadIdx.x < 32) sm.etab[threadIdx.x] = io.e_tab[threadIdx.x];

  for (;;) {
    if (threadIdx.x == 0) sm.task = atomicAdd(io.ticket, 1);
    if (threadIdx.x < NPAIR) {
      sm.full[threadIdx.x] = 0; sm.done[threadIdx.x] = 0;
    }
    for (int k = threadIdx.x; k < (NPAIR + 1) * HRING; k += blockDim.x)
      (&sm.hin[0][0])[k] = 0;   // no stale tags from an earlier task
    __syncthreads();
    const int task = sm.task;
    if (task >= ntask) break;
    const int g = task >> 1, comp = task & 1;
    const int i0 = 32 * (NPAIR * g + pr);
    const bool wact = i0 < H;
    const int nrows = wact ? min(32, H - i0) : 0;
    const int my_i = i0 + lane;
    const bool rowok = my_i < H;
    // VFCP_WAVE_PROFILE=strip0 times only the first strip (its own work, no waits on others)
    PhaseClock pc((io.stats && (!io.stats_strip0 || (task == 0 && pr == 0))) ? io.stats : nullptr);

    if (producer && wact) {
      // ===================================================== producer
      const int32_t* a = comp ? io.a1 : io.a0;
      const int32_t* q0p = comp ? io.q0_1 : io.q0_0;
      const uint32_t* pinp = comp ? io.pin_v : io.pin_u;
      int32_t* out_i = comp ? io.out_i1 : io.out_i0;
      uint16_t* symp = comp ? io.sym1 : io.sym0;
      // 16-byte moves: lane = (row 4k + lane/8, columns 4*(lane%8) .. +3),
      // a 32x32 int32 tile in 8 instructions per plane (rows are 128-byte
      // aligned: Wp is a multiple of 32)
      const int vr = lane >> 3, vc = 4 * (lane & 7);
      auto stage = [&](int x) {
        const int s = x % CNS;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int r = 4 * k + vr;
          const bool rv = r < nrows;
          const int64_t kk = (int64_t)(i0 + (rv ? r : 0)) * Wp + 32 * x + vc;
          cp_async<16>(&R.v[s][r][vc], a + kk, rv);
          if (ENC) cp_async<16>(&R.q0[s][r][vc], q0p + kk, rv);
        }
        const int64_t pb = (int64_t)(rowok ? my_i : i0) * nchunks + x;
        cp_async<4>(&R.pin[s][lane], pinp + pb, rowok);
        if (ENC) {
          // codes: 32 rows x 32 bytes, 16 bytes per lane, 2 instructions
#pragma unroll
          for (int k = 0; k < 2; k++) {
            const int r = 16 * k + (lane >> 1), h = 16 * (lane & 1);
            const bool rv = r < nrows;
            cp_async<16>(reinterpret_cast<unsigned char*>(&R.code[s][r][0]) + h,
                         io.codes + (int64_t)(i0 + (rv ? r : 0)) * Wp + 32 * x + h, rv);
          }
        }
      };
      // finished chunk -> global (columns past W land in the pitch padding)
      auto write_out = [&](int x) {
        const int s = x % CNS;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int r = 4 * k + vr;
          if (r < nrows) {
            const int64_t kk = (int64_t)(i0 + r) * Wp + 32 * x + vc;
            *reinterpret_cast<int4*>(out_i + kk) = *reinterpret_cast<const int4*>(&R.v[s][r][vc]);
            if (ENC) {
              const int4 q = *reinterpret_cast<const int4*>(&R.q0[s][r][vc]);
              uint2 w;
              w.x = ((uint32_t)q.x & 0xffffu) | ((uint32_t)q.y << 16);
              w.y = ((uint32_t)q.z & 0xffffu) | ((uint32_t)q.w << 16);
              *reinterpret_cast<uint2*>(symp + kk) = w;
            }
          }
        }
      };
      // chunk x lives in slot x % CNS from its staging to its write-out;
      // it is complete once C has swept blocks x and x+1 (done >= x+2)
      int next_out = 0;
      auto retire_before = [&](int x) {   // free the slot chunk x needs
        while (next_out <= x - CNS) {
          spin_ge<200>(&sm.done[pr], min(next_out + 2, nblocks));
          pc.lap(WP_X1, lane);
          write_out(next_out);
          next_out++;
          pc.lap(WP_WRITE, lane);
        }
      };
      stage(0);
      cp_async_commit();
      for (int x = 1; x <= nchunks; x++) {
        if (x < nchunks) {
          retire_before(x);
          stage(x);
        }
        cp_async_commit();
        cp_async_wait_group<1>();   // chunk x-1 has landed
        signal_set(&sm.full[pr], x, lane);
        pc.lap(WP_PRE, lane);
      }
      retire_before(nchunks + CNS - 1);
    } else if (wact) {
      // ===================================================== chain warp
      // Row i0-1 (the strip above's last row) arrives in hin[pr] (a ring of
      // HRING columns) with hprog[pr] = columns available: streamed every 8
      // steps by the chain warp above when it is in this CTA, fetched per
      // block from the tagged global slots otherwise.  This strip's last
      // row is streamed the same way into hin[pr+1], or put to the global
      // slots after each block for the next CTA.
      const bool has_next = i0 + 32 < H;
      const bool stream_out = has_next && pr + 1 < NPAIR;
      const uint32_t tag = io.tag_base + (uint32_t)task + 1u;
      uint64_t* my_gb = io.bnd + (int64_t)task * W;
      const uint64_t* up_gb = io.bnd + (int64_t)(task - 2) * W;
      const bool top = i0 > 0;
      const bool lane0 = lane == 0, lane31 = lane == 31;
      uint64_t* hin = sm.hin[pr];
      uint64_t* hout = sm.hin[pr + (stream_out ? 1 : 0)];
      int32_t l = 0, ul = 0;
      uint64_t bpre = 0;   // prefetched tagged boundary slot (pr == 0)
      if (top && pr == 0 && lane < W) bpre = ld_relaxed_u64(up_gb + lane);
      auto stamp = [&](int k) {
        if (io.tstamp && lane == 0) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          io.tstamp[(int64_t)(2 * g * NPAIR + 2 * pr + comp) * 3 + k] = t;
        }
      };
      stamp(0);
      for (int m = 0; m < nblocks; m++) {
        const int c0 = 32 * m;
        spin_ge(&sm.full[pr], min(m + 1, nchunks));
        pc.lap(WP_WAITPREV, lane);
        if (m == 1) stamp(1);
        if (top && pr == 0 && c0 < W) {
          // tagged slots of the strip above (other CTA); the load for this
          // block was issued during the previous block's sweep
          const int c = c0 + lane;
          const bool v = c < W;
          uint64_t w = v ? bpre : 0;
          bool ok = !v || (uint32_t)(w >> 32) == tag - 2;
          while (!__all_sync(FULL, ok)) {
            if (!ok) {
              w = ld_relaxed_u64(up_gb + c);
              ok = (uint32_t)(w >> 32) == tag - 2;
            }
          }
          hin[c & (HRING - 1)] = ((uint64_t)(c + 1) << 32) | (uint32_t)w;
          __syncwarp();
          const int cn = c + 32;
          if (cn < W) bpre = ld_relaxed_u64(up_gb + cn);
        }
        // the consumer below must be done with the ring entries we reuse
        if (stream_out) spin_ge(&sm.done[pr + 1], m - (HRING / 32 - 1));
        pc.lap(WP_WAITBND, lane);
        // boundary columns c0+jj .. c0+jj+7: lane k < 8 waits for column
        // c0+jj+k's tag and holds its value (0 outside the frame / top strip)
        auto bnd_group = [&](int jj) -> int32_t {
          const int c = c0 + jj + lane;
          const bool want = top && lane < 8 && c < W;
          const volatile uint64_t* e = hin + (c & (HRING - 1));
          uint64_t w = want ? *e : 0;
          bool ok = !want || (uint32_t)(w >> 32) == (uint32_t)(c + 1);
          while (!__all_sync(FULL, ok)) {
            if (!ok) {
              w = *e;
              ok = (uint32_t)(w >> 32) == (uint32_t)(c + 1);
            }
          }
          return want ? (int32_t)(uint32_t)w : 0;
        };
        // row 31 of this strip finished column c: stream it to the strip below
        auto put_bnd = [&](int c, int32_t r) {
          if (c >= 0) hout[c & (HRING - 1)] = ((uint64_t)(c + 1) << 32) | (uint32_t)r;
        };
        // ---- this lane's 32 columns c = c0 - lane + jj (two chunks).
        // vm: bit jj = pixel (my_i, cbase+jj) exists; pm: pinned or not
        // existing (those take their prepared value, 0 left of column 0, so
        // the left / up-left state entering column 0 is 0 with no test).
        const int cbase = c0 - lane;
        const int x_lo = cbase >> 5;   // -1 for the first block's lanes > 0
        const int s_lo = (x_lo + CNS) % CNS, s_hi = (x_lo + 1) % CNS;
        const uint32_t split = 32 - (cbase & 31);
        const int jlo = max(0, -cbase), jhi = min(32, W - cbase);
        const uint32_t vm =
            (rowok && jhi > jlo)
                ? ((jhi >= 32 ? 0xffffffffu : ((1u << jhi) - 1u)) & ~((1u << jlo) - 1u))
                : 0u;
        const uint32_t pm =
            __funnelshift_r(R.pin[s_lo][lane], R.pin[s_hi][lane], cbase & 31) | ~vm;
        if (!ENC) {
          int32_t av[32];
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            const int c = cbase + jj;
            const int sl = (uint32_t)jj < split ? s_lo : s_hi;
            const int32_t x = R.v[sl][lane][c & 31];
            av[jj] = c < 0 ? 0 : x;
          }
          int32_t bg = 0;
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            // the group's boundary values up front (lane k: column c0+jj+k)
            if ((jj & 7) == 0) bg = bnd_group(jj);
            const int32_t bb = __shfl_sync(FULL, bg, jj & 7);
            const int32_t up = __shfl_up_sync(FULL, l, 1);
            const int32_t nu = lane0 ? bb : up;
            const int32_t t = (int32_t)((uint32_t)av[jj] - (uint32_t)ul);
            const int32_t r = ((pm >> jj) & 1u) ? av[jj]
                : (int32_t)((uint32_t)nu + (uint32_t)l + (uint32_t)t);
            av[jj] = r;
            l = r;
            ul = nu;
            if (stream_out && lane31) put_bnd(c0 - 31 + jj, r);
          }
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            const int c = cbase + jj;
            const int sl = (uint32_t)jj < split ? s_lo : s_hi;
            if ((vm >> jj) & 1u) R.v[sl][lane][c & 31] = av[jj];
          }
        } else {
          const int32_t radius = io.radius;
          const int32_t l_s = l, ul_s = ul;
          const unsigned char* cb_lo =
              reinterpret_cast<const unsigned char*>(&R.code[s_lo][lane][0]);
          const unsigned char* cb_hi =
              reinterpret_cast<const unsigned char*>(&R.code[s_hi][lane][0]);
          // operands into registers first (the sweep's stores would keep
          // later loads from being hoisted past them): rr = R0 (or the
          // pinned err; 0 left of column 0), qq = Q0, ee = e (0 where
          // pinned / absent: no slow-path trigger there)
          int32_t rr[32], qq[32], ee[32];
#pragma unroll
          for (int jj = 0; jj < 32; jj++) {
            const int c = cbase + jj;
            const bool lo = (uint32_t)jj < split;
            const int sl = lo ? s_lo : s_hi;
            const int col = c & 31;
            const int32_t x = R.v[sl][lane][col];
            rr[jj] = c < 0 ? 0 : x;
            qq[jj] = R.q0[sl][lane][col];
            const int e = sm.etab[(lo ? cb_lo : cb_hi)[c & 31] & 31];
            ee[jj] = ((pm >> jj) & 1u) ? 0 : e;
          }
          pc.lap(WP_TASKS, lane);
          // fast steps 8 at a time; results before the first step with
          // |y| > 4e are exact, so completed groups are published at once
          bool redo = false;
#pragma unroll
          for (int g8 = 0; g8 < 32; g8 += 8) {
            if (!redo) {
              const int32_t bg = bnd_group(g8);
              bool slow = false;
#pragma unroll
              for (int k = 0; k < 8; k++) {
                const int jj = g8 + k;
                const int32_t R0 = rr[jj], q0 = qq[jj], e = ee[jj];
                const int32_t rho = R0 - q0 * (2 * e);
                const int32_t bb = __shfl_sync(FULL, bg, k);
                const int32_t up = __shfl_up_sync(FULL, l, 1);
                const int32_t nu = lane0 ? bb : up;
                const int32_t d = nu + l - ul;
                uint32_t sy;
                const int32_t er = enc_step_fast(R0, q0, rho, e, d, radius, &sy);
                const bool pin = (pm >> jj) & 1u;
                const int32_t r = pin ? R0 : er;
                qq[jj] = pin ? 0 : (int32_t)sy;
                // |y| > 4e: y + 4e outside [0, 8e] (no overflow, e < 2^28)
                slow |= (e != 0) & ((uint32_t)(rho - d + 4 * e) > (uint32_t)(8 * e));
                rr[jj] = r;
                l = r;
                ul = nu;
              }
              if (__any_sync(FULL, slow)) {
                redo = true;
              } else if (stream_out && lane31) {
                // exact results (no step of the group needed the exact
                // path): stream the group's row-31 values
#pragma unroll
                for (int k = 0; k < 8; k++) put_bnd(c0 - 31 + g8 + k, rr[g8 + k]);
              }
            }
          }
          if (redo) {
            // mixed steps: redo the block with the exact step
            if (io.stats && lane == 0) atomicAdd(io.stats + WP_X2, 1ull);
            l = l_s; ul = ul_s;
            int32_t bgr[4];
#pragma unroll
            for (int g = 0; g < 4; g++) bgr[g] = bnd_group(8 * g);
#pragma unroll 1
            for (int jj = 0; jj < 32; jj++) {
              const int c = cbase + jj;
              const bool lo = (uint32_t)jj < split;
              const int sl = lo ? s_lo : s_hi;
              const int col = c & 31;
              const bool valid = (vm >> jj) & 1u, pin = (pm >> jj) & 1u;
              const int32_t R0 = c < 0 ? 0 : R.v[sl][lane][col];
              const int32_t q0 = R.q0[sl][lane][col];
              const int32_t e = pin ? 0 : sm.etab[(lo ? cb_lo : cb_hi)[c & 31] & 31];
              const int32_t bgj = (jj < 8) ? bgr[0] : (jj < 16) ? bgr[1] : (jj < 24) ? bgr[2] : bgr[3];
              const int32_t bb = __shfl_sync(FULL, bgj, jj & 7);
              const int32_t up = __shfl_up_sync(FULL, l, 1);
              const int32_t nu = lane0 ? bb : up;
              const int32_t d = nu + l - ul;
              uint32_t sy = 0;
              const int32_t er =
                  e != 0 ? enc_step_exact(R0 - q0 * 2 * e, q0, e, d, radius, &sy) : 0;
              const int32_t r = pin ? R0 : er;
              if (valid) {
                R.v[sl][lane][col] = r;
                R.q0[sl][lane][col] = pin ? 0 : (int32_t)sy;
              }
              if (stream_out && lane31) put_bnd(c0 - 31 + jj, r);
              l = r;
              ul = nu;
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 32; jj++) {
              const int c = cbase + jj;
              const int sl = (uint32_t)jj < split ? s_lo : s_hi;
              const int col = c & 31;
              if ((vm >> jj) & 1u) {
                R.v[sl][lane][col] = rr[jj];
                R.q0[sl][lane][col] = qq[jj];
              }
            }
          }
        }
        __syncwarp();
        pc.lap(WP_CHAIN, lane);
        // ---- row 31 for the strip below in the next CTA (from the ring)
        if (has_next && !stream_out) {
          const int c = c0 - 31 + lane;   // the columns row 31 did now
          const bool cv = c >= 0 && c < W;
          const int sl = cv ? (c >> 5) % CNS : 0;
          const int32_t val = cv ? R.v[sl][31][c & 31] : 0;
          if (cv) TaggedSlot<int32_t>::put(my_gb + c, tag, val);
        }
        signal_set(&sm.done[pr], m + 1, lane);
        pc.lap(WP_X3, lane);
      }
      stamp(2);
    }
    cp_async_wait_all();
    __syncthreads();
  }
}

}  // namespace vfcp
