// The raster-order Lorenzo recurrence of one frame as a 2D block scan.
//
// Per component, with zero padding outside the frame and Z = recon -
// recon(t-1):
//   decoder:  Z = ZU + ZL - ZUL + A,  A = (sym - radius) * 2e   (exact)
//   encoder:  err = recon - orig = q*2e - x,  x = R0 - (errU + errL -
//             errUL),  q = rha(x / 2e),  R0 = orig - Lorenzo(orig, prev)
// so in the encoder err == -R0 + errU + errL - errUL (mod 2e) whenever the
// pixel is quantised with the same step e (err in [-e, e] is the
// representative of that residue; a residue of exactly e is a tie whose
// sign follows x, which rounds away from zero).  Over a 32x32 block whose
// pixels all share one step, have no pins and cannot escape (|R0| < (2
// radius - 4) e) -- a REG block -- every value is the block's 2D prefix sum
// plus its boundary:
//   v(i, j) = top(j) + left(i) - corner + sum_{a<=i, b<=j} X(a, b)
// with X = A (decoder, wrapping uint32 arithmetic is exact because the
// result fits int32) or X = -R0 mod 2e (encoder, whose prefix sum
// telescopes to -(delta(i,j) - delta(top,j) - delta(i,left) +
// delta(corner)), delta = orig - recon(t-1), see enc_block.cu).  Blocks whose
// values are known without the recurrence (KNOWN: all pixels pinned --
// semi-Lagrangian blocks, lossless areas) pass their edge values; any other
// block (mixed pins, mixed steps, possible escapes, a tie on its boundary)
// is swept exactly, pixel by pixel, given its exact boundary.
//
// Three phases per frame:
//   phase A  fully parallel, in the block kernels (enc_block.cu,
//            dec_block.cu): block class and the bottom row / right column of
//            the block-local prefix sums (LB, LR), or the known edge values;
//            KNOWN blocks are written there;
//   phase B  bs_chain_kernel, the only sequential part: block boundaries
//            travel down the block rows (one warp per block row and
//            component walks its row in chunks of BS_CH blocks; the exact
//            bottom rows are handed to the warp below) -- the critical path is
//            ~nby hand-offs + nbx / BS_CH chunk steps instead of H + W pixel
//            steps;
//   phase C  bs_interior_kernel, a programmatic dependent launch of phase B
//            that runs beside it and follows its per-segment progress marks:
//            one warp per block and both components, four pixels per lane --
//            recon(t), the encoder's symbols, the decoder's float64 output.
#pragma once

#include "frame.cuh"

namespace vfcp {

enum : uint8_t { BS_SLOW = 0, BS_KNOWN = 1, BS_REG = 2, BS_DONE = 3 };
// class word: kind | code << 2 | BS_NARROW (encoder: every |delta| of the
// block's tile with its halo is below 2^27, so the interior pass works in
// int32 on the integers themselves instead of residues)
constexpr int32_t BS_NARROW = 0x100;

struct BScanIO {
  const int32_t* a[2];
  int32_t* a_w[2];          // encoder: the same planes, written by the block
                            // kernel (R0 of the blocks the chain sweeps)
  const uint8_t* codes;     // frame codes (pitch cpitch)
  int cpitch;
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
  int dbg_skip_interior;       // VFCP_CHAIN_ONLY (timing experiments only)
  int vec4;                    // float32 rows 16-byte aligned (W % 4 == 0)
  unsigned long long* phase;   // optional [nby][8] clock cycles per chain phase (comp u)
  unsigned long long* prog;    // [2][nby]: frame tag << 32 | blocks finished
  uint32_t frame_tag;          // unique per frame of a call (t + 1)
  // decoder, frame t: the float64 output recon * inv_S (and optionally the
  // int64 fixed-point recon), pitch W -- written by the interior pass
  double* f64[2];
  int64_t* fix[2];
  double inv_S;
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
  uint32_t c32_tab[32];     // 2^32 mod 2e per code (0: lossless)
  // interior pass: (encoder) orig(t) (float32 / float64); recon(t-1)
  // (nullptr for frame 0) and recon(t) as interleaved (u, v) pairs, pitch Wp
  const void* orig[2];
  const int2* prevrec;
  int2* rec;
  double S;
};

constexpr int BS_NW = 8;        // block rows (warps) per chain CTA
constexpr int BS_HRING = 1024;   // shared boundary ring (columns), power of 2
constexpr int BS_SEG = 32;      // blocks per chain progress mark
constexpr int BS_CH = 4;        // blocks per chain step (a chunk; 8 lengthens
                                // the hand-off to the row below: slower)
constexpr int BS_SPIN_NS = 64;  // back-off of a waiting chain warp (its polls share the MIO pipe)
constexpr int BS_TW = BS_NW;    // blocks per interior task (a warp per block)

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
// x mod m for |x| < 2^32 (x = o - p with |o| < 2^30, |p| < 2^31); c32 =
// 2^32 mod m, M = floor(2^32 / m)
__device__ __forceinline__ uint32_t res_i64(int64_t x, uint32_t m, uint32_t M,
                                            uint32_t c32) {
  const uint32_t r = bs_umod((uint32_t)(uint64_t)x, m, M);
  return x < 0 ? bs_msub(r, c32, m) : r;
}
// |rha(x / m)| for a = |x| < 2^32 (m = 2e, M = floor(2^32 / m)): the
// estimate umulhi(a, M) is floor(a / m) or one less; ties (remainder e) round
// away from zero, as _rha does (predictors.py:25-30)
__device__ __forceinline__ uint32_t bs_qabs(uint32_t a, uint32_t e, uint32_t m,
                                            uint32_t M) {
  uint32_t q = __umulhi(a, M);
  uint32_t r = a - q * m;
  if (r >= m) { q++; r -= m; }
  return q + (r >= e ? 1u : 0u);
}
// k = the integer nearest to s / m (|s| < 2^31) and whether s - k m is the
// tie +-e (whose sign the caller settles in raster order)
__device__ __forceinline__ int32_t bs_knear(int32_t s, uint32_t e, uint32_t m,
                                            uint32_t M, bool* tie) {
  const uint32_t a = s < 0 ? (uint32_t)0 - (uint32_t)s : (uint32_t)s;
  uint32_t q = __umulhi(a, M);
  uint32_t r = a - q * m;
  if (r >= m) { q++; r -= m; }
  *tie = r == e;
  q += r > e ? 1u : 0u;
  return s < 0 ? -(int32_t)q : (int32_t)q;
}
// representative in [-e, e] of a residue that is not the tie e
__device__ __forceinline__ int32_t bs_rep(uint32_t r, uint32_t e, uint32_t m) {
  return r < e ? (int32_t)r : (int32_t)r - (int32_t)m;
}

// Exact encoder step (codec.py:140-155): x = R0 - d, q = rha(x / 2e);
// escape -> err 0, symbol 0.
__device__ __forceinline__ int32_t bs_enc_exact(int32_t R0, int32_t d,
                                                int32_t e, uint32_t M,
                                                int32_t radius,
                                                uint32_t* sym) {
  // |x| < 2^31 + 3 e < 2^32 (the neighbours' errors are bounded by tau' <
  // 2^29): the quotient from the magnitude, ties away from zero
  const int64_t x = (int64_t)R0 - d;
  const uint32_t m = 2u * (uint32_t)e;
  const uint32_t a = (uint32_t)(x < 0 ? -x : x);
  const uint32_t qa = bs_qabs(a, (uint32_t)e, m, M);
  if (qa >= (uint32_t)radius) { *sym = 0u; return 0; }
  const int32_t q = x < 0 ? -(int32_t)qa : (int32_t)qa;
  *sym = (uint32_t)(q + radius);
  return (int32_t)((int64_t)q * (int64_t)m - x);
}

// ------------------------------------------------------------ phase B
// Shared memory of the chain kernel.
struct BSChainSmem {
  int32_t etab[32];
  uint32_t mtab[32];
  int task;
  int done[BS_NW];   // blocks of the row above that warp w has read
  int pub[BS_NW];    // blocks warp w has handed to warp w + 1
  // (LB, LR, class) of two chunks per warp (cp.async ring)
  alignas(16) int32_t pfb[BS_NW][2][32 * BS_CH];
  alignas(16) int32_t pfr[BS_NW][2][32 * BS_CH];
  alignas(16) int32_t pfc[BS_NW][2][BS_CH];
  // bottom rows handed from warp w - 1 to warp w (a ring of columns)
  int32_t hin[BS_NW + 1][BS_HRING];
  // slow path tiles, [row][col] unpadded: the skewed sweep reads column
  // s - lane in row lane, distinct banks across lanes
  int32_t tv[BS_NW][32][32];
  // slow path (encoder): per pixel (e, floor(2^32 / 2e)) and the sweep's
  // symbols (rows 68 bytes apart)
  uint2 te[BS_NW][32][32];
  uint16_t ts[BS_NW][32][34];
};

// What the exact sweep of one block needs (passed by value to the
// out-of-line sweep, so the kernel's parameter struct stays in the constant
// bank)
struct BSSlowIO {
  const int32_t* a;
  const uint8_t* codes;
  const uint32_t* pin;
  int32_t* out;
  uint16_t* qd;
  const int64_t* qd_row_off;
  const int32_t* pre_nl;
  int32_t* row_ll;
  const void* orig;
  const int2* prevrec;
  double S;
  int cpitch, W, Wp, nchunks, radius;
};
__device__ __forceinline__ BSSlowIO bs_slow_io(const BScanIO& io, int comp) {
  BSSlowIO s;
  s.a = io.a[comp]; s.codes = io.codes; s.pin = io.pin[comp]; s.out = io.out[comp];
  s.qd = io.qd; s.qd_row_off = io.qd_row_off; s.pre_nl = io.pre_nl;
  s.row_ll = io.row_ll; s.orig = io.orig[comp]; s.prevrec = io.prevrec;
  s.S = io.S; s.cpitch = io.cpitch; s.W = io.W; s.Wp = io.Wp;
  s.nchunks = io.nchunks; s.radius = io.radius;
  return s;
}

// Encoder: R0 = D(orig - recon(t-1)) of a block whose R0 plane the block
// kernel did not write (a REG block with a tie on its edges); |R0| < 2^30
// there, so int32 is exact.  Lane = column, rows streamed.
template <typename F>
__device__ __forceinline__ void bs_r0_rows(const BSSlowIO& io, int comp,
                                           int r0, int c0, int nr, int ncl,
                                           int32_t (*tv)[32], int lane) {
  const unsigned FULL = 0xffffffffu;
  const F* op = static_cast<const F*>(io.orig);
  const int2* pv = io.prevrec;
  const int W = io.W, Wp = io.Wp;
  const int j = c0 + min(lane, ncl - 1);
  auto delta = [&](int i, int jj) -> int32_t {
    if (i < 0 || jj < 0) return 0;
    const int32_t o = fixed_t(__ldg(op + (int64_t)i * W + jj), io.S);
    const int2 pp = pv ? __ldg(pv + (int64_t)i * Wp + jj) : make_int2(0, 0);
    return o - (comp ? pp.y : pp.x);
  };
  int32_t dU = delta(r0 - 1, j);
  int32_t dUL = delta(r0 - 1, c0 - 1);
  for (int r = 0; r < nr; r++) {
    const int32_t d = delta(r0 + r, j);
    const int32_t dl0 = delta(r0 + r, c0 - 1);
    int32_t dl = __shfl_up_sync(FULL, d, 1);
    int32_t dul = __shfl_up_sync(FULL, dU, 1);
    if (lane == 0) { dl = dl0; dul = dUL; }
    tv[r][lane] = lane < ncl ? d - dU - dl + dul : 0;
    dU = d;
    dUL = dl0;
  }
}

template <bool ENC, typename F>
static __device__ __noinline__ void bs_slow_block(
    const BSSlowIO io, BSChainSmem& sm, int w, int comp, int bi, int bj,
    int nr, int ncl, int32_t top, int32_t left, int32_t corner, int lane,
    bool r0_in_plane) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const bool colok = lane < ncl;
  const int32_t* a = io.a;
  int32_t(*tv)[32] = sm.tv[w];
  uint2(*te)[32] = sm.te[w];        // encoder: (e, floor(2^32 / 2e)) per pixel
  uint16_t(*ts)[34] = sm.ts[w];     // encoder: the symbols of the sweep
  if (ENC && !r0_in_plane) bs_r0_rows<F>(io, comp, r0, c0, nr, ncl, tv, lane);
  // The tile's loads first, all rows in flight (into registers: the compiler
  // does not move a global load above a shared-memory store).  Encoder: the
  // pixel's step and reciprocal go into the (e, M) tile, and lane r keeps row
  // r's non-lossless bits (a code quantises iff it is below cmax).
  uint32_t mynl = 0u;
  {
    int32_t xv[32];
    uint8_t cv[32];
#pragma unroll
    for (int r = 0; r < 32; r++) {
      const bool ok = r < nr && colok;
      const int64_t k = (int64_t)(r0 + r) * io.Wp + c0 + lane;
      xv[r] = (ok && (!ENC || r0_in_plane)) ? __ldcg(a + k) : 0;
      cv[r] = (ok && ENC) ? __ldg(io.codes + (int64_t)(r0 + r) * io.cpitch + c0 + lane)
                          : (uint8_t)CODE_LOSSLESS;
    }
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (!ENC || r0_in_plane) tv[r][lane] = xv[r];
      if (ENC) {
        const int cd = cv[r] & 31;
        const uint32_t e = (uint32_t)sm.etab[cd];
        te[r][lane] = make_uint2(e, sm.mtab[cd]);
        const uint32_t nlw = __ballot_sync(FULL, e != 0u);
        if (lane == r) mynl = nlw;
      }
    }
  }
  const int32_t* myrow = tv[min(lane, nr - 1)];
  const uint2* myem = te[min(lane, nr - 1)];
  // encoder: no pins (lossless pixels have e = 0 and err 0; semi-Lagrangian
  // blocks are never swept); decoder: lossless, escaped and SL pixels
  const uint32_t pw = (!ENC && lane < nr) ? io.pin[(int64_t)(r0 + lane) * io.nchunks + bj] : 0u;
  __syncwarp();
  int32_t l = left;
  int32_t ul = __shfl_up_sync(FULL, left, 1);
  if (lane == 0) ul = corner;
  const uint32_t radius = (uint32_t)io.radius;
  // The skewed sweep: lane = row, step s visits column s - lane.  A lone warp
  // pays every dependent instruction's latency, so the step is kept to the
  // recurrence itself: the operands of step s + 1 are fetched during step s,
  // the quantiser is branch-free on magnitudes (|x| < 2^32), the error in
  // wrapping 32 bits, the symbols go to a tile and out to the stream after.
  int32_t xn = 0;
  uint2 emn = make_uint2(0u, 0u);
  auto operands = [&](int s) {
    const int jj = s - lane;
    const bool act = lane < nr && (unsigned)jj < (unsigned)ncl;
    const int jc = act ? jj : 0;
    xn = myrow[jc];
    if (ENC) {
      emn = myem[jc];
      if (!act) emn.x = 0u;
    }
  };
  operands(0);
#pragma unroll 1
  for (int s = 0; s < 63; s++) {
    const int32_t x = xn;
    const uint32_t e = emn.x, M = emn.y;
    if (s + 1 < 63) operands(s + 1);
    const int jj = s - lane;
    const bool act = lane < nr && (unsigned)jj < (unsigned)ncl;
    const int32_t bb = __shfl_sync(FULL, top, s & 31);
    const int32_t up = __shfl_up_sync(FULL, l, 1);
    const int32_t nu = lane == 0 ? bb : up;
    int32_t v;
    uint32_t sy = 0u;
    if (ENC) {
      // codec.py:140-155: x = R0 - d, q = rha(x / 2e); escape -> err 0, sym 0
      const bool lossy = e != 0u;
      const int64_t x64 = (int64_t)x - ((int64_t)nu + l - ul);
      const bool neg = x64 < 0;
      const uint32_t ax = (uint32_t)(neg ? -x64 : x64);
      const uint32_t m = lossy ? 2u * e : 2u;
      uint32_t q = __umulhi(ax, M);
      uint32_t r = ax - q * m;
      if (r >= m) { q++; r -= m; }
      q += r >= e ? 1u : 0u;
      const bool ok = lossy && q < radius;
      const uint32_t qs = neg ? 0u - q : q;
      v = ok ? (int32_t)(qs * m - (uint32_t)x64) : 0;
      sy = ok ? qs + radius : 0u;
    } else {
      v = ((pw >> (jj & 31)) & 1u)
              ? x
              : (int32_t)((uint32_t)nu + (uint32_t)l - (uint32_t)ul + (uint32_t)x);
    }
    if (act) {
      tv[lane][jj] = v;
      if (ENC) ts[lane][jj] = (uint16_t)sy;
      ul = nu;
      l = v;
    }
  }
  __syncwarp();
  int32_t* out = io.out;
  // err / Z of the block for the interior pass; encoder: the symbols of the
  // non-lossless pixels to their places in the stream (lane = column), the
  // escapes (symbol 0) counted per row for the ll stream
  int64_t myq = 0;
  if (ENC && lane < nr)
    myq = io.qd_row_off[r0 + lane] +
          2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] + comp;
  const unsigned lt = (1u << lane) - 1u;
  int nesc = 0;
  for (int r = 0; r < nr; r++) {
    const int64_t k = (int64_t)(r0 + r) * io.Wp + c0 + lane;
    if (colok) out[k] = tv[r][lane];
    if (ENC) {
      const uint32_t nlw = __shfl_sync(FULL, mynl, r);
      const int64_t qr = __shfl_sync(FULL, myq, r);
      const bool nl = (nlw >> lane) & 1u;
      const uint16_t sv = ts[r][lane];
      if (nl) io.qd[qr + 2 * __popc(nlw & lt)] = sv;
      const int ne = __popc(__ballot_sync(FULL, nl && sv == 0));
      if (lane == r) nesc = ne;
    }
  }
  if (ENC && nesc) atomicAdd(io.row_ll + r0 + lane, nesc);
}

template <typename F, int C>
__device__ __forceinline__ void bs_final_enc1(const BScanIO& io, int bi, int bj,
                                              int lane);
template <int C>
__device__ __forceinline__ void bs_final_dec1(const BScanIO& io, int bi, int bj,
                                              int lane);
template <typename F>
__device__ __forceinline__ void bs_final_enc(const BScanIO& io, int bi, int bj,
                                             int lane);

// One block step of the chain, the general form: any block kind, given the
// exact row above (top), the exact column to the left (left, lane = row) and
// the corner.  Returns the block's exact bottom row in *bot_out and its right
// column in *right_out; publish() hands a bottom row to the block row below
// (a REG bottom row goes down before the right column is known).
template <bool ENC, typename F, typename Publish>
__device__ __forceinline__ void bs_block_step(
    const BScanIO& io, BSChainSmem& sm, int w, int comp, int bi, int bj,
    int nr, int ncl, int32_t cls, int32_t lbv, int32_t lrv, int32_t top,
    int32_t left, int32_t corner, int lane, Publish&& publish,
    int32_t* bot_out, int32_t* right_out) {
  const unsigned FULL = 0xffffffffu;
  const bool colok = lane < ncl;
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int kind0 = cls & 3;
  int kind = kind0;
  int32_t bot = 0, right = 0;
  bool published = false;
  if (kind == BS_REG) {
    const int32_t ll = __shfl_sync(FULL, left, nr - 1);
    const int32_t tl = __shfl_sync(FULL, top, ncl - 1);
    if (ENC) {
      const int code = (cls >> 2) & 31;
      const uint32_t e = (uint32_t)sm.etab[code], m = 2u * e, M = sm.mtab[code];
      const uint32_t rc = bs_res(corner, m, M);
      const uint32_t pb = bs_madd(bs_res(ll, m, M), bs_msub((uint32_t)lbv, rc, m), m);
      const uint32_t pr = bs_madd(bs_res(left, m, M), bs_msub((uint32_t)lrv, rc, m), m);
      // the bottom row is exact unless one of its own residues is a tie:
      // hand it down first, the right column after
      const uint32_t rb = bs_madd(bs_res(top, m, M), pb, m);
      const bool btie = __any_sync(FULL, colok && rb == e);
      if (!btie) {
        bot = colok ? bs_rep(rb, e, m) : 0;
        publish(bot);
        published = true;
      }
      const uint32_t rr = bs_madd(pr, bs_res(tl, m, M), m);
      const bool rtie = __any_sync(FULL, lane < nr && rr == e);
      if (btie || rtie) kind = BS_SLOW;
      else right = bs_rep(rr, e, m);
    } else {
      const uint32_t pb = (uint32_t)ll - (uint32_t)corner + (uint32_t)lbv;
      const uint32_t pr = (uint32_t)left - (uint32_t)corner + (uint32_t)lrv;
      bot = colok ? (int32_t)((uint32_t)top + pb) : 0;
      publish(bot);
      published = true;
      right = (int32_t)(pr + (uint32_t)tl);
    }
  } else if (kind == BS_KNOWN) {
    bot = lbv;
    right = lrv;
  }
  if (kind == BS_SLOW) {
    bs_slow_block<ENC, F>(bs_slow_io(io, comp), sm, w, comp, bi, bj, nr, ncl, top, left, corner,
                          lane, kind0 != BS_REG);
    bot = sm.tv[w][nr - 1][lane];
    right = sm.tv[w][lane][ncl - 1];
    if (lane == 0) io.cls[comp * nblk + (int64_t)bi * io.nbx + bj] = BS_DONE;
    __syncwarp();
  }
  if (!colok) bot = 0;
  if (lane >= nr) right = 0;
  if (!published) publish(bot);
  *bot_out = bot;
  *right_out = right;
}

template <bool ENC, typename F = float>
__global__ void __launch_bounds__(32 * BS_NW, 1)
bs_chain_kernel(const __grid_constant__ BScanIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BSChainSmem& sm = *reinterpret_cast<BSChainSmem*>(smem_raw);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int H = io.H, W = io.W, nbx = io.nbx, nby = io.nby;
  const int64_t nblk = (int64_t)nbx * nby;
  const int ntask = bs_ntask(nby);
  // the interior kernel (a programmatic dependent launch) may start once
  // every chain CTA is resident; it follows the progress marks below
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x < 32) {
    sm.etab[threadIdx.x] = io.e_tab[threadIdx.x];
    sm.mtab[threadIdx.x] = io.mag_tab[threadIdx.x];
  }
  for (;;) {
    if (threadIdx.x == 0) sm.task = atomicAdd(io.ticket, 1);
    __syncthreads();
    const int task = sm.task;
    if (task >= ntask) break;
    // a chain task: fresh handoff counters
    if (threadIdx.x < BS_NW) {
      sm.done[threadIdx.x] = 0;
      sm.pub[threadIdx.x] = 0;
    }
    __syncthreads();
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
      const int64_t rowblk = comp * nblk + (int64_t)bi * nbx;
      const int32_t* clsp = io.cls + rowblk;
      const int32_t* lbp = io.lb + rowblk * 32;
      const int32_t* lrp = io.lr + rowblk * 32;
      int32_t* ebp = io.ebot + rowblk * 32 + lane;
      int32_t* erp = io.eright + rowblk * 32 + lane;
      int32_t left = 0, corner = 0;
      // first warp of a CTA (row above in another CTA): the tagged slots of
      // the next chunk are loaded ahead, so a chunk does not pay an L2 round
      // trip whenever the CTA above is ahead
      const bool gtop = w == 0 && bi > 0;
      uint64_t gq[BS_CH];
      auto gload = [&](int bk0) {
#pragma unroll
        for (int b = 0; b < BS_CH; b++) {
          const int c = 32 * (bk0 + b) + lane;
          gq[b] = c < W ? ld_relaxed_u64(up_gb + c) : 0;
        }
      };
      if (gtop) gload(0);
      // (LB, LR, class) of the next two chunks in flight (cp.async): they do
      // not depend on the recurrence, so the chain never waits on DRAM.  The
      // LB / LR rows of a chunk's blocks are contiguous: lane l copies 16
      // bytes of each (block l / 8); copies past the row's end fill zeros
      auto stage = [&](int ck) {
        const int bk0 = ck * BS_CH, slot = ck & 1;
#pragma unroll
        for (int h = 0; h < BS_CH / 4; h++) {
          const int l = lane + 32 * h;
          const bool vb = bk0 + (l >> 3) < nbx;
          const int off = vb ? 32 * bk0 + 4 * l : 0;
          cp_async<16>(&sm.pfb[w][slot][4 * l], lbp + off, vb);
          cp_async<16>(&sm.pfr[w][slot][4 * l], lrp + off, vb);
        }
        if (lane < BS_CH) {
          const bool vc = bk0 + lane < nbx;
          cp_async<4>(&sm.pfc[w][slot][lane], clsp + (vc ? bk0 + lane : 0), vc);
        }
        cp_async_commit();
      };
      stage(0);
      stage(1);
      auto stamp = [&](int k) {
        if (io.stamps && lane == 0) {
          unsigned long long tn;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
          io.stamps[((int64_t)comp * nby + bi) * 3 + k] = tn;
        }
      };
      stamp(0);
      // the ring slots of block b - HRING/32 must have been read before
      // block b is handed down
      auto ring_wait = [&](int blast) {
        if (out_smem && blast >= BS_HRING / 32)
          spin_ge<BS_SPIN_NS>(&sm.done[w + 1], blast - (BS_HRING / 32 - 1));
      };
      auto put_bot = [&](int bj, int32_t b) {
        const int c = 32 * bj + lane;
        if (!has_next || c >= W) return;
        if (out_smem) sm.hin[w + 1][c & (BS_HRING - 1)] = b;
        else TaggedSlot<int32_t>::put(my_gb + c, tag_me, b);
      };
      // blocks [0, n) of this row are in the ring of the warp below
      auto put_done = [&](int n) {
        if (out_smem) signal_set(&sm.pub[w], n, lane);
      };
      const int32_t e0 = ENC ? sm.etab[0] : 0, m0 = 2 * e0;
#ifdef VFCP_CHAIN_PHASES
      long long pc_t = clock64();
      unsigned long long pc_acc[6] = {0, 0, 0, 0, 0, 0};
#define BS_PHASE(k)                                   \
  if (io.phase) {                                     \
    const long long n_ = clock64();                   \
    pc_acc[k] += (unsigned long long)(n_ - pc_t);     \
    pc_t = n_;                                        \
  }
#else
#define BS_PHASE(k)
#endif
      const int nchunk = (nbx + BS_CH - 1) / BS_CH;
      const int32_t e = e0, m = m0;
      auto add32 = [](int32_t a, int32_t b) -> int32_t {
        return (int32_t)((uint32_t)a + (uint32_t)b);
      };
      auto sub32 = [](int32_t a, int32_t b) -> int32_t {
        return (int32_t)((uint32_t)a - (uint32_t)b);
      };
      // x in [-m, 2m) -> [0, m)
      auto norm = [&](int32_t x) -> int32_t {
        if (!ENC) return x;
        if (x < 0) x += m;
        if (x >= m) x -= m;
        return x;
      };
      // x in [-e - m, e + m] -> [-e, e]
      auto center = [&](int32_t x) -> int32_t {
        if (!ENC) return x;
        if (x > e) x -= m;
        else if (x < -e) x += m;
        return x;
      };
#pragma unroll 1
      for (int ck = 0; ck < nchunk; ck++) {
        const int bk = ck * BS_CH;
        const int nb = min(BS_CH, nbx - bk);
        // ---- the chunk's (class, LB, LR), then the chunk after the next
        // staged into its slot
        cp_async_wait_group<1>();
        __syncwarp();
        const int slot = ck & 1;
        const int32_t cls_l = lane < nb ? sm.pfc[w][slot][lane] : (int32_t)BS_KNOWN;
        int32_t lbv[BS_CH], lrv[BS_CH];
#pragma unroll
        for (int b = 0; b < BS_CH; b++) {
          lbv[b] = sm.pfb[w][slot][32 * b + lane];
          lrv[b] = sm.pfr[w][slot][32 * b + lane];
        }
        // LB at the block's last column (the block's own G term)
        const int ncl_l = max(1, min(32, W - 32 * (bk + lane)));
        const int32_t lk_l = lane < nb ? sm.pfb[w][slot][32 * lane + ncl_l - 1] : 0;
        __syncwarp();
        stage(ck + 2);
        BS_PHASE(0)
        const int kind_l = cls_l & 3;
        // the chunk's fast form: every block KNOWN or REG with the largest
        // step (code 0: e = tau' bounds every error of the frame, so the
        // sums below stay within two moduli); anything else block by block
        bool general = __any_sync(
            FULL, kind_l == BS_SLOW || (ENC && kind_l == BS_REG && ((cls_l >> 2) & 31) != 0));
        // ---- The blocks of a row are coupled only through scalars: with C
        // the block's bottom-right value and T the value above its last
        // column, bottom(j) = top(j) + (C - T)(previous block) + LB(j) and
        // right(i) = left(i) + (T - T(previous block)) + LR(i); for a REG
        // block G = C - T = G(previous) + LB(last column), whatever the row
        // above holds (mod 2e in the encoder; wrapping integers in the
        // decoder).  Lane b holds the scalars of block bk + b.  A chunk of
        // REG blocks has its G chain and q = G(previous) + LB before the row
        // above arrives, so a bottom row is one addition away from its top.
        const bool early = !general && !__any_sync(FULL, lane < nb && kind_l != BS_REG);
        int32_t t31_l = 0;
        int kb[BS_CH];
        int32_t q[BS_CH];
        auto prep = [&]() {
          const int32_t ll = __shfl_sync(FULL, left, nr - 1);
          const int32_t Gin = norm(center(sub32(ll, corner)));
          int32_t G_l = 0, ps_l = 0;
#pragma unroll
          for (int b = 0; b < BS_CH; b++) {
            int32_t gp = __shfl_up_sync(FULL, G_l, 1);
            if (b == 0) gp = Gin;
            if (lane == b) {
              ps_l = gp;
              G_l = kind_l == BS_REG ? norm(add32(gp, lk_l))
                                     : norm(center(sub32(lk_l, t31_l)));
            }
          }
#pragma unroll
          for (int b = 0; b < BS_CH; b++) {
            kb[b] = __shfl_sync(FULL, kind_l, b);
            q[b] = add32(__shfl_sync(FULL, ps_l, b), lbv[b]);   // [0, 2m)
            if (ENC && q[b] >= m) q[b] -= m;
          }
        };
        // T of block bk + lane (only a row's last block can be ragged)
        int32_t top[BS_CH];
        auto gather_t31 = [&]() {
#pragma unroll
          for (int b = 0; b < BS_CH; b++) {
            const int nclb = max(1, min(32, W - 32 * (bk + b)));
            const int32_t x = __shfl_sync(FULL, top[b], nclb - 1);
            if (lane == b) t31_l = x;
          }
        };
        if (early) {
          prep();
          ring_wait(bk + nb - 1);
        }
        BS_PHASE(1)
        // ---- the exact rows above the chunk's blocks
#pragma unroll
        for (int b = 0; b < BS_CH; b++) top[b] = 0;
        if (bi > 0) {
          if (gtop) {
#pragma unroll
            for (int b = 0; b < BS_CH; b++) {
              const int c = 32 * (bk + b) + lane;
              const bool cv = b < nb && c < W;
              uint64_t wv = cv ? gq[b] : 0;
              bool ok = !cv || (uint32_t)(wv >> 32) == tag_up;
              while (!__all_sync(FULL, ok)) {
                if (!ok) {
                  wv = ld_relaxed_u64(up_gb + c);
                  ok = (uint32_t)(wv >> 32) == tag_up;
                }
              }
              top[b] = cv ? (int32_t)(uint32_t)wv : 0;
            }
          } else {
            spin_ge<0>(&sm.pub[w - 1], bk + nb);   // on the critical path: no back-off
#pragma unroll
            for (int b = 0; b < BS_CH; b++) {
              const int c = 32 * (bk + b) + lane;
              if (b < nb && c < W) top[b] = sm.hin[w][c & (BS_HRING - 1)];
            }
          }
        }
        if (ck == 0) stamp(1);
        BS_PHASE(2)
        int32_t bot[BS_CH], right[BS_CH];
        if (!general) {
          if (!early) {
            gather_t31();
            prep();
            ring_wait(bk + nb - 1);
          }
          // ---- bottom rows
          bool tie = false;
#pragma unroll
          for (int b = 0; b < BS_CH; b++) {
            const bool cv = b < nb && 32 * (bk + b) + lane < W;
            int32_t x = add32(top[b], q[b]);    // [-e, m + e)
            if (ENC && x > e) x -= m;
            tie |= ENC && kb[b] == BS_REG && cv && (x == e || x == -e);
            bot[b] = cv ? (kb[b] == BS_REG ? x : lbv[b]) : 0;
          }
          if (ENC && __any_sync(FULL, tie)) {
            general = true;   // a tie on a bottom row: block by block
          } else {
#pragma unroll
            for (int b = 0; b < BS_CH; b++)
              if (b < nb) put_bot(bk + b, bot[b]);
            put_done(bk + nb);
          }
        }
        // the ring reads are complete (the tops are in registers); the next
        // chunk's slots of the CTA above
        if (bi > 0) {
          if (gtop) gload(bk + BS_CH);
          else signal_set(&sm.done[w], bk + nb, lane);
        }
        BS_PHASE(3)
        if (!general) {
          // ---- right columns (lane = row): left -> right, block by block
          if (early) gather_t31();
          int32_t cor_l = __shfl_up_sync(FULL, t31_l, 1);
          if (lane == 0) cor_l = corner;
          const int32_t prs_l = sub32(t31_l, cor_l);
          const int32_t left0 = left;
          bool rtie = false;
#pragma unroll
          for (int b = 0; b < BS_CH; b++) {
            if (b >= nb) break;
            const int32_t ps = __shfl_sync(FULL, prs_l, b);
            int32_t x = center(add32(left, ps));   // [-e, e]
            x = add32(x, lrv[b]);                  // [-e, e + m)
            if (ENC && x > e) x -= m;
            rtie |= ENC && kb[b] == BS_REG && lane < nr && (x == e || x == -e);
            int32_t rg = kb[b] == BS_REG ? x : lrv[b];
            if (lane >= nr) rg = 0;
            right[b] = rg;
            left = rg;
          }
          if (ENC && __any_sync(FULL, rtie)) {
            // a tie on a right column (rare): again block by block, the
            // block with the tie swept exactly (its bottom row went down
            // already and is unchanged)
            left = left0;
#pragma unroll
            for (int b = 0; b < BS_CH; b++) {
              if (b >= nb) break;
              const int32_t ps = __shfl_sync(FULL, prs_l, b);
              int32_t x = center(add32(left, ps));
              x = add32(x, lrv[b]);
              if (x > e) x -= m;
              const bool tb = kb[b] == BS_REG && lane < nr && (x == e || x == -e);
              int32_t rg = kb[b] == BS_REG ? x : lrv[b];
              if (__any_sync(FULL, tb)) {
                const int bj = bk + b, ncl = min(32, W - 32 * bj);
                const int32_t cb = __shfl_sync(FULL, cor_l, b);
                bs_slow_block<ENC, F>(bs_slow_io(io, comp), sm, w, comp, bi, bj,
                                      nr, ncl, top[b], left, cb, lane, false);
                rg = sm.tv[w][lane][ncl - 1];
                if (lane == 0) io.cls[rowblk + bj] = BS_DONE;
                __syncwarp();
              }
              if (lane >= nr) rg = 0;
              right[b] = rg;
              left = rg;
            }
          }
          // (only a row's last block can be ragged: t31 is column 31 here)
          corner = __shfl_sync(FULL, t31_l, nb - 1);
        }
        if (general) {
          // ---- block by block, any block kind (not unrolled: the chunk's
          // registers are picked by selects so the loop body stays small)
#pragma unroll 1
          for (int b = 0; b < nb; b++) {
            const int bj = bk + b, ncl = min(32, W - 32 * bj);
            const int32_t cls = __shfl_sync(FULL, cls_l, b);
            int32_t tb = top[0], lb = lbv[0], lr = lrv[0];
#pragma unroll
            for (int k = 1; k < BS_CH; k++)
              if (b == k) { tb = top[k]; lb = lbv[k]; lr = lrv[k]; }
            ring_wait(bj);
            int32_t bo, ri;
            bs_block_step<ENC, F>(io, sm, w, comp, bi, bj, nr, ncl, cls, lb, lr,
                                  tb, left, corner, lane,
                                  [&](int32_t v) {
                                    put_bot(bj, v);
                                    put_done(bj + 1);
                                  },
                                  &bo, &ri);
#pragma unroll
            for (int k = 0; k < BS_CH; k++)
              if (b == k) { bot[k] = bo; right[k] = ri; }
            corner = __shfl_sync(FULL, tb, 31);
            left = ri;
          }
        }
        BS_PHASE(4)
        // ---- the blocks' exact edges for the interior pass (coalesced)
#pragma unroll
        for (int b = 0; b < BS_CH; b++) {
          if (b >= nb) break;
          ebp[(int64_t)(bk + b) * 32] = bot[b];
          erp[(int64_t)(bk + b) * 32] = right[b];
        }
        // progress for the interior kernel: the block edges (and any swept
        // block) are visible GPU-wide before the mark
        if ((bk + nb) % BS_SEG == 0 || bk + nb == nbx) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            st_release_gpu_u64(io.prog + (int64_t)comp * nby + bi,
                               ((unsigned long long)io.frame_tag << 32) | (unsigned)(bk + nb));
        }
        BS_PHASE(5)
      }
#ifdef VFCP_CHAIN_PHASES
      if (io.phase && comp == 0 && lane == 0)
        for (int k = 0; k < 6; k++) io.phase[bi * 8 + k] = pc_acc[k];
#endif
#undef BS_PHASE
      cp_async_wait_all();   // the staged chunks past the row's end
      stamp(2);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ phase C
// The interior of block (bi, bj), component C, by one warp (lane = column,
// rows streamed with three rows of loads in flight).
// Encoder (bs_final_enc1):
//   REG       err(i, j) = rep(zT(j) + zL(i) - zC - delta(i, j))  (mod m)
//             with zT = errT + deltaT etc. (Z = recon - prev of the exact
//             boundary, enc_block.cu), ties in raster order; the symbol is
//             (R0 + D(err)) / m exactly;
//   SLOW/DONE err from the chain's sweep (its symbols are written);
//   KNOWN     recon(t) already written by the block kernel;
// recon(t) = orig + err goes into component C of the (u, v) pair plane.
// Decoder (bs_final_dec1): REG: Z = ZU + ZL - ZUL + A, i.e. per row
// Z(i, j) = Z(i-1, j) + (ZL(i) - ZL(i-1)) + sum_{b<=j} A(i, b) (warp scan;
// wrapping uint32 arithmetic is exact: recon fits int32) with A =
// (sym - radius) * 2e; SLOW: Z from the chain's sweep; KNOWN: written by
// the block kernel (dec_block.cu).  recon = recon(t-1) + Z goes out to the
// pair plane, as float64 (codec.py:425-426 recon * (1/S), exact) and
// optionally as int64.
template <typename F, int C>
__device__ __forceinline__ void bs_final_enc1(const BScanIO& io, int bi, int bj,
                                              int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, io.H - r0), ncl = min(32, io.W - c0);
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int Wp = io.Wp, W = io.W;
  const int32_t cl = __ldcg(io.cls + C * nblk + blk);
  const int kind = cl & 3, code = (cl >> 2) & 31;
  if (kind == BS_KNOWN) return;
  const bool reg = kind == BS_REG;
  const bool colok = lane < ncl;
  const int j = c0 + (colok ? lane : ncl - 1);
  const F* op = static_cast<const F*>(io.orig[C]);
  const int32_t* pvc = io.prevrec ? reinterpret_cast<const int32_t*>(io.prevrec) + C : nullptr;
  auto pvat = [&](int i, int jj) -> int32_t {
    return pvc ? __ldg(pvc + 2 * ((int64_t)i * Wp + jj)) : 0;
  };
  auto fx = [&](int i, int jj) -> int32_t {
    return fixed_t(__ldg(op + (int64_t)i * W + jj), io.S);
  };
  int32_t* recw = reinterpret_cast<int32_t*>(io.rec) + C;
  if (!reg) {
    // SLOW / DONE: err from the chain's sweep
#pragma unroll 4
    for (int i = 0; i < nr; i++) {
      if (colok) {
        const int32_t err = __ldcg(io.out[C] + (int64_t)(r0 + i) * Wp + j);
        recw[2 * ((int64_t)(r0 + i) * Wp + j)] = fx(r0 + i, j) + err;
      }
    }
    return;
  }
  const uint32_t e = (uint32_t)io.e_tab[code], m = 2u * e;
  const uint32_t M = io.mag_tab[code], c32 = io.c32_tab[code];
  const int32_t* eb = io.ebot + C * nblk * 32;
  const int32_t* er = io.eright + C * nblk * 32;
  const int32_t errT = (bi > 0 && colok) ? __ldcg(eb + (blk - io.nbx) * 32 + lane) : 0;
  const int32_t errL = (bj > 0 && lane < nr) ? __ldcg(er + (blk - 1) * 32 + lane) : 0;
  const int32_t errC = (bi > 0 && bj > 0) ? __ldcg(eb + (blk - io.nbx - 1) * 32 + 31) : 0;
  int64_t dT = 0, dL = 0, dC = 0;
  if (bi > 0) {
    dT = colok ? (int64_t)fx(r0 - 1, j) - pvat(r0 - 1, j) : 0;
    if (bj > 0) dC = (int64_t)fx(r0 - 1, c0 - 1) - pvat(r0 - 1, c0 - 1);
  }
  if (bj > 0 && lane < nr) dL = (int64_t)fx(r0 + lane, c0 - 1) - pvat(r0 + lane, c0 - 1);
  const uint32_t zT = bs_madd(bs_res(errT, m, M), res_i64(dT, m, M, c32), m);
  const uint32_t zC = bs_madd(bs_res(errC, m, M), res_i64(dC, m, M, c32), m);
  const uint32_t zL = bs_madd(bs_res(errL, m, M), res_i64(dL, m, M, c32), m);
  const uint32_t base = bs_msub(zT, zC, m);
  int32_t dU = (int32_t)dT, eU = errT, dLU = (int32_t)dC, eLU = errC;
  int64_t qb = 0;
  if (lane < nr)
    qb = io.qd_row_off[r0 + lane] +
         2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] + C;
  F bo[4];
  int32_t bp[4];
  auto issue = [&](int i, int sl) {
    if (i < nr) {
      bo[sl] = __ldg(op + (int64_t)(r0 + i) * W + j);
      bp[sl] = pvat(r0 + i, j);
    }
  };
  issue(0, 0);
  issue(1, 1);
  issue(2, 2);
  for (int i0 = 0; i0 < nr; i0 += 4)
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    const int i = i0 + kk;
    if (i >= nr) break;
    issue(i + 3, (kk + 3) & 3);
    const int32_t o = fixed_t(bo[kk], io.S);
    const int32_t pr = bp[kk];
    const int64_t d64 = (int64_t)o - pr;
    const int32_t d32 = (int32_t)d64;
    const int32_t dLi = __shfl_sync(FULL, (int32_t)dL, i);
    const int32_t errLi = __shfl_sync(FULL, errL, i);
    int32_t dl = __shfl_up_sync(FULL, d32, 1);
    int32_t dul = __shfl_up_sync(FULL, dU, 1);
    if (lane == 0) { dl = dLi; dul = dLU; }
    const int32_t R0 = d32 - dU - dl + dul;
    const uint32_t zl = __shfl_sync(FULL, zL, i);
    const uint32_t sres = bs_msub(bs_madd(base, zl, m), res_i64(d64, m, M, c32), m);
    const bool tie = colok && sres == e;
    int32_t err = bs_rep(sres, e, m);
    uint32_t tm = __ballot_sync(FULL, tie);
    if (tm) {
      // raster order within the row: x = R0 - (errU + errL - errUL)
      int32_t cur = tie ? 0 : err;
      while (tm) {
        const int jj = __ffs(tm) - 1;
        tm &= tm - 1u;
        int32_t el = __shfl_up_sync(FULL, cur, 1);
        int32_t eul = __shfl_up_sync(FULL, eU, 1);
        if (lane == 0) { el = errLi; eul = eLU; }
        if (lane == jj) {
          const int64_t x = (int64_t)R0 - ((int64_t)eU + el - eul);
          cur = x > 0 ? (int32_t)e : -(int32_t)e;
        }
      }
      err = cur;
    }
    int32_t el = __shfl_up_sync(FULL, err, 1);
    int32_t eul = __shfl_up_sync(FULL, eU, 1);
    if (lane == 0) { el = errLi; eul = eLU; }
    // x + err = q * m exactly (|R0| < 2^30 in a REG block)
    const int64_t n = (int64_t)R0 + err - eU - el + eul;
    const uint32_t an = (uint32_t)(n < 0 ? -n : n);
    uint32_t qa = __umulhi(an, M);
    if (qa * m != an) qa++;
    const int32_t q = n < 0 ? -(int32_t)qa : (int32_t)qa;
    const int64_t qr = __shfl_sync(FULL, qb, i);
    if (colok) {
      recw[2 * ((int64_t)(r0 + i) * Wp + j)] = o + err;
      io.qd[qr + 2 * lane] = (uint16_t)(q + io.radius);
    }
    dU = d32;
    eU = colok ? err : 0;
    dLU = dLi;
    eLU = errLi;
  }
}

// Both components of a block that is REG and narrow in both (the usual
// case): with s(i, j) = ZT(j) + ZL(i) - ZC - delta(i, j) as integers (ZT =
// errT + deltaT etc. of the exact boundary; |s| < 2^31) the error is err = s
// - k m with k the integer nearest to s / m, and since D(s) = -R0 the symbol
// is (R0 + D(err)) / m = -D(k) with k = 0 on the boundary: one rounding per
// pixel and two shuffles, no residues.  A tie (s - k m = +-e) takes the sign
// of x = R0 - (errU + errL - errUL) in raster order (rare).
template <typename F>
__device__ __forceinline__ void bs_final_enc2(const BScanIO& io, int bi, int bj,
                                              int lane, int code) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, io.H - r0), ncl = min(32, io.W - c0);
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int Wp = io.Wp, W = io.W;
  const bool colok = lane < ncl;
  const int j = c0 + (colok ? lane : ncl - 1);
  const F* opu = static_cast<const F*>(io.orig[0]);
  const F* opv = static_cast<const F*>(io.orig[1]);
  const int2* pv = io.prevrec;
  const float Sf = (float)io.S;
  auto delta_at = [&](int i, int jj) -> int2 {
    const int2 p = pv ? __ldg(pv + (int64_t)i * Wp + jj) : make_int2(0, 0);
    return make_int2(fixed_t(__ldg(opu + (int64_t)i * W + jj), io.S) - p.x,
                     fixed_t(__ldg(opv + (int64_t)i * W + jj), io.S) - p.y);
  };
  (void)Sf;
  const uint32_t e = (uint32_t)io.e_tab[code], m = 2u * e, M = io.mag_tab[code];
  const int32_t* ebu = io.ebot;
  const int32_t* ebv = io.ebot + nblk * 32;
  const int32_t* eru = io.eright;
  const int32_t* erv = io.eright + nblk * 32;
  // exact boundary: Z = err + delta of the row above, the column to the left
  // and the corner (zero outside the frame)
  int32_t eTu = 0, eTv = 0, eLu = 0, eLv = 0, eCu = 0, eCv = 0;
  int2 dT = make_int2(0, 0), dL = make_int2(0, 0), dC = make_int2(0, 0);
  if (bi > 0) {
    eTu = colok ? __ldcg(ebu + (blk - io.nbx) * 32 + lane) : 0;
    eTv = colok ? __ldcg(ebv + (blk - io.nbx) * 32 + lane) : 0;
    if (colok) dT = delta_at(r0 - 1, j);
    if (bj > 0) {
      eCu = __ldcg(ebu + (blk - io.nbx - 1) * 32 + 31);
      eCv = __ldcg(ebv + (blk - io.nbx - 1) * 32 + 31);
      dC = delta_at(r0 - 1, c0 - 1);
    }
  }
  if (bj > 0 && lane < nr) {
    eLu = __ldcg(eru + (blk - 1) * 32 + lane);
    eLv = __ldcg(erv + (blk - 1) * 32 + lane);
    dL = delta_at(r0 + lane, c0 - 1);
  }
  const int32_t baseu = (eTu + dT.x) - (eCu + dC.x);
  const int32_t basev = (eTv + dT.y) - (eCv + dC.y);
  const int32_t ZLu = eLu + dL.x, ZLv = eLv + dL.y;   // lane = row
  // symbol positions relative to the block's first row (32 rows x 2 W
  // symbols fit 32 bits)
  const int64_t q0 = io.qd_row_off[r0] + 2 * (int64_t)io.pre_nl[(int64_t)r0 * io.nchunks + bj];
  uint32_t qrel = 0;
  if (lane < nr)
    qrel = (uint32_t)(io.qd_row_off[r0 + lane] +
                      2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] - q0);
  uint16_t* qdb = io.qd + q0 + 2 * lane;
  int2* recp = io.rec + (int64_t)r0 * Wp + j;
  int32_t dUu = dT.x, dUv = dT.y, eUu = eTu, eUv = eTv, kUu = 0, kUv = 0;
  F bu[4], bv[4];
  int2 bp[4];
  auto issue = [&](int i, int sl) {
    if (i < nr) {
      bu[sl] = __ldg(opu + (int64_t)(r0 + i) * W + j);
      bv[sl] = __ldg(opv + (int64_t)(r0 + i) * W + j);
      bp[sl] = pv ? __ldg(pv + (int64_t)(r0 + i) * Wp + j) : make_int2(0, 0);
    }
  };
  issue(0, 0);
  issue(1, 1);
  issue(2, 2);
  for (int i0 = 0; i0 < nr; i0 += 4)
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    const int i = i0 + kk;
    if (i >= nr) break;
    issue(i + 3, (kk + 3) & 3);
    const int32_t ou = fixed_t(bu[kk], io.S), ov = fixed_t(bv[kk], io.S);
    const int32_t du = ou - bp[kk].x, dv = ov - bp[kk].y;
    const int32_t su = baseu + __shfl_sync(FULL, ZLu, i) - du;
    const int32_t sv = basev + __shfl_sync(FULL, ZLv, i) - dv;
    bool tu, tv;
    int32_t ku = bs_knear(su, e, m, M, &tu);
    int32_t kv = bs_knear(sv, e, m, M, &tv);
    int32_t eu = su - ku * (int32_t)m, ev = sv - kv * (int32_t)m;
    if (__any_sync(FULL, colok && (tu | tv))) {
      // ties in raster order within the row, per component
      const int iu = max(i - 1, 0);
#pragma unroll
      for (int c = 0; c < 2; c++) {
        unsigned tm = __ballot_sync(FULL, colok && (c ? tv : tu));
        if (!tm) continue;
        const int32_t d = c ? dv : du, dU = c ? dUv : dUu, eU = c ? eUv : eUu;
        const int32_t eL = c ? eLv : eLu, ZL = c ? ZLv : ZLu;
        // left boundary of this row and of the row above (lane 0 only)
        const int32_t eLi = __shfl_sync(FULL, eL, i), dLi = __shfl_sync(FULL, ZL - eL, i);
        int32_t eLp = __shfl_sync(FULL, eL, iu), dLp = __shfl_sync(FULL, ZL - eL, iu);
        if (i == 0) { eLp = c ? eCv : eCu; dLp = c ? dC.y : dC.x; }
        const int32_t err0 = c ? ev : eu;
        int32_t cur = (c ? tv : tu) ? 0 : err0;
        while (tm) {
          const int jj = __ffs(tm) - 1;
          tm &= tm - 1u;
          int32_t el = __shfl_up_sync(FULL, cur, 1);
          int32_t eul = __shfl_up_sync(FULL, eU, 1);
          int32_t dl = __shfl_up_sync(FULL, d, 1);
          int32_t dul = __shfl_up_sync(FULL, dU, 1);
          if (lane == 0) { el = eLi; eul = eLp; dl = dLi; dul = dLp; }
          if (lane == jj) {
            const int64_t R0 = (int64_t)d - dU - dl + dul;
            const int64_t x = R0 - ((int64_t)eU + el - eul);
            cur = x > 0 ? (int32_t)e : -(int32_t)e;
          }
        }
        // err = s - k m: the other sign of a tie moves k by one
        if ((c ? tv : tu) && cur != err0) {
          if (c) { kv += err0 > cur ? 1 : -1; ev = cur; }
          else { ku += err0 > cur ? 1 : -1; eu = cur; }
        }
      }
    }
    int32_t kLu = __shfl_up_sync(FULL, ku, 1), kLv = __shfl_up_sync(FULL, kv, 1);
    int32_t kULu = __shfl_up_sync(FULL, kUu, 1), kULv = __shfl_up_sync(FULL, kUv, 1);
    if (lane == 0) { kLu = kLv = kULu = kULv = 0; }
    const int32_t qu = kUu + kLu - kULu - ku, qv = kUv + kLv - kULv - kv;
    const uint32_t qo = __shfl_sync(FULL, qrel, i);
    if (colok) {
      recp[(int64_t)i * Wp] = make_int2(ou + eu, ov + ev);
      *reinterpret_cast<uint32_t*>(qdb + qo) =
          (uint32_t)(qu + io.radius) | ((uint32_t)(qv + io.radius) << 16);
    }
    kUu = ku; kUv = kv;
    dUu = du; dUv = dv;
    eUu = colok ? eu : 0; eUv = colok ? ev : 0;
  }
}

// The same block four pixels per lane (float32 input, full 32x32 block, rows
// 16-byte aligned): lane = (row in a group of four, column quad), eight
// groups per block, 16-byte loads with three groups in flight.  Every k is
// independent of the others (see above); the symbol needs the k of the
// left / upper / upper-left pixels, which come from the lane's own quad, the
// lane to the left and the group of rows above (one rotation by 8 lanes
// carries the previous group's last row into lanes 0-7).  A tie anywhere
// sends the block to the row-streamed form.  Returns false on a tie.
__device__ __forceinline__ bool bs_final_enc4(const BScanIO& io, int bi, int bj,
                                              int lane, int code) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int Wp = io.Wp, W = io.W;
  const int rq = lane >> 3, cq = lane & 7;
  const float* opu = static_cast<const float*>(io.orig[0]);
  const float* opv = static_cast<const float*>(io.orig[1]);
  const int2* pv = io.prevrec;
  const float Sf = (float)io.S;
  const uint32_t e = (uint32_t)io.e_tab[code], m = 2u * e, M = io.mag_tab[code];
  const int32_t* ebu = io.ebot;
  const int32_t* ebv = io.ebot + nblk * 32;
  const int32_t* eru = io.eright;
  const int32_t* erv = io.eright + nblk * 32;
  // delta = orig - recon(t-1) of four pixels (u0 v0 u1 v1 ...)
  struct Quad { float4 u, v; int4 p01, p23; };
  auto load_quad = [&](int i) -> Quad {
    Quad q;
    const int64_t n = (int64_t)i * W + c0 + 4 * cq;
    q.u = __ldg(reinterpret_cast<const float4*>(opu + n));
    q.v = __ldg(reinterpret_cast<const float4*>(opv + n));
    if (pv) {
      const int4* pp = reinterpret_cast<const int4*>(pv + (int64_t)i * Wp + c0 + 4 * cq);
      q.p01 = __ldg(pp);
      q.p23 = __ldg(pp + 1);
    } else {
      q.p01 = q.p23 = make_int4(0, 0, 0, 0);
    }
    return q;
  };
  // exact boundary: Z = err + delta of the row above (the lane's four
  // columns), the column to the left (lane = row) and the corner
  int32_t bu[4] = {0, 0, 0, 0}, bv[4] = {0, 0, 0, 0};
  int32_t ZLu = 0, ZLv = 0, eLu = 0, eLv = 0;
  auto delta1 = [&](int i, int jj) -> int2 {
    const int2 p = pv ? __ldg(pv + (int64_t)i * Wp + jj) : make_int2(0, 0);
    return make_int2(fixed_of_f32(__ldg(opu + (int64_t)i * W + jj), Sf) - p.x,
                     fixed_of_f32(__ldg(opv + (int64_t)i * W + jj), Sf) - p.y);
  };
  if (bi > 0) {
    const int4 tu = __ldcg(reinterpret_cast<const int4*>(ebu + (blk - io.nbx) * 32) + cq);
    const int4 tv = __ldcg(reinterpret_cast<const int4*>(ebv + (blk - io.nbx) * 32) + cq);
    const Quad q = load_quad(r0 - 1);
    int32_t zcu = 0, zcv = 0;
    if (bj > 0) {
      const int2 dC = delta1(r0 - 1, c0 - 1);
      zcu = __ldcg(ebu + (blk - io.nbx - 1) * 32 + 31) + dC.x;
      zcv = __ldcg(ebv + (blk - io.nbx - 1) * 32 + 31) + dC.y;
    }
    bu[0] = tu.x + (fixed_of_f32(q.u.x, Sf) - q.p01.x) - zcu;
    bu[1] = tu.y + (fixed_of_f32(q.u.y, Sf) - q.p01.z) - zcu;
    bu[2] = tu.z + (fixed_of_f32(q.u.z, Sf) - q.p23.x) - zcu;
    bu[3] = tu.w + (fixed_of_f32(q.u.w, Sf) - q.p23.z) - zcu;
    bv[0] = tv.x + (fixed_of_f32(q.v.x, Sf) - q.p01.y) - zcv;
    bv[1] = tv.y + (fixed_of_f32(q.v.y, Sf) - q.p01.w) - zcv;
    bv[2] = tv.z + (fixed_of_f32(q.v.z, Sf) - q.p23.y) - zcv;
    bv[3] = tv.w + (fixed_of_f32(q.v.w, Sf) - q.p23.w) - zcv;
  }
  if (bj > 0) {
    eLu = __ldcg(eru + (blk - 1) * 32 + lane);
    eLv = __ldcg(erv + (blk - 1) * 32 + lane);
    const int2 dL = delta1(r0 + lane, c0 - 1);
    ZLu = eLu + dL.x;
    ZLv = eLv + dL.y;
  }
  // symbol positions relative to the block's first row (lane = row)
  const int64_t q0 = io.qd_row_off[r0] + 2 * (int64_t)io.pre_nl[(int64_t)r0 * io.nchunks + bj];
  const uint32_t qrel =
      (uint32_t)(io.qd_row_off[r0 + lane] +
                 2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] - q0);
  uint32_t* qdb = reinterpret_cast<uint32_t*>(io.qd + q0) + 4 * cq;
  int4* recp = reinterpret_cast<int4*>(io.rec + (int64_t)(r0 + rq) * Wp + c0 + 4 * cq);
  const int32_t rad = io.radius;
  int32_t kqu[4] = {0, 0, 0, 0}, kqv[4] = {0, 0, 0, 0};   // k of the group above
  Quad st[3];
  st[0] = load_quad(r0 + rq);
  st[1] = load_quad(r0 + 4 + rq);
#pragma unroll
  for (int it = 0; it < 8; it++) {
    if (it + 2 < 8) st[(it + 2) % 3] = load_quad(r0 + 4 * (it + 2) + rq);
    const Quad& q = st[it % 3];
    const int i = 4 * it + rq;
    const int32_t zlu = __shfl_sync(FULL, ZLu, i), zlv = __shfl_sync(FULL, ZLv, i);
    int32_t ou[4], ov[4], ku[4], kv[4];
    ou[0] = fixed_of_f32(q.u.x, Sf); ou[1] = fixed_of_f32(q.u.y, Sf);
    ou[2] = fixed_of_f32(q.u.z, Sf); ou[3] = fixed_of_f32(q.u.w, Sf);
    ov[0] = fixed_of_f32(q.v.x, Sf); ov[1] = fixed_of_f32(q.v.y, Sf);
    ov[2] = fixed_of_f32(q.v.z, Sf); ov[3] = fixed_of_f32(q.v.w, Sf);
    const int32_t pu[4] = {q.p01.x, q.p01.z, q.p23.x, q.p23.z};
    const int32_t pw[4] = {q.p01.y, q.p01.w, q.p23.y, q.p23.w};
    bool tie = false;
    int32_t ru[4], rv[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
      bool tu, tv;
      const int32_t su = bu[c] + zlu - (ou[c] - pu[c]);
      const int32_t sv = bv[c] + zlv - (ov[c] - pw[c]);
      ku[c] = bs_knear(su, e, m, M, &tu);
      kv[c] = bs_knear(sv, e, m, M, &tv);
      tie |= tu | tv;
      ru[c] = ou[c] + (su - ku[c] * (int32_t)m);
      rv[c] = ov[c] + (sv - kv[c] * (int32_t)m);
    }
    if (__any_sync(FULL, tie)) return false;
    // k of the row above: a rotation by one group (lanes 0-7 get the last
    // row of the group before), then of the pixel to the left
    int32_t kUu[4], kUv[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
      kUu[c] = __shfl_sync(FULL, rq == 3 ? kqu[c] : ku[c], (lane + 24) & 31);
      kUv[c] = __shfl_sync(FULL, rq == 3 ? kqv[c] : kv[c], (lane + 24) & 31);
    }
    int32_t kLu = __shfl_up_sync(FULL, ku[3], 1), kLv = __shfl_up_sync(FULL, kv[3], 1);
    int32_t kULu = __shfl_up_sync(FULL, kUu[3], 1), kULv = __shfl_up_sync(FULL, kUv[3], 1);
    if (cq == 0) { kLu = kLv = kULu = kULv = 0; }
    uint32_t sy[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int32_t lu = c ? ku[c - 1] : kLu, lv = c ? kv[c - 1] : kLv;
      const int32_t ulu = c ? kUu[c - 1] : kULu, ulv = c ? kUv[c - 1] : kULv;
      const int32_t qu = kUu[c] + lu - ulu - ku[c], qv = kUv[c] + lv - ulv - kv[c];
      sy[c] = (uint32_t)(qu + rad) | ((uint32_t)(qv + rad) << 16);
      kqu[c] = ku[c];
      kqv[c] = kv[c];
    }
    const uint32_t qo = __shfl_sync(FULL, qrel, i);
    int4* rp = recp + (int64_t)it * 2 * Wp;   // four rows of Wp pairs down
    rp[0] = make_int4(ru[0], rv[0], ru[1], rv[1]);
    rp[1] = make_int4(ru[2], rv[2], ru[3], rv[3]);
    uint32_t* qp = qdb + (qo >> 1);
    qp[0] = sy[0]; qp[1] = sy[1]; qp[2] = sy[2]; qp[3] = sy[3];
  }
  return true;
}

template <typename F>
__device__ __forceinline__ void bs_final_enc(const BScanIO& io, int bi, int bj,
                                             int lane) {
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int32_t cu = __ldcg(io.cls + blk), cv = __ldcg(io.cls + nblk + blk);
  const int32_t want = BS_REG | BS_NARROW;
  if ((cu & (3 | BS_NARROW)) == want && (cv & (3 | BS_NARROW)) == want) {
    if (sizeof(F) == 4 && io.vec4 && 32 * bi + 32 <= io.H && 32 * bj + 32 <= io.W &&
        bs_final_enc4(io, bi, bj, lane, (cu >> 2) & 31))
      return;
    bs_final_enc2<F>(io, bi, bj, lane, (cu >> 2) & 31);
  } else {
    bs_final_enc1<F, 0>(io, bi, bj, lane);
    bs_final_enc1<F, 1>(io, bi, bj, lane);
  }
}

// Decoder, both components of a full block whose pixels share one code (the
// decoder's fast block kernel marks it BS_NARROW): four pixels per lane, lane
// = (band of eight rows, column quad).  Z = ZT(j) + ZL(i) - ZC + P(i, j), P
// the block's 2D prefix sum of A = (sym - radius) * 2e (wrapping uint32).
// Pass 1 sums the band's columns (lane-local) and scans them along the row,
// which gives P at the band's last row, hence the offsets of the bands
// below; pass 2 walks the band's rows: one row scan each, the column sums
// running in registers.  The symbols stay in registers between the passes.
__device__ __forceinline__ void bs_final_dec4(const BScanIO& io, int bi, int bj,
                                              int lane, int code) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int Wp = io.Wp, W = io.W;
  const int rq = lane >> 3, cq = lane & 7;
  const uint32_t e2 = 2u * (uint32_t)io.e_tab[code], rad = (uint32_t)io.radius;
  const int32_t* ebu = io.ebot;
  const int32_t* ebv = io.ebot + nblk * 32;
  const int32_t* eru = io.eright;
  const int32_t* erv = io.eright + nblk * 32;
  // symbols of the band's eight rows (lane = row holds the row offsets)
  const int64_t q0 = io.qd_row_off[r0] + 2 * (int64_t)io.pre_nl[(int64_t)r0 * io.nchunks + bj];
  const uint32_t qrel =
      (uint32_t)(io.qd_row_off[r0 + lane] +
                 2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] - q0);
  const uint32_t* qdb = reinterpret_cast<const uint32_t*>(io.qd + q0) + 4 * cq;
  // pass 1 reads the band's symbols, pass 2 reads them again (L2 hits)
  auto load_sym = [&](int it, uint32_t (&x)[4]) {
    const uint32_t qo = __shfl_sync(FULL, qrel, 8 * rq + it);
    const uint32_t* sp = qdb + (qo >> 1);
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = __ldg(sp + k);
  };
  // recon(t-1) of the band's first rows in flight
  const int2* pv = io.prevrec;
  auto load_prev = [&](int it, int4& a, int4& b) {
    if (pv) {
      const int4* pp = reinterpret_cast<const int4*>(
          pv + (int64_t)(r0 + 8 * rq + it) * Wp + c0 + 4 * cq);
      a = __ldg(pp);
      b = __ldg(pp + 1);
    } else {
      a = b = make_int4(0, 0, 0, 0);
    }
  };
  // exact boundary (Z of the row above, the column to the left, the corner)
  uint32_t ou[4] = {0, 0, 0, 0}, ov[4] = {0, 0, 0, 0};   // ZT(j) - ZC + band offset
  uint32_t zLu = 0, zLv = 0;
  if (bi > 0) {
    const int4 tu = __ldcg(reinterpret_cast<const int4*>(ebu + (blk - io.nbx) * 32) + cq);
    const int4 tv = __ldcg(reinterpret_cast<const int4*>(ebv + (blk - io.nbx) * 32) + cq);
    uint32_t zcu = 0, zcv = 0;
    if (bj > 0) {
      zcu = (uint32_t)__ldcg(ebu + (blk - io.nbx - 1) * 32 + 31);
      zcv = (uint32_t)__ldcg(ebv + (blk - io.nbx - 1) * 32 + 31);
    }
    ou[0] = (uint32_t)tu.x - zcu; ou[1] = (uint32_t)tu.y - zcu;
    ou[2] = (uint32_t)tu.z - zcu; ou[3] = (uint32_t)tu.w - zcu;
    ov[0] = (uint32_t)tv.x - zcv; ov[1] = (uint32_t)tv.y - zcv;
    ov[2] = (uint32_t)tv.z - zcv; ov[3] = (uint32_t)tv.w - zcv;
  }
  if (bj > 0) {
    zLu = (uint32_t)__ldcg(eru + (blk - 1) * 32 + lane);
    zLv = (uint32_t)__ldcg(erv + (blk - 1) * 32 + lane);
  }
  auto amp = [&](uint32_t s2, uint32_t& au, uint32_t& av) {
    au = ((s2 & 0xffffu) - rad) * e2;
    av = ((s2 >> 16) - rad) * e2;
  };
  // inclusive scan of the lane's quad along the row (8 lanes per row)
  auto row_scan = [&](uint32_t (&x)[4]) {
    x[1] += x[0]; x[2] += x[1]; x[3] += x[2];
    uint32_t t = x[3];
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, t, o, 8);
      if (cq >= o) t += y;
    }
    const uint32_t ex = t - x[3];
    x[0] += ex; x[1] += ex; x[2] += ex; x[3] += ex;
  };
  // ---- pass 1: P at the band's last row, offsets of the bands below
  {
    uint32_t cu[4] = {0, 0, 0, 0}, cv[4] = {0, 0, 0, 0};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      uint32_t sy[4][4];
#pragma unroll
      for (int it = 0; it < 4; it++) load_sym(4 * h + it, sy[it]);
#pragma unroll
      for (int it = 0; it < 4; it++)
#pragma unroll
        for (int k = 0; k < 4; k++) {
          uint32_t au, av;
          amp(sy[it][k], au, av);
          cu[k] += au;
          cv[k] += av;
        }
    }
    row_scan(cu);
    row_scan(cv);
    // exclusive scan over the four bands (lanes l, l + 8, l + 16, l + 24)
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t tu = cu[k], tv = cv[k];
      uint32_t y = __shfl_up_sync(FULL, tu, 8), z = __shfl_up_sync(FULL, tv, 8);
      if (rq >= 1) { tu += y; tv += z; }
      y = __shfl_up_sync(FULL, tu, 16); z = __shfl_up_sync(FULL, tv, 16);
      if (rq >= 2) { tu += y; tv += z; }
      ou[k] += tu - cu[k];
      ov[k] += tv - cv[k];
    }
  }
  // ---- pass 2: the band's rows
  int4* recp = reinterpret_cast<int4*>(io.rec + (int64_t)(r0 + 8 * rq) * Wp + c0 + 4 * cq);
  double2* fu = reinterpret_cast<double2*>(io.f64[0] + (int64_t)(r0 + 8 * rq) * W + c0 + 4 * cq);
  double2* fv = reinterpret_cast<double2*>(io.f64[1] + (int64_t)(r0 + 8 * rq) * W + c0 + 4 * cq);
  const double inv_S = io.inv_S;
  int4 pa[3], pb[3];
  uint32_t sq[3][4];
  load_prev(0, pa[0], pb[0]);
  load_sym(0, sq[0]);
  load_prev(1, pa[1], pb[1]);
  load_sym(1, sq[1]);
#pragma unroll
  for (int it = 0; it < 8; it++) {
    if (it + 2 < 8) {
      load_prev(it + 2, pa[(it + 2) % 3], pb[(it + 2) % 3]);
      load_sym(it + 2, sq[(it + 2) % 3]);
    }
    const int i = 8 * rq + it;
    const uint32_t zlu = __shfl_sync(FULL, zLu, i), zlv = __shfl_sync(FULL, zLv, i);
    uint32_t au[4], av[4];
#pragma unroll
    for (int k = 0; k < 4; k++) amp(sq[it % 3][k], au[k], av[k]);
    row_scan(au);
    row_scan(av);
    const int4 p01 = pa[it % 3], p23 = pb[it % 3];
    const uint32_t pu[4] = {(uint32_t)p01.x, (uint32_t)p01.z, (uint32_t)p23.x, (uint32_t)p23.z};
    const uint32_t pw[4] = {(uint32_t)p01.y, (uint32_t)p01.w, (uint32_t)p23.y, (uint32_t)p23.w};
    int32_t ru[4], rv[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      ou[k] += au[k];   // column sums run down the band
      ov[k] += av[k];
      ru[k] = (int32_t)(ou[k] + zlu + pu[k]);
      rv[k] = (int32_t)(ov[k] + zlv + pw[k]);
    }
    int4* rp = recp + (int64_t)it * (Wp / 2);
    rp[0] = make_int4(ru[0], rv[0], ru[1], rv[1]);
    rp[1] = make_int4(ru[2], rv[2], ru[3], rv[3]);
    double2* du = fu + (int64_t)it * (W / 2);
    double2* dv = fv + (int64_t)it * (W / 2);
    du[0] = make_double2(__dmul_rn((double)ru[0], inv_S), __dmul_rn((double)ru[1], inv_S));
    du[1] = make_double2(__dmul_rn((double)ru[2], inv_S), __dmul_rn((double)ru[3], inv_S));
    dv[0] = make_double2(__dmul_rn((double)rv[0], inv_S), __dmul_rn((double)rv[1], inv_S));
    dv[1] = make_double2(__dmul_rn((double)rv[2], inv_S), __dmul_rn((double)rv[3], inv_S));
  }
}

template <int C>
__device__ __forceinline__ void bs_final_dec1(const BScanIO& io, int bi, int bj,
                                              int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, io.H - r0), ncl = min(32, io.W - c0);
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t blk = (int64_t)bi * io.nbx + bj;
  const int Wp = io.Wp, W = io.W;
  const int kind = __ldcg(io.cls + C * nblk + blk) & 3;
  if (kind == BS_KNOWN) return;
  const bool reg = kind == BS_REG;
  const bool colok = lane < ncl;
  const int j = c0 + (colok ? lane : ncl - 1);
  const int32_t* eb = io.ebot + C * nblk * 32;
  const int32_t* er = io.eright + C * nblk * 32;
  int32_t zU = (bi > 0 && colok) ? __ldcg(eb + (blk - io.nbx) * 32 + lane) : 0;
  const int32_t zL = (bj > 0 && lane < nr) ? __ldcg(er + (blk - 1) * 32 + lane) : 0;
  int32_t zLp = (bi > 0 && bj > 0) ? __ldcg(eb + (blk - io.nbx - 1) * 32 + 31) : 0;
  int64_t qb = 0;
  if (reg && lane < nr)
    qb = io.qd_row_off[r0 + lane] +
         2 * (int64_t)io.pre_nl[(int64_t)(r0 + lane) * io.nchunks + bj] + C;
  const int32_t* pvc = io.prevrec ? reinterpret_cast<const int32_t*>(io.prevrec) + C : nullptr;
  int32_t* recw = reinterpret_cast<int32_t*>(io.rec) + C;
  double* f64 = io.f64[C];
  int64_t* fix = io.fix[C];
  uint32_t bz[4];
  int bcd[4] = {0, 0, 0, 0};
  int32_t bpp[4];
  auto issue = [&](int i, int sl) {
    const int ic = min(i, nr - 1);
    const int64_t qr = __shfl_sync(FULL, qb, ic);
    if (i < nr) {
      const int64_t pk = (int64_t)(r0 + i) * Wp + j;
      if (reg) {
        bz[sl] = colok ? (uint32_t)__ldg(io.qd + qr + 2 * lane) : 0u;
        bcd[sl] = __ldg(io.codes + (int64_t)(r0 + i) * io.cpitch + j);
      } else {
        bz[sl] = colok ? (uint32_t)__ldcg(io.out[C] + pk) : 0u;
      }
      bpp[sl] = pvc ? __ldg(pvc + 2 * pk) : 0;
    }
  };
  issue(0, 0);
  issue(1, 1);
  issue(2, 2);
  for (int i0 = 0; i0 < nr; i0 += 4)
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    const int i = i0 + kk;
    if (i >= nr) break;
    issue(i + 3, (kk + 3) & 3);
    int32_t z;
    const int32_t zl = __shfl_sync(FULL, zL, i);
    if (reg) {
      const uint32_t e2 = 2u * (uint32_t)io.e_tab[bcd[kk] & 31];
      uint32_t acc = colok ? (uint32_t)((int32_t)bz[kk] - io.radius) * e2 : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, acc, o);
        if (lane >= o) acc += y;
      }
      z = (int32_t)((uint32_t)zU + (uint32_t)zl - (uint32_t)zLp + acc);
    } else {
      z = (int32_t)bz[kk];
    }
    zU = z;
    zLp = zl;
    if (colok) {
      const int64_t pk = (int64_t)(r0 + i) * Wp + j;
      const int32_t r = (int32_t)((uint32_t)z + (uint32_t)bpp[kk]);
      const int64_t ko = (int64_t)(r0 + i) * W + j;
      recw[2 * pk] = r;
      f64[ko] = __dmul_rn((double)r, io.inv_S);
      if (fix) fix[ko] = r;
    }
  }
}

// Phase C as its own kernel, launched as a programmatic dependent of the
// chain kernel so that it runs beside it: a warp takes a ticket of four
// blocks of one block row and waits until the chain has marked the segment
// (32 blocks) in that row and in the row above, both components.  Tickets
// follow the chain's front: the frame in cells of 32 block rows x one
// segment, cells by anti-diagonals (a band of rows starts about one segment
// time after the band above).
template <bool ENC, typename F = float>
__global__ void __launch_bounds__(256, 2)
bs_interior_kernel(const __grid_constant__ BScanIO io) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int nbx = io.nbx, nby = io.nby;
  const int64_t nblk = (int64_t)nbx * nby;
  const int nseg = (nbx + BS_SEG - 1) / BS_SEG, nband = (nby + 31) / 32;
  // blocks per ticket: four on a large frame, one where the frame has few
  // blocks per warp (a warp walks its ticket's blocks one after another)
  const int tb = nblk >= 16384 ? 4 : 1, ngrp = BS_SEG / tb, percell = 32 * ngrp;
  const int ntick = nseg * nband * percell;
  for (;;) {
    int tk = 0;
    if (lane == 0) tk = atomicAdd(io.ticket + 1, 1);
    tk = __shfl_sync(FULL, tk, 0);
    if (tk >= ntick) break;
    const int cell = tk / percell, incell = tk - cell * percell;
    int rem = cell, d = 0, kmin = 0;
    for (;;) {
      kmin = max(0, d - (nseg - 1));
      const int cnt = min(d, nband - 1) - kmin + 1;
      if (rem < cnt) break;
      rem -= cnt;
      d++;
    }
    const int band = kmin + rem, seg = d - band;
    const int bi = 32 * band + incell / ngrp;
    const int bj0 = BS_SEG * seg + tb * (incell % ngrp);
    if (bi >= nby || bj0 >= nbx) continue;
    if (lane < 4) {
      const int comp = lane & 1, r = bi - (lane >> 1);
      if (r >= 0) {
        const unsigned long long need =
            ((unsigned long long)io.frame_tag << 32) | (unsigned)min(nbx, BS_SEG * (seg + 1));
        const unsigned long long* pg = io.prog + (int64_t)comp * nby + r;
        long long spins = 0;
        while (ld_acquire_gpu_u64(pg) < need) {
          __nanosleep(256);
          if (++spins > (1ll << 26)) __trap();   // never: a hang guard
        }
      }
    }
    __syncwarp();
    for (int bj = bj0; bj < min(nbx, bj0 + tb); bj++) {
      const int64_t blk = (int64_t)bi * nbx + bj;
      if (ENC) {
        bs_final_enc<F>(io, bi, bj, lane);
      } else {
        const int32_t cu = __ldcg(io.cls + blk), cv = __ldcg(io.cls + nblk + blk);
        const int32_t want = BS_REG | BS_NARROW;
        if (io.vec4 && (cu & (3 | BS_NARROW)) == want && (cv & (3 | BS_NARROW)) == want) {
          bs_final_dec4(io, bi, bj, lane, (cu >> 2) & 31);
        } else {
          bs_final_dec1<0>(io, bi, bj, lane);
          bs_final_dec1<1>(io, bi, bj, lane);
        }
      }
    }
  }
}

template <bool ENC, typename F = float>
cudaError_t launch_bs_chain(const BScanIO& io, int nsm, cudaStream_t st) {
  const size_t smem = sizeof(BSChainSmem);
  static OncePerDevice occ_once;
  int occ = 1;
  cudaError_t e = occ_once.get(
      [&](int* o) {
        cudaError_t r = cudaFuncSetAttribute(
            bs_chain_kernel<ENC, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
            (int)smem);
        if (r != cudaSuccess) return r;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            o, bs_chain_kernel<ENC, F>, 32 * BS_NW, smem);
      },
      &occ);
  if (e != cudaSuccess) return e;
  // persistent: every CTA is resident; tickets hand out the chain tasks in
  // block-row order (a task waits only for tasks with smaller tickets)
  bs_chain_kernel<ENC, F><<<min(max(occ, 1) * nsm, bs_ntask(io.nby)), 32 * BS_NW, smem, st>>>(io);
  e = cudaGetLastError();
  if (e != cudaSuccess || io.dbg_skip_interior) return e;
  static OncePerDevice occ2_once;
  int occ2 = 1;
  e = occ2_once.get(
      [&](int* o) {
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            o, bs_interior_kernel<ENC, F>, 256, 0);
      },
      &occ2);
  if (e != cudaSuccess) return e;
  const int nseg = (io.nbx + BS_SEG - 1) / BS_SEG, nband = (io.nby + 31) / 32;
  const int64_t nblk = (int64_t)io.nbx * io.nby;
  const int64_t want = (int64_t)nseg * nband * (nblk >= 16384 ? 32 : 128),
                cap = (int64_t)max(occ2, 1) * nsm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(want < cap ? want : cap));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, bs_interior_kernel<ENC, F>, io);
}

}  // namespace vfcp
