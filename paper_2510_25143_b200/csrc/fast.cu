// Frame-parallel preparation kernels around the block-scan chain
// (bscan.cuh).
//
// Per frame t the compress path runs
//   enc_r0_kernel    R0 = orig - Lorenzo(orig, prev), the frame t-1
//                    reconstruction as (u, v) pairs, the padded codes copy;
//   enc_mop_kernel   (t >= 1, MoP) the per-block mode decision;
//   enc_pix_kernel   lossless pins, semi-Lagrangian pixels (prediction,
//                    symbol, pinned err), per-chunk bit words;
//   launch_bscan<ENC>  the raster recurrence, the Lorenzo symbols into the
//                    stream;
// and the decompress path
//   dec_prep_kernel  pins (lossless, escapes, semi-Lagrangian pixels) and
//                    A = Pd + (sym-radius)*2e;
//   the block scan (bscan.cuh), whose interior pass also writes the
//   float64 output.
// The reconstruction of frame t-1 is read as orig + err (encoder) or the int
// recon frame (decoder).  Stream positions come from per-(row, chunk) prefix
// counts, so any block can place its symbols and ll values.
#include "bscan.cuh"

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

// ------------------------------------------------------ 2D value sources
// The frame t-1 reconstruction (fixed point) as (u, v) pairs: the encoder
// writes it interleaved while preparing frame t (one 8-byte gather per
// bilinear tap); the decoder reads its two recon planes.
struct PairPlane {
  const int2* p;  // pitch Wp
  int Wp;
  __device__ __forceinline__ void get(int i, int j, double& u, double& v) const {
    const int2 x = __ldg(p + (int64_t)i * Wp + j);
    u = (double)x.x;
    v = (double)x.y;
  }
};
struct TwoPlanes {
  const int32_t* u;
  const int32_t* v;
  int Wp;
  __device__ __forceinline__ void get(int i, int j, double& a, double& b) const {
    const int64_t k = (int64_t)i * Wp + j;
    a = (double)__ldg(u + k);
    b = (double)__ldg(v + k);
  }
};

// predictors.py:33-59 (shared weights for u and v)
template <typename Src>
__device__ __forceinline__ void bilinear2(const Src& s, int H, int W,
                                          double i_f, double j_f,
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
  double u00, v00, u01, v01, u10, v10, u11, v11;
  s.get(i0, j0, u00, v00);
  s.get(i0, j1, u01, v01);
  s.get(i1, j0, u10, v10);
  s.get(i1, j1, u11, v11);
  const double a = __dsub_rn(i_f, (double)i0), b = __dsub_rn(j_f, (double)j0);
  const double oma = __dsub_rn(1.0, a), omb = __dsub_rn(1.0, b);
  const double w00 = __dmul_rn(oma, omb), w01 = __dmul_rn(oma, b);
  const double w10 = __dmul_rn(a, omb), w11 = __dmul_rn(a, b);
  double vu = __dmul_rn(w00, u00);
  vu = __dadd_rn(vu, __dmul_rn(w01, u01));
  vu = __dadd_rn(vu, __dmul_rn(w10, u10));
  vu = __dadd_rn(vu, __dmul_rn(w11, u11));
  double vv = __dmul_rn(w00, v00);
  vv = __dadd_rn(vv, __dmul_rn(w01, v01));
  vv = __dadd_rn(vv, __dmul_rn(w10, v10));
  vv = __dadd_rn(vv, __dmul_rn(w11, v11));
  *pu = rha_d(vu);
  *pv = rha_d(vv);
}

// predictors.py:76-108 + the prediction sample at the departure point
template <typename Src>
__device__ __forceinline__ void sl_predict2(const Src& s, int H, int W, int i,
                                            int j, double cfl_x, double cfl_y,
                                            double d_max, int n_max,
                                            int64_t* pu, int64_t* pv) {
  double u0, v0;
  s.get(i, j, u0, v0);
  const double ax = __dmul_rn(fabs(u0), cfl_x), ay = __dmul_rn(fabs(v0), cfl_y);
  const double d_inf = ay > ax ? ay : ax;
  double fi, fj;
  if (d_inf <= d_max) {
    const double ih = __dsub_rn((double)i, __dmul_rn(__dmul_rn(0.5, v0), cfl_y));
    const double jh = __dsub_rn((double)j, __dmul_rn(__dmul_rn(0.5, u0), cfl_x));
    int64_t um, vm;
    bilinear2(s, H, W, ih, jh, &um, &vm);
    fi = __dsub_rn((double)i, __dmul_rn((double)vm, cfl_y));
    fj = __dsub_rn((double)j, __dmul_rn((double)um, cfl_x));
  } else {
    int64_t n = (int64_t)ceil(__ddiv_rn(d_inf, d_max));
    if (n > n_max) n = n_max;
    const double dn = (double)n;
    fi = (double)i;
    fj = (double)j;
    for (int64_t k = 0; k < n; k++) {
      int64_t us, vs;
      bilinear2(s, H, W, fi, fj, &us, &vs);
      fi = __dsub_rn(fi, __ddiv_rn(__dmul_rn((double)vs, cfl_y), dn));
      fj = __dsub_rn(fj, __ddiv_rn(__dmul_rn((double)us, cfl_x), dn));
      if (fi < 0.0) fi = 0.0;
      else if (fi > (double)(H - 1)) fi = (double)(H - 1);
      if (fj < 0.0) fj = 0.0;
      else if (fj > (double)(W - 1)) fj = (double)(W - 1);
    }
  }
  bilinear2(s, H, W, fi, fj, pu, pv);
}

// The RK2 branch of sl_predict2 only (d_inf <= d_max), branch-free so a
// batch of samples overlaps its gathers; returns false (outputs unset) when
// the sample needs the Euler-substep branch.
template <typename Src>
__device__ __forceinline__ bool sl_predict_rk2(const Src& s, int H, int W,
                                               int i, int j, double cfl_x,
                                               double cfl_y, double d_max,
                                               int64_t* pu, int64_t* pv) {
  double u0, v0;
  s.get(i, j, u0, v0);
  const double ax = __dmul_rn(fabs(u0), cfl_x), ay = __dmul_rn(fabs(v0), cfl_y);
  const double d_inf = ay > ax ? ay : ax;
  const double ih = __dsub_rn((double)i, __dmul_rn(__dmul_rn(0.5, v0), cfl_y));
  const double jh = __dsub_rn((double)j, __dmul_rn(__dmul_rn(0.5, u0), cfl_x));
  int64_t um, vm;
  bilinear2(s, H, W, ih, jh, &um, &vm);
  const double fi = __dsub_rn((double)i, __dmul_rn((double)vm, cfl_y));
  const double fj = __dsub_rn((double)j, __dmul_rn((double)um, cfl_x));
  bilinear2(s, H, W, fi, fj, pu, pv);
  return d_inf <= d_max;
}

// ------------------------------------------------ first-touch block entropy
// mop.py:118-138.  samp[sp] = |idx| of sample sp (sequence order: raster
// (i, j), u then v) or -1 for an overflow sample.  The reference sums
// h*log2(h) over the distinct values in first-touch order (float64, so the
// order is part of the result).  One warp, 32 samples per step in sequence
// order: __match_any_sync groups equal values, the group leader (its first
// occurrence) adds the group's count, and a value's first touch appends it
// to an ordered list; values >= ETB take the generic path.
constexpr int ETB = 512;
__device__ double block_rate(const int16_t* samp, int ns, int16_t* cnt,
                             int16_t* order, const double* log2tab,
                             double lam, double rmeta, int lane) {
  const unsigned FULL = 0xffffffffu;
  const unsigned below = (1u << lane) - 1u;
  int n_ok = 0, lp = 0, nd = 0;
  for (int c = 0; c < ns; c += 32) {
    const int sp = c + lane;
    const int a = sp < ns ? samp[sp] : -2;
    n_ok += a >= 0;
    lp += a == -1;
    const bool small = a >= 0 && a < ETB;
    const int key = small ? a : -1;
    const unsigned grp = __match_any_sync(FULL, key);
    const bool leader = small && (grp & below) == 0;
    int prev = 0;
    if (leader) prev = cnt[key];
    bool fresh = leader && prev == 0;
    if (a >= ETB) {   // rare: first touch by search
      fresh = true;
      for (int q = 0; q < sp; q++)
        if (samp[q] == a) { fresh = false; break; }
    }
    const unsigned fm = __ballot_sync(FULL, fresh);
    if (leader) cnt[key] = (int16_t)(prev + __popc(grp));
    if (fresh) order[nd + __popc(fm & below)] = (int16_t)(small ? key : -(sp + 1));
    nd += __popc(fm);
  }
  for (int o = 16; o; o >>= 1) {
    n_ok += __shfl_xor_sync(FULL, n_ok, o);
    lp += __shfl_xor_sync(FULL, lp, o);
  }
  __syncwarp();
  double acc = 0.0;
  for (int k0 = 0; k0 < nd; k0 += 32) {
    const int k = k0 + lane;
    double term = 0.0;
    if (k < nd) {
      const int key = order[k];
      int h = 0;
      if (key >= 0) {
        h = cnt[key];
      } else {
        const int a = samp[-key - 1];
        for (int q = 0; q < ns; q++) h += samp[q] == a;
      }
      term = __dmul_rn((double)h, log2tab[h]);
    }
    const int nk = min(32, nd - k0);
    for (int b = 0; b < nk; b++) acc = __dadd_rn(acc, __shfl_sync(FULL, term, b));
  }
  __syncwarp();
  for (int k = lane; k < nd; k += 32)
    if (order[k] >= 0) cnt[order[k]] = 0;
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
// Three frame-parallel kernels per frame t:
//   enc_r0_kernel   CTA per 32x32 block (tile + one-pixel halo in shared
//                   memory): R0 = orig - Lorenzo(orig, prev) (zero padding
//                   outside the frame), the frame t-1 reconstruction as
//                   (u, v) pairs, the padded codes copy, the int32 overflow
//                   flag, and phase A of the block scan (bscan.cuh): the
//                   block class and the edge sums LB / LR of -R0 mod 2e;
//   enc_mop_kernel  CTA per 32x32 block (frames t >= 1 with MoP): the mode
//                   decision of mop.py:79-151;
//   enc_pix_kernel  warp per (row, chunk): lossless pins, semi-Lagrangian
//                   pixels (prediction, symbol, pinned err), the per-chunk
//                   non-lossless / pinned bit words, the per-row ll counts
//                   and the known edges of semi-Lagrangian blocks.
//
template <typename F>
__global__ void __launch_bounds__(256)
enc_r0_kernel(const F* __restrict__ u, const F* __restrict__ v,
              const uint8_t* __restrict__ codes,
              const int32_t* __restrict__ err_prev_u,
              const int32_t* __restrict__ err_prev_v, PrepParams p,
              BScanIO bio,
              int32_t* __restrict__ a0, int32_t* __restrict__ a1,
              int2* __restrict__ prevrec, uint8_t* __restrict__ codes_p,
              int* __restrict__ overflow) {
  // one 32x32 tile per CTA; every input value is converted to fixed point
  // once, into shared memory with a one-pixel halo above and to the left
  __shared__ int32_t so[2][33][33];   // orig(t)
  __shared__ int32_t sp[2][33][33];   // recon(t-1) = orig(t-1) + err(t-1)
  __shared__ uint32_t sx[2][32][33];  // phase A: -R0 mod 2e
  __shared__ int sflag[3];            // non-uniform / possible escape (u, v); lossy
  const int H = p.H, W = p.W, Wp = p.Wp;
  const int c0 = 32 * blockIdx.x, r0 = 32 * blockIdx.y;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t HW = (int64_t)H * W;
  const F* uo = u + (int64_t)p.t * HW;
  const F* vo = v + (int64_t)p.t * HW;
  const bool has_prev = p.t > 0;
  const F* up_ = u + (int64_t)(p.t - 1) * HW;
  const F* vp_ = v + (int64_t)(p.t - 1) * HW;
  // all loads of the thread first (5 x 6 in flight), then the conversions
  constexpr int NK = (33 * 33 + 255) / 256;
  F xo_u[NK], xo_v[NK], xp_u[NK], xp_v[NK];
  int32_t xe_u[NK], xe_v[NK];
  bool okk[NK];
#pragma unroll
  for (int q = 0; q < NK; q++) {
    const int k = tid + 256 * q;
    const int rr = k / 33, cc = k - rr * 33;
    const int i = r0 - 1 + rr, j = c0 - 1 + cc;
    const bool ok = k < 33 * 33 && i >= 0 && j >= 0 && i < H && j < W;
    okk[q] = ok;
    const int64_t n = ok ? (int64_t)i * W + j : 0;
    const int64_t m = ok ? (int64_t)i * Wp + j : 0;
    xo_u[q] = ok ? __ldg(uo + n) : F(0);
    xo_v[q] = ok ? __ldg(vo + n) : F(0);
    const bool okp = ok && has_prev;
    xp_u[q] = okp ? __ldg(up_ + n) : F(0);
    xp_v[q] = okp ? __ldg(vp_ + n) : F(0);
    xe_u[q] = okp ? __ldg(err_prev_u + m) : 0;
    xe_v[q] = okp ? __ldg(err_prev_v + m) : 0;
  }
#pragma unroll
  for (int q = 0; q < NK; q++) {
    const int k = tid + 256 * q;
    if (k >= 33 * 33) break;
    const int rr = k / 33, cc = k - rr * 33;
    const bool ok = okk[q];
    so[0][rr][cc] = ok ? fixed_t(xo_u[q], p.S) : 0;
    so[1][rr][cc] = ok ? fixed_t(xo_v[q], p.S) : 0;
    sp[0][rr][cc] = (ok && has_prev) ? fixed_t(xp_u[q], p.S) + xe_u[q] : 0;
    sp[1][rr][cc] = (ok && has_prev) ? fixed_t(xp_v[q], p.S) + xe_v[q] : 0;
  }
  const uint8_t* cf = codes + (int64_t)p.t * HW;
  const int code0 = cf[(int64_t)r0 * W + c0];
  const int32_t e0 = (int32_t)p.lad.e[code0 & 31];
  const uint32_t m = e0 > 0 ? 2u * (uint32_t)e0 : 2u;
  const uint32_t M = (uint32_t)((((uint64_t)1) << 32) / m);
  int64_t lim = (2 * (int64_t)p.radius - 4) * (int64_t)e0;
  if (lim > (int64_t)1 << 30) lim = (int64_t)1 << 30;   // int32 symbols in phase C
  if (tid < 3) sflag[tid] = 0;
  __syncthreads();
  bool ovf = false, bad_u = false, bad_v = false, lossy = false;
  const int j = c0 + tx;
  const bool colok = j < W;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int rr = ty + 8 * q;
    const int i = r0 + rr;
    if (i >= H) break;
    const int64_t R_u = (int64_t)so[0][rr + 1][tx + 1] -
                        ((int64_t)so[0][rr][tx + 1] + so[0][rr + 1][tx] - so[0][rr][tx]) -
                        ((int64_t)sp[0][rr + 1][tx + 1] - sp[0][rr][tx + 1] -
                         sp[0][rr + 1][tx] + sp[0][rr][tx]);
    const int64_t R_v = (int64_t)so[1][rr + 1][tx + 1] -
                        ((int64_t)so[1][rr][tx + 1] + so[1][rr + 1][tx] - so[1][rr][tx]) -
                        ((int64_t)sp[1][rr + 1][tx + 1] - sp[1][rr][tx + 1] -
                         sp[1][rr + 1][tx] + sp[1][rr][tx]);
    const bool o = colok && (R_u >= 2147483647LL || R_u <= -2147483647LL ||
                             R_v >= 2147483647LL || R_v <= -2147483647LL);
    ovf |= o;
    const int64_t pr = (int64_t)i * Wp + j;
    const int cd = colok ? cf[(int64_t)i * W + j] : CODE_LOSSLESS;
    a0[pr] = colok ? (int32_t)R_u : 0;
    a1[pr] = colok ? (int32_t)R_v : 0;
    // phase A of the block scan (bscan.cuh)
    if (colok) {
      lossy |= (p.lossy_mask >> (cd & 31)) & 1u;
      bad_u |= cd != code0 || (R_u < 0 ? -R_u : R_u) >= lim;
      bad_v |= cd != code0 || (R_v < 0 ? -R_v : R_v) >= lim;
    }
    sx[0][rr][tx] = colok ? bs_negres((int32_t)R_u, m, M) : 0u;
    sx[1][rr][tx] = colok ? bs_negres((int32_t)R_v, m, M) : 0u;
    if (has_prev) prevrec[pr] = make_int2(sp[0][rr + 1][tx + 1], sp[1][rr + 1][tx + 1]);
    codes_p[pr] = (uint8_t)cd;
  }
  for (int q = H - r0; q < 32; q++)   // rows past the frame
    if (ty == 0) { sx[0][q][tx] = 0u; sx[1][q][tx] = 0u; }
  if (ovf) atomicOr(overflow, 1);
  if (bad_u) sflag[0] = 1;
  if (bad_v) sflag[1] = 1;
  if (lossy) sflag[2] = 1;
  __syncthreads();
  if (tid >= 64) return;
  // warp = component: LB(j) = prefix over columns of the column sums,
  // LR(i) = prefix over rows of the row sums (mod 2e)
  const int comp = tid >> 5, lane = tid & 31;
  const bool lossless = sflag[2] == 0;
  const bool reg = e0 > 0 && lim > 0 && sflag[comp] == 0;
  uint32_t cs = 0, rs = 0;
#pragma unroll 8
  for (int k = 0; k < 32; k++) {
    cs = bs_madd(cs, sx[comp][k][lane], m);
    rs = bs_madd(rs, sx[comp][lane][k], m);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t pc = __shfl_up_sync(0xffffffffu, cs, o);
    const uint32_t pr = __shfl_up_sync(0xffffffffu, rs, o);
    if (lane >= o) {
      cs = bs_madd(cs, pc, m);
      rs = bs_madd(rs, pr, m);
    }
  }
  const int64_t nblk = (int64_t)p.nbx * p.nby;
  const int64_t blk = (int64_t)blockIdx.y * p.nbx + blockIdx.x;
  // all lossless: every value is known (0); otherwise regular or swept.
  // Semi-Lagrangian blocks are reclassified as known by enc_pix.
  bio.lb[(comp * nblk + blk) * 32 + lane] = lossless ? 0 : (int32_t)cs;
  bio.lr[(comp * nblk + blk) * 32 + lane] = lossless ? 0 : (int32_t)rs;
  if (lane == 0)
    bio.cls[comp * nblk + blk] =
        lossless ? BS_KNOWN : (reg ? (BS_REG | (code0 << 2)) : BS_SLOW);
}

// MoP trial step with one step size e for the whole block (mop.py:88-110):
// the neighbours' trial errors lie in [-e, e], so y = rho - d is within
// [-4e, 4e] and q = q0 + g follows from comparisons of y with +-e, +-3e
__device__ __forceinline__ int32_t trial_step(int32_t rho, int32_t q0,
                                              int32_t e, int32_t d,
                                              int32_t radius, int32_t* qabs) {
  const int32_t y = rho - d;
  const int32_t e3 = 3 * e;
  const int32_t gf = (y >= e) + (y >= e3) - (y < -e) - (y < -e3);
  const int32_t ay = y < 0 ? -y : y;
  const bool tie = (ay == e) | (ay == e3);
  const int32_t qf = q0 + gf;
  const int32_t q = qf - ((tie && qf <= 0) ? 1 : 0);
  const bool esc = (uint32_t)(q + radius - 1) >= (uint32_t)(2 * radius - 1);
  *qabs = esc ? -1 : (q < 0 ? -q : q);
  return esc ? 0 : (q - q0) * 2 * e - y;
}

// One CTA of 4 warps per 32x32 block: warps 0 / 1 run the Lorenzo trial of
// u / v, then all four warps the semi-Lagrangian trial at the stride samples
// (warps 2 / 3 start on it at once); then warp 0 rates the Lorenzo samples
// while warp 2 rates the SL samples (first-touch order, mop.py:118-138).
struct MopSmem {
  int32_t r0[2][32][33];   // [comp][row][col] R0 tile, then rho
  int32_t q0[2][32][33];   // [comp][row][col] Q0 = rha(R0 / 2 tau')
  // int16: |idx| < radius <= 2^15, counts and positions <= 512
  int16_t samp[2][512];    // [trial] |idx| per sample (-1: escape)
  int16_t order[2][ETB];   // distinct |idx| in first-touch order
  int16_t cnt[2][ETB];
  double rate[2];
};

template <typename F>
__global__ void __launch_bounds__(128, 8)
enc_mop_kernel(const F* __restrict__ u, const F* __restrict__ v,
               const int32_t* __restrict__ a0, const int32_t* __restrict__ a1,
               const int2* __restrict__ prevrec, PrepParams p,
               const double* __restrict__ log2tab,
               uint8_t* __restrict__ modes_t) {
  __shared__ MopSmem sm;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int bi = blockIdx.y, bj = blockIdx.x;
  const int blk = bi * p.nbx + bj;
  const int H = p.H, W = p.W, Wp = p.Wp;
  const int r0 = 32 * bi, c0 = 32 * bj;
  const int nr = min(32, H - r0), ncl = min(32, W - c0);
  const unsigned FULL = 0xffffffffu;
  const int nsx = (ncl + p.stride - 1) / p.stride;
  const int nsy = (nr + p.stride - 1) / p.stride;
  const int nsamp = nsx * nsy;
  const int ns = 2 * nsamp;
  const int32_t e = (int32_t)p.tau;     // fast path: tau' < 2^28
  const double inv = 1.0 / (double)(2 * p.tau);
  const int32_t radius = p.radius;
  const int64_t tau = p.tau;
  for (int k = threadIdx.x; k < 2 * ETB; k += 128) (&sm.cnt[0][0])[k] = 0;
  const int64_t HW = (int64_t)H * W;
  const F* uo = u + (int64_t)p.t * HW;
  const F* vo = v + (int64_t)p.t * HW;
  // semi-Lagrangian samples of this thread: sidx = tid and tid + 128; the
  // originals are loaded first (warps 2 / 3 start on their gathers at once,
  // warps 0 / 1 after the Lorenzo trial)
  constexpr int NSB = 2;
  F sou[NSB], sov[NSB];
#pragma unroll
  for (int b = 0; b < NSB; b++) {
    const int sidx = min((int)threadIdx.x + 128 * b, nsamp - 1);
    const int si = sidx / nsx, sj = sidx - si * nsx;
    const int64_t k = (int64_t)(r0 + si * p.stride) * W + c0 + sj * p.stride;
    sou[b] = __ldg(uo + k);
    sov[b] = __ldg(vo + k);
  }
  bool swept = false;
  if (wid < 2) {
    // Lorenzo trial of component wid with block-local errors (mop.py:88-110).
    // Every pixel uses the step tau', so unless a pixel can escape
    // (|R0| >= (2 radius - 4) tau') the trial errors are the representatives
    // of the block's 2D prefix sums of -R0 mod 2 tau' (see bscan.cuh), with
    // a zero boundary (outside the block the candidate is the original).
    // (|R0| < 2^30 as well: the sample arithmetic below is then exact in
    // int32.)  The R0 tile (lane = column) goes to shared memory together
    // with its residues.
    const int comp = wid;
    const int32_t* ap = wid ? a1 : a0;
    int64_t lim64 = (2 * (int64_t)radius - 4) * tau;
    if (lim64 > ((int64_t)1 << 30)) lim64 = (int64_t)1 << 30;
    const int32_t lim = (int32_t)(lim64 > 0 ? lim64 : 0);
    const uint32_t m = 2u * (uint32_t)e, ue = (uint32_t)e;
    const uint32_t M = (uint32_t)((((uint64_t)1) << 32) / m);
    int32_t(*v)[33] = sm.q0[comp];
    int32_t(*x)[33] = sm.r0[comp];
    bool safe = lim > 0;
#pragma unroll 8
    for (int r = 0; r < 32; r++) {
      const int32_t x0 = r < nr ? __ldg(ap + (int64_t)(r0 + r) * Wp + c0 + lane) : 0;
      x[r][lane] = x0;
      v[r][lane] = (int32_t)bs_negres(x0, m, M);
      safe &= (x0 < 0 ? -x0 : x0) < lim;   // |R0| < 2^31 - 1 (enc_r0)
    }
    swept = !__all_sync(FULL, safe);
    __syncwarp();
    if (!swept) {
      uint32_t acc = 0;
#pragma unroll 8
      for (int k = 0; k < 32; k++) {   // row prefix, lane = row
        acc = bs_madd(acc, (uint32_t)v[lane][k], m);
        v[lane][k] = (int32_t)acc;
      }
      __syncwarp();
      acc = 0;
#pragma unroll 8
      for (int k = 0; k < 32; k++) {   // column prefix, lane = column
        acc = bs_madd(acc, (uint32_t)v[k][lane], m);
        v[k][lane] = (int32_t)acc;
      }
      uint32_t tierows = 0;
#pragma unroll
      for (int r = 0; r < 32; r++) {
        const uint32_t sres = (uint32_t)v[r][lane];
        const bool tie = sres == ue && r < nr && lane < ncl;
        tierows |= (__any_sync(FULL, tie) ? 1u : 0u) << r;
        v[r][lane] = tie ? INT32_MIN : bs_rep(sres, ue, m);
      }
      __syncwarp();
      if (tierows) {
        // raster order: the tie's sign follows x = R0 - D, whose neighbours
        // may be earlier ties
#pragma unroll 1
        for (int r = 0; r < 32; r++) {
          if (!((tierows >> r) & 1u)) continue;   // warp-uniform
          uint32_t tm = __ballot_sync(FULL, lane < ncl && v[r][lane] == INT32_MIN);
          while (tm) {
            const int j = __ffs(tm) - 1;
            tm &= tm - 1u;
            if (lane == j) {
              const int64_t d = (r > 0 ? (int64_t)v[r - 1][j] : 0) +
                                (j > 0 ? (int64_t)v[r][j - 1] : 0) -
                                ((r > 0 && j > 0) ? (int64_t)v[r - 1][j - 1] : 0);
              v[r][j] = ((int64_t)x[r][j] - d) > 0 ? e : -e;
            }
            __syncwarp();
          }
        }
      }
      __syncwarp();
      // |idx| at the stride samples: x + err = q * 2 tau' exactly
      auto sample = [&](int r, int j) {
        const int32_t d = (r > 0 ? v[r - 1][j] : 0) + (j > 0 ? v[r][j - 1] : 0) -
                          ((r > 0 && j > 0) ? v[r - 1][j - 1] : 0);
        const int32_t n = x[r][j] - d + v[r][j];
        const uint32_t an = (uint32_t)(n < 0 ? -n : n);
        uint32_t qa = __umulhi(an, M);
        if (qa * m != an) qa++;
        return (int32_t)qa;
      };
      if (p.stride == 2) {
        // lane = (sample column, row parity): two sample rows per step
        const int sj = lane & 15, j = 2 * sj, rp = lane >> 4;
#pragma unroll 2
        for (int r = 2 * rp; r < nr; r += 4)
          if (j < ncl) sm.samp[0][2 * ((r >> 1) * nsx + sj) + comp] = (int16_t)sample(r, j);
      } else {
        const bool scol = lane < ncl && (lane % p.stride) == 0;
        const int sj = lane / p.stride;
        int srow = 0;
#pragma unroll 1
        for (int r = 0; r < nr; r += p.stride, srow += nsx)
          if (scol) sm.samp[0][2 * (srow + sj) + comp] = (int16_t)sample(r, lane);
      }
    }
  }
  if (wid < 2 && swept) {
    // escapes possible: the exact sweep.  Split R0 = Q0*2e + rho for the
    // whole tile first (independent per pixel, lane = column), so the
    // sweep below is only the recurrence
    {
      const int comp = wid;
#pragma unroll 8
      for (int r = 0; r < 32; r++) {
        const int32_t x0 = sm.r0[comp][r][lane];
        const int32_t q0 = quant32(x0, e, inv);
        sm.q0[comp][r][lane] = q0;
        sm.r0[comp][r][lane] = x0 - q0 * 2 * e;
      }
      __syncwarp();
    }
    // Lorenzo trial of component wid, block-local errors (mop.py:88-110)
    const int comp = wid;
    const int i = lane;
    const bool rowok = i < nr;
    int32_t eL = 0, eUL = 0;
    // sample bookkeeping without divisions in the loop: row i is a sample
    // row iff i % stride == 0; the column phase advances with jj
    const bool srow = (i % p.stride) == 0;
    const int sbase = 2 * ((i / p.stride) * nsx) + comp;
    int jm = 0, jq = 0;   // jj % stride, jj / stride once jj >= 0
#pragma unroll 7
    for (int s = 0; s < 63; s++) {
      const int jj = s - lane;
      const bool act = rowok && jj >= 0 && jj < ncl;
      const int32_t rho = act ? sm.r0[comp][i][jj] : 0;
      const int32_t q0 = act ? sm.q0[comp][i][jj] : 0;
      const int32_t up = __shfl_up_sync(FULL, eL, 1);
      const int32_t eU = (lane == 0 || !act) ? 0 : up;
      const int32_t d = eU + (jj > 0 ? eL : 0) - ((jj > 0 && lane > 0) ? eUL : 0);
      int32_t qa;
      const int32_t er = trial_step(rho, q0, e, d, radius, &qa);
      eUL = eU;
      if (act) eL = er;
      if (act && srow && jm == 0) sm.samp[0][sbase + 2 * jq] = (int16_t)qa;
      if (jj >= 0) {
        if (++jm == p.stride) { jm = 0; jq++; }
      }
    }
  }
  {
    // semi-Lagrangian trial at the stride samples, all 128 threads, NSB
    // samples each in lockstep so their departure-point gathers overlap
    const PairPlane src{prevrec, Wp};
    int64_t pr_u[NSB], pr_v[NSB];
    int si_i[NSB], si_j[NSB];
    bool slow[NSB];
#pragma unroll
    for (int b = 0; b < NSB; b++) {
      const int sidx = min((int)threadIdx.x + 128 * b, nsamp - 1);
      const int si = sidx / nsx, sj = sidx - si * nsx;
      si_i[b] = r0 + si * p.stride;
      si_j[b] = c0 + sj * p.stride;
      slow[b] = !sl_predict_rk2(src, H, W, si_i[b], si_j[b], p.cfl_x, p.cfl_y,
                                p.d_max, &pr_u[b], &pr_v[b]);
    }
#pragma unroll
    for (int b = 0; b < NSB; b++) {
      const int sidx = threadIdx.x + 128 * b;
      if (sidx >= nsamp) continue;
      if (slow[b])
        sl_predict2(src, H, W, si_i[b], si_j[b], p.cfl_x, p.cfl_y, p.d_max,
                    p.n_max, &pr_u[b], &pr_v[b]);
      const int64_t ru = (int64_t)fixed_t(sou[b], p.S) - pr_u[b];
      const int64_t rv = (int64_t)fixed_t(sov[b], p.S) - pr_v[b];
      const int64_t qu = quant_rha(ru, tau, inv), qv = quant_rha(rv, tau, inv);
      sm.samp[1][2 * sidx] = (int16_t)((qu > -radius && qu < radius) ? (qu < 0 ? -qu : qu) : -1);
      sm.samp[1][2 * sidx + 1] = (int16_t)((qv > -radius && qv < radius) ? (qv < 0 ? -qv : qv) : -1);
    }
  }
  __syncthreads();
  if (wid == 0 || wid == 2) {
    const int tr = wid >> 1;
    const double r = block_rate(sm.samp[tr], ns, sm.cnt[tr], sm.order[tr],
                                log2tab, p.lam, p.rmeta, lane);
    if (lane == 0) sm.rate[tr] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double r_lor = sm.rate[0], r_sl = sm.rate[1];
    modes_t[blk] =
        (r_lor > 0.0 && __ddiv_rn(__dsub_rn(r_lor, r_sl), r_lor) > p.theta) ? 1 : 0;
  }
}

template <typename F>
__global__ void __launch_bounds__(256, 5)
enc_pix_kernel(const F* __restrict__ u, const F* __restrict__ v,
               const uint8_t* __restrict__ codes_p,
               const int2* __restrict__ prevrec,
               const int64_t* __restrict__ qd_row_off,
               const int32_t* __restrict__ pre_nl, PrepParams p,
               const uint8_t* __restrict__ modes_t, BScanIO bio,
               int32_t* __restrict__ a0,
               int32_t* __restrict__ a1, uint32_t* __restrict__ pin_u,
               uint32_t* __restrict__ pin_v, uint32_t* __restrict__ nlw,
               uint16_t* __restrict__ qd, int32_t* __restrict__ row_ll) {
  const int lane = threadIdx.x & 31;
  // grid (chunk groups of 8, row pairs): warp = two rows of one 32-column
  // chunk (both in the same block row), so the semi-Lagrangian departure
  // gathers of the two rows overlap
  constexpr int NRW = 2;
  const int bj = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (bj >= p.nchunks) return;
  const int H = p.H, W = p.W, Wp = p.Wp, nchunks = p.nchunks;
  const int ib = NRW * blockIdx.y;
  const int j = 32 * bj + lane;
  const bool colok = j < W;
  const int64_t HW = (int64_t)H * W;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  const int mode = p.mop ? modes_t[(ib >> 5) * p.nbx + bj] : p.force_sl;
  const F* uo = u + (int64_t)p.t * HW;
  const F* vo = v + (int64_t)p.t * HW;
  int cd[NRW];
  F fu[NRW], fv[NRW];
  int64_t spu[NRW], spv[NRW];
#pragma unroll
  for (int q = 0; q < NRW; q++) {
    const int i = min(ib + q, H - 1);
    cd[q] = codes_p[(int64_t)i * Wp + j];
    if (mode == 1) {   // originals first: in flight during the gathers
      fu[q] = colok ? __ldg(uo + (int64_t)i * W + j) : F(0);
      fv[q] = colok ? __ldg(vo + (int64_t)i * W + j) : F(0);
    }
  }
  if (mode == 1) {
    const PairPlane src{prevrec, Wp};
    bool slow[NRW];
    const int jc = min(j, W - 1);
#pragma unroll
    for (int q = 0; q < NRW; q++)
      slow[q] = !sl_predict_rk2(src, H, W, min(ib + q, H - 1), jc, p.cfl_x,
                                p.cfl_y, p.d_max, &spu[q], &spv[q]);
#pragma unroll
    for (int q = 0; q < NRW; q++)
      if (slow[q] && colok && ib + q < H)
        sl_predict2(src, H, W, ib + q, j, p.cfl_x, p.cfl_y, p.d_max, p.n_max,
                    &spu[q], &spv[q]);
  }
#pragma unroll
  for (int q = 0; q < NRW; q++) {
    const int i = ib + q;
    if (i >= H) break;   // warp-uniform
    const int64_t row = (int64_t)p.t * H + i;
    const int64_t pr = (int64_t)i * Wp + j;
    const int64_t e = p.lad.e[cd[q]];
    const bool nl = colok && e != 0;
    const unsigned bnl = __ballot_sync(FULL, nl);
    const bool sl = nl && mode == 1;
    int nll = (colok && !nl) ? 2 : 0;
    bool pu = !nl, pv = !nl;   // lossless pixels are pinned (err 0)
    int32_t vu = 0, vv = 0;
    if (sl) {
      const int64_t two_e = 2 * e;
      const double inv = p.lad.inv2e[cd[q]];
      const int64_t ou = fixed_t(fu[q], p.S), ov = fixed_t(fv[q], p.S);
      const int64_t qu = quant_rha(ou - spu[q], e, inv), qv = quant_rha(ov - spv[q], e, inv);
      const bool oku = qu > -p.radius && qu < p.radius;
      const bool okv = qv > -p.radius && qv < p.radius;
      vu = oku ? (int32_t)(spu[q] + qu * two_e - ou) : 0;
      vv = okv ? (int32_t)(spv[q] + qv * two_e - ov) : 0;
      a0[pr] = vu;
      a1[pr] = vv;
      const uint32_t syu = oku ? (uint32_t)(qu + p.radius) : 0u;
      const uint32_t syv = okv ? (uint32_t)(qv + p.radius) : 0u;
      const int64_t pos = qd_row_off[row] +
                          2 * ((int64_t)pre_nl[row * nchunks + bj] + __popc(bnl & lt));
      *reinterpret_cast<uint32_t*>(qd + pos) = syu | (syv << 16);
      pu = pv = true;
      nll = (oku ? 0 : 1) + (okv ? 0 : 1);
    } else if (colok && !nl) {
      a0[pr] = 0;
      a1[pr] = 0;
    }
    const unsigned b_pu = __ballot_sync(FULL, colok && pu);
    const unsigned b_pv = __ballot_sync(FULL, colok && pv);
    const int tot = __reduce_add_sync(FULL, nll);
    if (lane == 0) {
      const int64_t pb = (int64_t)i * nchunks + bj;
      pin_u[pb] = b_pu;
      pin_v[pb] = b_pv;
      nlw[pb] = bnl;
      if (tot) atomicAdd(row_ll + row, tot);
    }
    if (mode == 1) {
      // every pixel of a semi-Lagrangian block is pinned: its values are
      // known, and its edges go to the block scan directly
      const int r0 = i & ~31, ri = i - r0;
      const int nr = min(32, H - r0), ncl = min(32, W - 32 * bj);
      const int64_t nblk = (int64_t)p.nbx * p.nby;
      const int64_t blk = (int64_t)(i >> 5) * p.nbx + bj;
      if (ri == nr - 1) {
        bio.lb[blk * 32 + lane] = vu;
        bio.lb[(nblk + blk) * 32 + lane] = vv;
      }
      if (lane == ncl - 1) {
        bio.lr[blk * 32 + ri] = vu;
        bio.lr[(nblk + blk) * 32 + ri] = vv;
      }
      if (ri == 0 && lane == 0) {
        bio.cls[blk] = BS_KNOWN;
        bio.cls[nblk + blk] = BS_KNOWN;
      }
    }
  }
}

// ---------------------------------------------------------- decoder prep
// One 32x32 tile per CTA (8 warps x 4 rows, lane = column).  The decoder's
// recurrence recon = reconU + reconL - reconUL + Pd + (sym-radius)*2e
// (Pd = p - pU - pL + pUL of the previous frame p) is run on
// Z = recon - p, for which the previous frame drops out:
//   Z = ZU + ZL - ZUL + (sym-radius)*2e     (Lorenzo pixels)
//   Z = recon - p                           (pins: lossless, escapes,
//                                            semi-Lagrangian pixels)
// so only pinned pixels read p; the interior pass adds p back.  The four
// rows of a warp are processed together so their stream loads overlap.
template <typename SYM>
__global__ void __launch_bounds__(256, 4)
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
  const int H = p.H, W = p.W, Wp = p.Wp, nchunks = p.nchunks;
  const int bj = blockIdx.x, bi = blockIdx.y;
  const int c0 = 32 * bj, r0 = 32 * bi;
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int64_t HW = (int64_t)H * W;
  const bool has_prev = p.t > 0;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  const bool sl_blk = has_prev && modes_t && modes_t[bi * p.nbx + bj] == 1;
  const int j = c0 + lane;
  const bool colok = j < W;
  constexpr int NR = 4;
  int cd[NR];
  int64_t qrow[NR], lrow[NR];
  int32_t pnl[NR], pll[NR];
  bool rv[NR];
#pragma unroll
  for (int q = 0; q < NR; q++) {
    const int i = r0 + ty + 8 * q;
    rv[q] = i < H;
    const int ic = rv[q] ? i : r0;
    const int64_t row = (int64_t)p.t * H + ic;
    cd[q] = (colok && rv[q]) ? codes[(int64_t)p.t * HW + (int64_t)ic * W + j] : CODE_LOSSLESS;
    qrow[q] = qd_row_off[row];
    lrow[q] = ll_row_off[row];
    pnl[q] = pre_nl[row * nchunks + bj];
    pll[q] = pre_ll[row * nchunks + bj];
  }
  int64_t syu[NR], syv[NR];
  unsigned bnl[NR];
#pragma unroll
  for (int q = 0; q < NR; q++) {
    const bool nl = colok && p.lad.e[cd[q]] != 0;
    bnl[q] = __ballot_sync(FULL, nl);
    syu[q] = 0; syv[q] = 0;
    if (nl) {
      const int64_t k = qrow[q] + 2 * ((int64_t)pnl[q] + __popc(bnl[q] & lt));
      if (sizeof(SYM) == 2) {   // the (u, v) pair as one 4-byte load (k even)
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(qd + k));
        syu[q] = w & 0xffffu;
        syv[q] = w >> 16;
      } else {
        syu[q] = qd[k];
        syv[q] = qd[k + 1];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NR; q++) {
    if (!rv[q]) continue;   // warp-uniform
    const int rr = ty + 8 * q;
    const int i = r0 + rr;
    const int64_t e = p.lad.e[cd[q]];
    const bool nl = colok && e != 0;
    const bool eu = (colok && !nl) || (nl && syu[q] == 0);
    const bool ev = (colok && !nl) || (nl && syv[q] == 0);
    const unsigned b_eu = __ballot_sync(FULL, eu);
    const unsigned b_ev = __ballot_sync(FULL, ev);
    int64_t lidx = lrow[q] + pll[q] + __popc(b_eu & lt) + __popc(b_ev & lt);
    const int64_t two_e = 2 * e;
    const int64_t qu = syu[q] - p.radius, qv = syv[q] - p.radius;
    uint32_t val_u = (uint32_t)(qu * two_e);
    uint32_t val_v = (uint32_t)(qv * two_e);
    const bool sl = nl && sl_blk;
    if (sl) {
      int64_t pr_u, pr_v;
      sl_predict2(TwoPlanes{rec_prev_u, rec_prev_v, Wp}, H, W, i, j, p.cfl_x,
                  p.cfl_y, p.d_max, p.n_max, &pr_u, &pr_v);
      val_u = (uint32_t)(pr_u + qu * two_e);
      val_v = (uint32_t)(pr_v + qv * two_e);
    }
    if (eu) { val_u = (uint32_t)ll[lidx]; lidx++; }
    if (ev) val_v = (uint32_t)ll[lidx];
    const bool pu = colok && (eu || sl), pv = colok && (ev || sl);
    const unsigned b_pu = __ballot_sync(FULL, pu);
    const unsigned b_pv = __ballot_sync(FULL, pv);
    const int64_t pr = (int64_t)i * Wp + j;
    if (has_prev) {   // pinned: Z = recon - p
      if (pu) val_u -= (uint32_t)__ldg(rec_prev_u + pr);
      if (pv) val_v -= (uint32_t)__ldg(rec_prev_v + pr);
    }
    a0[pr] = colok ? (int32_t)val_u : 0;
    a1[pr] = colok ? (int32_t)val_v : 0;
    if (lane == 0) {
      const int64_t pb = (int64_t)i * nchunks + bj;
      pin_u[pb] = b_pu;
      pin_v[pb] = b_pv;
    }
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
cudaError_t launch_enc_r0(const F* u, const F* v, const uint8_t* codes,
                          const int32_t* eu, const int32_t* ev,
                          const PrepParams& p, const BScanIO& bio,
                          int32_t* a0, int32_t* a1,
                          int32_t* prevrec, uint8_t* codes_p, int* overflow,
                          cudaStream_t st) {
  const dim3 grid(p.nchunks, p.nby);
  enc_r0_kernel<F><<<grid, 256, 0, st>>>(
      u, v, codes, eu, ev, p, bio, a0, a1,
      reinterpret_cast<int2*>(prevrec), codes_p, overflow);
  return cudaGetLastError();
}

template <typename F>
cudaError_t launch_enc_mop(const F* u, const F* v, const int32_t* a0,
                           const int32_t* a1, const int32_t* prevrec,
                           const PrepParams& p, const double* log2tab,
                           uint8_t* modes_t, cudaStream_t st) {
  enc_mop_kernel<F><<<dim3(p.nbx, p.nby), 128, 0, st>>>(
      u, v, a0, a1, reinterpret_cast<const int2*>(prevrec), p, log2tab, modes_t);
  return cudaGetLastError();
}

template <typename F>
cudaError_t launch_enc_pix(const F* u, const F* v, const uint8_t* codes_p,
                           const int32_t* prevrec, const int64_t* qd_row_off,
                           const int32_t* pre_nl, const PrepParams& p,
                           const uint8_t* modes_t, const BScanIO& bio,
                           int32_t* a0, int32_t* a1,
                           uint32_t* pin_u, uint32_t* pin_v, uint32_t* nlw,
                           uint16_t* qd, int32_t* row_ll, cudaStream_t st) {
  const dim3 grid((p.nchunks + 7) / 8, (p.H + 1) / 2);
  enc_pix_kernel<F><<<grid, 256, 0, st>>>(
      u, v, codes_p, reinterpret_cast<const int2*>(prevrec), qd_row_off,
      pre_nl, p, modes_t, bio, a0, a1, pin_u, pin_v, nlw, qd, row_ll);
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
  const dim3 grid(p.nchunks, p.nby);
  dec_prep_kernel<SYM><<<grid, 256, 0, st>>>(
      codes, qd, ll, modes_t, ru, rv, qd_row_off, ll_row_off, pre_nl, pre_ll,
      p, a0, a1, pin_u, pin_v);
  return cudaGetLastError();
}



template cudaError_t launch_chunk_prefix<uint16_t>(const uint8_t*,
                                                   const uint16_t*,
                                                   const int64_t*, int64_t,
                                                   int, int, int64_t,
                                                   int32_t*, int32_t*,
                                                   cudaStream_t);
template cudaError_t launch_enc_r0<float>(const float*, const float*,
                                          const uint8_t*, const int32_t*,
                                          const int32_t*, const PrepParams&,
                                          const BScanIO&, int32_t*, int32_t*,
                                          int32_t*, uint8_t*, int*,
                                          cudaStream_t);
template cudaError_t launch_enc_mop<float>(const float*, const float*,
                                           const int32_t*, const int32_t*,
                                           const int32_t*, const PrepParams&,
                                           const double*, uint8_t*,
                                           cudaStream_t);
template cudaError_t launch_enc_pix<float>(
    const float*, const float*, const uint8_t*, const int32_t*, const int64_t*,
    const int32_t*, const PrepParams&, const uint8_t*, const BScanIO&,
    int32_t*, int32_t*, uint32_t*, uint32_t*, uint32_t*, uint16_t*, int32_t*,
    cudaStream_t);
template cudaError_t launch_enc_r0<double>(const double*, const double*,
                                          const uint8_t*, const int32_t*,
                                          const int32_t*, const PrepParams&,
                                          const BScanIO&, int32_t*, int32_t*,
                                          int32_t*, uint8_t*, int*,
                                          cudaStream_t);
template cudaError_t launch_enc_mop<double>(const double*, const double*,
                                           const int32_t*, const int32_t*,
                                           const int32_t*, const PrepParams&,
                                           const double*, uint8_t*,
                                           cudaStream_t);
template cudaError_t launch_enc_pix<double>(
    const double*, const double*, const uint8_t*, const int32_t*, const int64_t*,
    const int32_t*, const PrepParams&, const uint8_t*, const BScanIO&,
    int32_t*, int32_t*, uint32_t*, uint32_t*, uint32_t*, uint16_t*, int32_t*,
    cudaStream_t);
template cudaError_t launch_dec_prep<uint16_t>(
    const uint8_t*, const uint16_t*, const int64_t*, const uint8_t*,
    const int32_t*, const int32_t*, const int64_t*, const int64_t*,
    const int32_t*, const int32_t*, const PrepParams&, int32_t*, int32_t*,
    uint32_t*, uint32_t*, cudaStream_t);

}  // namespace vfcp
