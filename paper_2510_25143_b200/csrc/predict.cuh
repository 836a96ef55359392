// Semi-Lagrangian prediction (predictors.py:33-108), the MoP block
// entropy estimate (mop.py:118-151) and the MoP Lorenzo trial step, shared by
// the encoder's block kernel (enc_block.cu), the decoder's prepare kernel
// and the older frame kernels (fast.cu).
#pragma once

#include "frame.cuh"

namespace vfcp {

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

// recon(t-1) tile: the block plus SLH cells on every side, so the
// semi-Lagrangian departure points of the trial and of SL blocks mostly
// gather from shared memory (TileSrc falls back to global memory outside)
constexpr int SLH = 8;
constexpr int SLT = 32 + 2 * SLH;

// Value source of the semi-Lagrangian sampler (below): recon(t-1)
// from the block's shared tile, or global memory outside it.
struct TileSrc {
  const int2 (*t)[SLT];
  int ti0, tj0;           // frame coordinates of t[0][0]
  const int2* g;          // recon(t-1), pitch Wp
  int Wp;
  __device__ __forceinline__ void get(int i, int j, double& u, double& v) const {
    const int a = i - ti0, b = j - tj0;
    const int2 x = ((unsigned)a < (unsigned)SLT && (unsigned)b < (unsigned)SLT)
                       ? t[a][b]
                       : __ldg(g + (int64_t)i * Wp + j);
    u = (double)x.x;
    v = (double)x.y;
  }
};


// Load the recon(t-1) tile of the block at (r0, c0) with its SLH margin
// (zero outside the frame; all of the CTA's threads, 16-byte loads:
// c0 - SLH is even).
__device__ __forceinline__ void load_prev_tile(int2 (*tile)[SLT],
                                               const int2* prev, int H, int W,
                                               int Wp, int r0, int c0,
                                               int tid, int nthreads) {
  const int ti0 = r0 - SLH, tj0 = c0 - SLH;
  int4* dst = reinterpret_cast<int4*>(&tile[0][0]);
  constexpr int NQ = SLT * SLT / 2;
#pragma unroll 3
  for (int k = tid; k < NQ; k += nthreads) {
    const int a = k / (SLT / 2), b2 = (k - a * (SLT / 2)) * 2;
    const int i = ti0 + a, j = tj0 + b2;
    int4 x = make_int4(0, 0, 0, 0);
    if (prev && i >= 0 && i < H && j >= 0) {
      const int2* src = prev + (int64_t)i * Wp + j;
      if (j + 1 < W) {
        x = __ldg(reinterpret_cast<const int4*>(src));
      } else if (j < W) {
        const int2 y = __ldg(src);
        x = make_int4(y.x, y.y, 0, 0);
      }
    }
    dst[k] = x;
  }
}

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
  // |recon| < 2^30 + 2^29 on the block path, so is every interpolated value
  *pu = rha_d32(vu);
  *pv = rha_d32(vv);
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

// The general predictor (Euler substeps when d_inf > d_max) out of line:
// one copy of its code per kernel, taken by the rare samples whose RK2 fast
// path does not apply.
static __device__ __noinline__ void sl_general(const int2* prev, int Wp, int H,
                                               int W, int i, int j,
                                               double cfl_x, double cfl_y,
                                               double d_max, int n_max,
                                               int64_t* pu, int64_t* pv) {
  sl_predict2(PairPlane{prev, Wp}, H, W, i, j, cfl_x, cfl_y, d_max, n_max, pu, pv);
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
static __device__ double block_rate(const int16_t* samp, int ns, int16_t* cnt,
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
  return esc ? 0 : (int32_t)((int64_t)(q - q0) * 2 * e - y);
}

}  // namespace vfcp
