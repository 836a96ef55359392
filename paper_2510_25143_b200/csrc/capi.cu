// C ABI (include/vfcp_b200.h): host-side orchestration of the B200 kernels.
//
// The frame loop mirrors codec.py:359-376 (compress) and codec.py:427-446
// (decompress): modes for frame t >= 1 are selected on the reconstruction of
// frame t-1, then frame t is encoded; two frame buffers per component ring in
// HBM.  Scratch memory comes from the stream-ordered allocator.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vfcp_b200.h"
#include "bscan.cuh"
#include "common.cuh"
#include "wavefront.cuh"

namespace vfcp {
// analyze.cu
template <typename F>
cudaError_t launch_range(const F*, const F*, int64_t, double*, int,
                         cudaStream_t);
template <typename F>
cudaError_t launch_analyze(const F*, const F*, int, int, int, double, int64_t,
                           uint8_t*, uint32_t*, uint16_t*, int32_t*,
                           uint64_t*, unsigned long long*, int*,
                           unsigned long long, int, cudaStream_t);
template <typename F>
cudaError_t launch_analyze_slab(const F*, const F*, int, int, int, int, int,
                                double, int64_t, uint8_t*, uint32_t*,
                                uint16_t*, int32_t*, uint64_t*,
                                unsigned long long*, int*, unsigned long long,
                                int, cudaStream_t);
cudaError_t launch_row_scan(const int32_t*, int64_t, int, int, int64_t*,
                            cudaStream_t);
// encode.cu
template <typename F, typename I>
cudaError_t launch_mop(const F*, const F*, const I*, const I*,
                       const FrameParams&, const double*, uint8_t*, double*,
                       cudaStream_t);
template <typename F, typename I, typename SYM>
cudaError_t launch_encode(const F*, const F*, const uint8_t*, const I*,
                          const I*, I*, I*, const uint8_t*,
                          const FrameParams&, const Ladder&, const int64_t*,
                          SYM*, int32_t*, I*, int*, int*, cudaStream_t);
template <typename F, typename SYM>
cudaError_t launch_ll_write(const F*, const F*, const uint8_t*, const SYM*,
                            const int64_t*, const int32_t*, const int64_t*,
                            int64_t, int, int, double, int64_t*,
                            cudaStream_t);
// decode.cu
cudaError_t launch_decode_rows(const uint8_t*, const uint8_t*, int64_t, int,
                               int64_t, int32_t*, int*, cudaStream_t);
template <typename SYM>
cudaError_t launch_decode_ll(const SYM*, const int64_t*, const int32_t*,
                             int64_t, int32_t*, cudaStream_t);
template <typename IW, typename SYM>
cudaError_t launch_decode(const uint8_t*, const SYM*, const int64_t*,
                          const uint8_t*, const DecodeParams&, const Ladder&,
                          const int64_t*, const int64_t*, double*, double*,
                          int64_t*, int64_t*, IW*, int, uint64_t*,
                          const WaveSched&, int, int, cudaStream_t);
// fast.cu
template <typename SYM>
cudaError_t launch_chunk_prefix(const uint8_t*, const SYM*, const int64_t*,
                                int64_t, int, int, int64_t, int32_t*,
                                int32_t*, cudaStream_t);
// enc_block.cu
template <typename F>
cudaError_t launch_enc_block(const F*, const F*, const uint8_t*,
                             const int32_t*, int32_t*, const PrepParams&,
                             const BScanIO&, const double*, uint8_t*,
                             const int64_t*, const int32_t*, uint16_t*,
                             int32_t*, int*, cudaStream_t);
// dec_block.cu
template <typename SYM>
bool dec_block_split(const uint8_t*, const PrepParams&);
template <typename SYM>
cudaError_t launch_dec_block_fast(const uint8_t*, const SYM*, const uint8_t*,
                                  bool, const int64_t*, const int32_t*,
                                  const PrepParams&, const BScanIO&,
                                  const int32_t*, int*, int*, cudaStream_t);
template <typename SYM>
cudaError_t launch_dec_block(const uint8_t*, const SYM*, const int64_t*,
                             const uint8_t*, const int32_t*, int32_t*,
                             const int64_t*, const int64_t*, const int32_t*,
                             const int32_t*, const PrepParams&, const BScanIO&,
                             uint32_t*, uint32_t*, double*, double*, int64_t*,
                             int64_t*, double, const int*, const int*, int,
                             cudaStream_t);
}  // namespace vfcp

using namespace vfcp;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(...)                                                            \
  do {                                                                     \
    cudaError_t _e = (__VA_ARGS__);                                        \
    if (_e != cudaSuccess)                                                 \
      return fail(VFCP_ECUDA, std::string(#__VA_ARGS__) + ": " +           \
                                  cudaGetErrorString(_e));                 \
  } while (0)

// ---- launch accounting: every kernel launch goes through LAUNCH(), which
// counts it and, when profiling is on, brackets it with CUDA events on the
// launching stream (vfcp_prof_*).
enum KClass { K_RANGE, K_ANALYZE, K_SCAN, K_MOP, K_ENCODE, K_LLW, K_DROWS,
              K_DLL, K_DECODE, K_AUX, K_EBLK, K_DBLK, K_BSC, K_NCLS };
struct Prof {
  bool on = false;
  int64_t launches = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
};
Prof g_prof;

#define LAUNCH(cls, st, ...)                                               \
  do {                                                                     \
    cudaEvent_t _a = nullptr, _b = nullptr;                                \
    if (g_prof.on) {                                                       \
      cudaEventCreate(&_a);                                                \
      cudaEventCreate(&_b);                                                \
      cudaEventRecord(_a, st);                                             \
    }                                                                      \
    CK(__VA_ARGS__);                                                       \
    g_prof.launches++;                                                     \
    if (g_prof.on) {                                                       \
      cudaEventRecord(_b, st);                                             \
      g_prof.ev.push_back({(int)(cls), {_a, _b}});                         \
    }                                                                      \
  } while (0)

// Stream-ordered scratch from the device's default memory pool.  The pool
// keeps freed memory (release threshold = max) so repeated calls do not
// re-map gigabytes of scratch at every synchronisation.
void keep_pool_memory() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) { keep_pool_memory(); }
  template <typename T>
  cudaError_t get(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, count * sizeof(T) + 16, st);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = (T*)q;
    return e;
  }
  ~Scratch() {
    for (void* q : ptrs) cudaFreeAsync(q, st);
  }
};

int check_params(const vfcp_params* p) {
  if (!p) return fail(VFCP_EINVAL, "null params");
  if (p->H < 2 || p->W < 2 || p->T < 2)
    return fail(VFCP_EINVAL, "dims must be >= 2");
  if (p->bx < 1 || p->by < 1 || p->stride < 1)
    return fail(VFCP_EINVAL, "block grid / stride must be positive");
  if (p->radius < 1) return fail(VFCP_EINVAL, "radius must be positive");
  if (p->tau < 0) return fail(VFCP_EINVAL, "tau must be non-negative");
  if (p->predictor < 0 || p->predictor > 2)
    return fail(VFCP_EINVAL, "unknown predictor");
  return VFCP_OK;
}

Ladder make_ladder(int64_t tau) {
  Ladder L;
  for (int k = 0; k < 32; k++) {
    int64_t e = (k == CODE_LOSSLESS || tau <= 0) ? 0 : (tau >> (k > 62 ? 62 : k));
    L.e[k] = e;
    L.inv2e[k] = e ? 1.0 / (2.0 * (double)e) : 0.0;
  }
  return L;
}

bool narrow_frames(int64_t tau) { return tau < (((int64_t)1) << 30) - 1; }
bool narrow_symbols(int radius) { return radius <= 32768; }

FrameParams frame_params(const vfcp_params* p, int t) {
  FrameParams f;
  f.H = p->H; f.W = p->W; f.T = p->T; f.t = t;
  f.S = p->scale;
  f.tau = p->tau;
  f.radius = p->radius;
  f.bx = p->bx; f.by = p->by; f.stride = p->stride;
  f.nbx = (p->W + p->bx - 1) / p->bx;
  f.nby = (p->H + p->by - 1) / p->by;
  f.lam = p->lam; f.theta = p->theta;
  f.rmeta = 1.0 / (double)(p->bx * p->by * 2);
  f.d_max = p->d_max;
  f.n_max = p->n_max;
  f.cfl_x = (p->dt / p->dx) / p->scale;   // predictors.py:117-119
  f.cfl_y = (p->dt / p->dy) / p->scale;
  f.use_modes = t >= 1;
  return f;
}

template <typename I>
__global__ void widen_kernel(const I* a, const I* b, int64_t n, int64_t* oa,
                             int64_t* ob) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    oa[k] = a[k];
    ob[k] = b[k];
  }
}

// Fast path, optional recon output: recon(t) from the (u, v) pair plane
// (pitch Wp) as int64 [2][T][H][W] (the layout of the generic path's
// widen_kernel).
__global__ void recon_pairs_kernel(const int2* __restrict__ rec, int H, int W,
                                   int Wp, int t, int64_t N,
                                   int64_t* __restrict__ recon) {
  const int64_t HW = (int64_t)H * W;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < HW;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / W, j = k - i * W;
    const int2 r = rec[i * Wp + j];
    const int64_t g = (int64_t)t * HW + k;
    recon[g] = r.x;
    recon[N + g] = r.y;
  }
}

template <typename F, typename I, typename SYM>
int encode_impl(const vfcp_params* p, const F* u, const F* v,
                const uint8_t* codes, const int64_t* qd_row_off, SYM* qd,
                uint8_t* modes, double* scores, int32_t* row_ll,
                int64_t* recon, cudaStream_t st) {
  const int H = p->H, W = p->W, T = p->T;
  const int64_t HW = (int64_t)H * W, N = HW * T;
  const int nstrips = (H + 31) / 32;
  const int nbx = (W + p->bx - 1) / p->bx, nby = (H + p->by - 1) / p->by;
  const int64_t nblk = (int64_t)nbx * nby;
  Scratch sc(st);
  I *fr, *bnd;
  int *progress, *ticket;
  double* log2tab = nullptr;
  CK(sc.get(&fr, 4 * (size_t)HW));
  CK(sc.get(&bnd, (size_t)nstrips * W * 2));
  CK(sc.get(&progress, (size_t)nstrips + 1));
  CK(sc.get(&ticket, 1));
  const bool mop = p->predictor == VFCP_PRED_MOP && p->tau > 0;
  if (mop) {
    int nlog = 2 * p->bx * p->by + 1;
    std::vector<double> tab(nlog);
    tab[0] = 0.0;
    for (int h = 1; h < nlog; h++) tab[h] = std::log2((double)h);
    CK(sc.get(&log2tab, (size_t)nlog));
    CK(cudaMemcpyAsync(log2tab, tab.data(), sizeof(double) * nlog,
                       cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // tab is a host temporary
  }
  if (T > 1)
    CK(cudaMemsetAsync(modes,
                       (p->predictor == VFCP_PRED_SL && p->tau > 0) ? 1 : 0,
                       (size_t)(T - 1) * nblk, st));
  if (scores && T > 1)
    CK(cudaMemsetAsync(scores, 0, sizeof(double) * 2 * (T - 1) * nblk, st));
  I* pu = fr;
  I* pv = fr + HW;
  I* cu = fr + 2 * HW;
  I* cv = fr + 3 * HW;
  CK(cudaMemsetAsync(pu, 0, sizeof(I) * 2 * HW, st));
  Ladder lad = make_ladder(p->tau);
  for (int t = 0; t < T; t++) {
    FrameParams fp = frame_params(p, t);
    const uint8_t* modes_t = t >= 1 ? modes + (size_t)(t - 1) * nblk : modes;
    if (mop && t >= 1) {
      LAUNCH(K_MOP, st, launch_mop<F, I>(u, v, pu, pv, fp, log2tab, modes,
                                        scores, st));
    }
    LAUNCH(K_ENCODE, st,
           launch_encode<F, I, SYM>(u, v, codes, pu, pv, cu, cv, modes_t, fp,
                                    lad, qd_row_off, qd, row_ll, bnd,
                                    progress, ticket, st));
    if (recon)
      LAUNCH(K_AUX, st,
             (widen_kernel<I><<<1184, 256, 0, st>>>(cu, cv, HW, recon + t * HW,
                                                    recon + N + t * HW),
              cudaGetLastError()));
    std::swap(pu, cu);
    std::swap(pv, cv);
  }
  CK(cudaGetLastError());
  return VFCP_OK;
}

// Semi-Lagrangian reach (cells) of a departure point plus its bilinear
// stencil: |displacement| <= max|prev| * cfl (predictors.py:76-108, RK2 and
// substeps alike), +1 for the i1/j1 tap, +1 margin.
int sl_reach(double maxabs_fixed, double cfl, int lim) {
  double r = std::ceil(maxabs_fixed * cfl) + 2.0;
  if (!(r < (double)lim)) return lim;
  return (int)r;
}

template <typename I, typename SYM>
int decode_impl(const vfcp_params* p, const uint8_t* codes, const SYM* qd,
                int64_t n_qd, const int64_t* ll, int64_t n_ll,
                const uint8_t* modes,
                const int64_t* qd_row_off, const int64_t* ll_row_off,
                double* out_u, double* out_v, int64_t* fix_u, int64_t* fix_v,
                cudaStream_t st) {
  const int H = p->H, W = p->W, T = p->T;
  const int K = (H + 31) / 32;
  const int nbx = (W + p->bx - 1) / p->bx, nby = (H + p->by - 1) / p->by;
  const int64_t nblk = (int64_t)nbx * nby;
  int dev = 0, nsm = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // any semi-Lagrangian block at all?  (decides the inter-frame reach)
  bool any_sl = false;
  if (T > 1) {
    std::vector<uint8_t> hm((size_t)(T - 1) * nblk);
    CK(cudaMemcpyAsync(hm.data(), modes, hm.size(), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    for (uint8_t x : hm) if (x) { any_sl = true; break; }
  }
  Scratch sc(st);
  uint64_t* bnd;
  int *sched;
  const size_t nbnd = (size_t)T * K * 2 * W * (sizeof(I) / 4);
  CK(sc.get(&bnd, nbnd));
  // int recon frames, rows padded to 32 elements (128 B lines never straddle
  // a strip / chunk boundary, so cp.async through L1 can never see a stale
  // line of a frame written earlier in the same kernel)
  const int Wp = (W + 31) / 32 * 32;
  I* rec;
  CK(sc.get(&rec, (size_t)T * 2 * H * Wp));
  CK(cudaMemsetAsync(bnd, 0, sizeof(uint64_t) * nbnd, st));
  CK(sc.get(&sched, (size_t)2 * T * K + 1));
  CK(cudaMemsetAsync(sched, 0, sizeof(int) * (2 * (size_t)T * K + 1), st));
  WaveSched ws;
  ws.ticket = sched;
  ws.prog = sched + 1;
  ws.bprog = sched + 1 + (size_t)T * K;
  ws.K = K;
  const double cfl_x = (p->dt / p->dx) / p->scale;
  const double cfl_y = (p->dt / p->dy) / p->scale;
  // recon magnitude <= 2^30 + tau' (|fixed| < 2^30, |err| <= e <= tau')
  const double bound = 1073741824.0 + (double)p->tau;
  const int reach_rows = any_sl ? sl_reach(bound, cfl_y, H) : 0;
  ws.reach_cols = any_sl ? sl_reach(bound, cfl_x, W) : 0;
  ws.reach_strips = (reach_rows + 31) / 32;
  ws.stats = nullptr;
  const bool wprof = getenv("VFCP_WAVE_PROFILE") != nullptr;
  if (wprof) {
    CK(sc.get(&ws.stats, WP_N));
    CK(cudaMemsetAsync(ws.stats, 0, sizeof(unsigned long long) * WP_N, st));
  }
  DecodeParams dp;
  dp.H = H; dp.W = W; dp.T = T; dp.t = 0;
  dp.n_qd = n_qd;
  dp.n_ll = n_ll;
  dp.inv_S = 1.0 / p->scale;
  dp.S = p->scale;
  dp.radius = p->radius;
  dp.bx = p->bx; dp.by = p->by; dp.nbx = nbx;
  dp.d_max = p->d_max;
  dp.n_max = p->n_max;
  dp.cfl_x = cfl_x;
  dp.cfl_y = cfl_y;
  dp.use_modes = any_sl ? 1 : 0;
  Ladder lad = make_ladder(p->tau);
  LAUNCH(K_DECODE, st,
         launch_decode<I, SYM>(codes, qd, ll, modes, dp, lad, qd_row_off,
                               ll_row_off, out_u, out_v, fix_u, fix_v, rec,
                               Wp, bnd, ws, reach_rows, nsm, st));
  if (wprof) {
    unsigned long long h[WP_N];
    CK(cudaMemcpyAsync(h, ws.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fprintf(stderr,
            "[wave decode] tasks=%llu total=%.3g waitprev=%.3g pre=%.3g "
            "waitbnd=%.3g chain=%.3g write=%.3g preload=%.3g sweep=%.3g "
            "stage+bndput=%.3g (warp-cycles)\n",
            h[WP_TASKS], (double)h[WP_TOTAL], (double)h[WP_WAITPREV],
            (double)h[WP_PRE], (double)h[WP_WAITBND], (double)h[WP_CHAIN],
            (double)h[WP_WRITE], (double)h[WP_X1], (double)h[WP_X2],
            (double)h[WP_X3]);
  }
  return VFCP_OK;
}

// ------------------------------------------------------------ fast paths
// Block kernels + block scan (enc_block.cu, dec_block.cu, bscan.cuh).  Valid
// for the default 32x32 block grid, 16-bit symbols and tau' < 2^29 (errors,
// recon values and the residue moduli 2e then fit 32 bits; the few sums that
// can exceed them are taken in int64); the caller falls back to the generic
// kernels otherwise.
bool fast_ok(const vfcp_params* p) {
  return p->bx == 32 && p->by == 32 && p->radius <= 32768 &&
         p->tau < ((int64_t)1 << 29) && p->stride >= 2 && p->H <= 65535;
}

PrepParams prep_params(const vfcp_params* p, int t, const Ladder& lad) {
  PrepParams pp;
  pp.H = p->H; pp.W = p->W;
  pp.nchunks = (p->W + 31) / 32;
  pp.Wp = 32 * pp.nchunks;
  pp.nbx = pp.nchunks;
  pp.nby = (p->H + 31) / 32;
  pp.t = t;
  pp.S = p->scale;
  pp.cfl_x = (p->dt / p->dx) / p->scale;
  pp.cfl_y = (p->dt / p->dy) / p->scale;
  pp.d_max = p->d_max;
  pp.lam = p->lam;
  pp.theta = p->theta;
  pp.rmeta = 1.0 / (double)(p->bx * p->by * 2);
  pp.n_max = p->n_max;
  pp.stride = p->stride;
  pp.radius = p->radius;
  pp.tau = p->tau;
  pp.mop = p->predictor == VFCP_PRED_MOP && t >= 1 && p->tau > 0;
  pp.force_sl = p->predictor == VFCP_PRED_SL && t >= 1 && p->tau > 0;
  pp.lad = lad;
  pp.lossy_mask = 0;
  for (int k = 0; k < 32; k++)
    if (lad.e[k] > 0) pp.lossy_mask |= 1u << k;
  return pp;
}

// Tables and scratch of the block-scan chain (bscan.cuh).
int bscan_setup(Scratch& sc, const Ladder& lad, int H, int W, int radius,
                cudaStream_t st, BScanIO* b) {
  memset(b, 0, sizeof(*b));
  const int nchunks = (W + 31) / 32, nby = (H + 31) / 32;
  const int64_t nblk = (int64_t)nchunks * nby;
  const int ntask = bs_ntask(nby);
  CK(sc.get(&b->lb, (size_t)2 * nblk * 32));
  CK(sc.get(&b->lr, (size_t)2 * nblk * 32));
  CK(sc.get(&b->ebot, (size_t)2 * nblk * 32));
  CK(sc.get(&b->prog, (size_t)2 * nby));
  CK(cudaMemsetAsync(b->prog, 0, sizeof(unsigned long long) * 2 * nby, st));
  CK(sc.get(&b->eright, (size_t)2 * nblk * 32));
  CK(sc.get(&b->cls, (size_t)2 * nblk));
  CK(sc.get(&b->bnd, (size_t)ntask * W));
  CK(cudaMemsetAsync(b->bnd, 0, sizeof(uint64_t) * ntask * W, st));
  b->H = H; b->W = W; b->Wp = 32 * nchunks; b->nchunks = nchunks;
  b->nbx = nchunks; b->nby = nby;
  b->radius = radius;
  for (int k = 0; k < 32; k++) {
    const int64_t e = lad.e[k];
    b->e_tab[k] = (int32_t)e;
    b->mag_tab[k] = e > 0 ? (uint32_t)((((uint64_t)1) << 32) / (2 * (uint64_t)e)) : 0u;
    b->c32_tab[k] = e > 0 ? (uint32_t)((((uint64_t)1) << 32) % (2 * (uint64_t)e)) : 0u;
  }
  return VFCP_OK;
}

// VFCP_CHAIN_STAMPS: per block row start / first block / end of frame 1's
// chain (ns from the first start), to separate pipeline lag from step time
void print_chain_stamps(const BScanIO& b, cudaStream_t st) {
  std::vector<unsigned long long> h((size_t)2 * b.nby * 3);
  if (cudaMemcpyAsync(h.data(), b.stamps, sizeof(unsigned long long) * h.size(),
                      cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return;
  unsigned long long t0 = ~0ull;
  for (int k = 0; k < b.nby; k++) t0 = h[k * 3] < t0 ? h[k * 3] : t0;
  if (b.phase) {
    std::vector<unsigned long long> ph((size_t)b.nby * 8);
    if (cudaMemcpy(ph.data(), b.phase, sizeof(unsigned long long) * ph.size(),
                   cudaMemcpyDeviceToHost) == cudaSuccess) {
      fprintf(stderr, "[chain phases] row: topwait meta chain+bots ringwait rights writes (kcycles)\n");
      for (int k = 0; k < b.nby; k += (b.nby > 16 ? b.nby / 16 : 1))
        fprintf(stderr, "  %5d %8.1f %8.1f %8.1f %8.1f %8.1f %8.1f\n", k,
                ph[k * 8] * 1e-3, ph[k * 8 + 1] * 1e-3, ph[k * 8 + 2] * 1e-3,
                ph[k * 8 + 3] * 1e-3, ph[k * 8 + 4] * 1e-3, ph[k * 8 + 5] * 1e-3);
    }
  }
  fprintf(stderr, "[chain stamps] block row: start first-top end (us, comp u)\n");
  for (int k = 0; k < b.nby; k += (b.nby > 32 ? b.nby / 32 : 1))
    fprintf(stderr, "  %5d %9.1f %9.1f %9.1f\n", k, (h[k * 3] - t0) * 1e-3,
            (h[k * 3 + 1] - t0) * 1e-3, (h[k * 3 + 2] - t0) * 1e-3);
}

// VFCP_CLS_STATS: block classes of a frame after its chain (DONE = swept)
void print_cls_stats(const BScanIO& b, int t, cudaStream_t st) {
  const int64_t nblk = (int64_t)b.nbx * b.nby;
  std::vector<int32_t> h((size_t)2 * nblk);
  if (cudaMemcpyAsync(h.data(), b.cls, sizeof(int32_t) * h.size(),
                      cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return;
  long cnt[2][4] = {{0}}, codes[32] = {0};
  for (int c = 0; c < 2; c++)
    for (int64_t k = 0; k < nblk; k++) {
      cnt[c][h[c * nblk + k] & 3]++;
      if ((h[c * nblk + k] & 3) == BS_REG) codes[(h[c * nblk + k] >> 2) & 31]++;
    }
  fprintf(stderr, "[cls] t=%d u: slow %ld known %ld reg %ld swept %ld | v: slow %ld known %ld reg %ld swept %ld | reg codes:",
          t, cnt[0][0], cnt[0][1], cnt[0][2], cnt[0][3], cnt[1][0], cnt[1][1], cnt[1][2], cnt[1][3]);
  for (int k = 0; k < 32; k++) if (codes[k]) fprintf(stderr, " %d:%ld", k, codes[k]);
  fprintf(stderr, "\n");
}

int nsm_of() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

// D2H of finished frames' symbols on a side stream (vfcp_encode_host)
struct HostOut {
  uint16_t* host_qd = nullptr;
  const int64_t* frame_off = nullptr;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  int init(int T) {
    if (!host_qd) return VFCP_OK;
    CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    ev.resize(T);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return VFCP_OK;
  }
  int frame(int t, const uint16_t* qd, cudaStream_t st) {
    if (!host_qd) return VFCP_OK;
    const int64_t a = frame_off[t], n = frame_off[t + 1] - a;
    if (n <= 0) return VFCP_OK;
    CK(cudaEventRecord(ev[t], st));
    CK(cudaStreamWaitEvent(side, ev[t], 0));
    CK(cudaMemcpyAsync(host_qd + a, qd + a, sizeof(uint16_t) * n,
                       cudaMemcpyDeviceToHost, side));
    return VFCP_OK;
  }
  int finish() {
    if (!side) return VFCP_OK;
    CK(cudaStreamSynchronize(side));
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(side);
    side = nullptr;
    return VFCP_OK;
  }
  ~HostOut() { finish(); }
};

// The frame loop of the block path as a stepping context: begin() sets up
// the scratch and tables, frame(t) enqueues frame t (enc_block_kernel:
// tiles, MoP, SL blocks, block classes and edges; then the block-scan chain
// with the interior pass, bscan.cuh, which writes recon(t) and the Lorenzo
// symbols), end() reads the int32-overflow flag.  vfcp_encode runs the
// frames back to back; vfcp_encode_stream_* lets the caller enqueue frame t
// as soon as its inputs (orig(t), codes(t), qd_row_off of its rows) exist,
// e.g. while later frames are still crossing PCIe.
struct EncFramesBase {
  virtual ~EncFramesBase() {}
  virtual int begin(bool prefix_all) = 0;
  virtual int frame(int t) = 0;
  virtual int end(bool* overflowed) = 0;
};

template <typename F>
struct EncFrames : EncFramesBase {
  vfcp_params P;
  const F *u, *v;
  const uint8_t* codes;
  const int64_t* qd_row_off;
  uint16_t* qd;
  uint8_t* modes;
  int32_t* row_ll;
  int64_t* recon;
  cudaStream_t st;
  Scratch sc;
  int H, W, T, nchunks, Wp, nby, nsm;
  int64_t nblk, HW, plane, cplane;
  int32_t *pre_nl = nullptr, *a = nullptr, *out = nullptr, *rec = nullptr;
  int *ticket = nullptr, *ovf = nullptr;
  double* log2tab = nullptr;
  std::vector<double> tab;
  Ladder lad;
  BScanIO bio;
  bool cls_stats = false, prefix_all = true;

  EncFrames(const vfcp_params* p, const F* u_, const F* v_,
            const uint8_t* codes_, const int64_t* qd_row_off_, uint16_t* qd_,
            uint8_t* modes_, int32_t* row_ll_, int64_t* recon_,
            cudaStream_t st_)
      : P(*p), u(u_), v(v_), codes(codes_), qd_row_off(qd_row_off_), qd(qd_),
        modes(modes_), row_ll(row_ll_), recon(recon_), st(st_), sc(st_) {
    H = P.H; W = P.W; T = P.T;
    nchunks = (W + 31) / 32; Wp = 32 * nchunks;
    nby = (H + 31) / 32;
    nblk = (int64_t)nchunks * nby;
    HW = (int64_t)H * W;
    plane = (int64_t)H * Wp; cplane = (int64_t)H * nchunks;
    nsm = nsm_of();
  }

  int begin(bool prefix_all_) override {
    prefix_all = prefix_all_;
    const vfcp_params* p = &P;
    CK(sc.get(&pre_nl, (size_t)T * cplane));
    CK(sc.get(&a, (size_t)2 * plane));      // R0 of swept blocks
    CK(sc.get(&out, (size_t)2 * plane));    // err of swept blocks
    CK(sc.get(&rec, (size_t)4 * plane));    // recon ping-pong, (u, v) pairs
    CK(sc.get(&ticket, (size_t)2 * T));   // per frame: chain / interior
    CK(sc.get(&ovf, 1));
    CK(cudaMemsetAsync(ticket, 0, sizeof(int) * 2 * T, st));
    CK(cudaMemsetAsync(ovf, 0, sizeof(int), st));
    CK(cudaMemsetAsync(row_ll, 0, sizeof(int32_t) * (size_t)T * H, st));
    const bool mop = p->predictor == VFCP_PRED_MOP && p->tau > 0;
    if (mop) {
      const int nlog = 2 * p->bx * p->by + 1;
      tab.resize(nlog);
      tab[0] = 0.0;
      for (int h = 1; h < nlog; h++) tab[h] = std::log2((double)h);
      CK(sc.get(&log2tab, (size_t)nlog));
      CK(cudaMemcpyAsync(log2tab, tab.data(), sizeof(double) * nlog,
                         cudaMemcpyHostToDevice, st));
    }
    if (T > 1)
      CK(cudaMemsetAsync(modes,
                         (p->predictor == VFCP_PRED_SL && p->tau > 0) ? 1 : 0,
                         (size_t)(T - 1) * nblk, st));
    if (prefix_all)
      LAUNCH(K_SCAN, st,
             launch_chunk_prefix<uint16_t>(codes, nullptr, nullptr,
                                           (int64_t)T * H, W, nchunks, p->tau,
                                           pre_nl, nullptr, st));
    lad = make_ladder(p->tau);
    {
      int rc = bscan_setup(sc, lad, H, W, p->radius, st, &bio);
      if (rc) return rc;
    }
    bio.a[0] = a; bio.a[1] = a + plane;
    bio.a_w[0] = a; bio.a_w[1] = a + plane;
    bio.out[0] = out; bio.out[1] = out + plane;
    bio.qd = qd;
    bio.cpitch = W;
    bio.S = p->scale;
    if (getenv("VFCP_CHAIN_STAMPS")) {
      CK(sc.get(&bio.stamps, (size_t)2 * nby * 3));
      CK(sc.get(&bio.phase, (size_t)nby * 8));
    }
    cls_stats = getenv("VFCP_CLS_STATS") != nullptr;
    bio.dbg_skip_interior = getenv("VFCP_CHAIN_ONLY") != nullptr;
    bio.vec4 = sizeof(F) == 4 && (W & 3) == 0 &&
               (((uintptr_t)u | (uintptr_t)v | (uintptr_t)qd) & 15) == 0;
    return VFCP_OK;
  }

  int frame(int t) override {
    const vfcp_params* p = &P;
    if (t < 0 || t >= T) return fail(VFCP_EINVAL, "frame out of range");
    if (!prefix_all)
      LAUNCH(K_SCAN, st,
             launch_chunk_prefix<uint16_t>(codes + (size_t)t * HW, nullptr,
                                           nullptr, (int64_t)H, W, nchunks,
                                           p->tau, pre_nl + (size_t)t * cplane,
                                           nullptr, st));
    const PrepParams pp = prep_params(p, t, lad);
    int32_t* rprev = rec + 2 * plane * ((t + 1) & 1);
    int32_t* rcur = rec + 2 * plane * (t & 1);
    uint8_t* modes_t = t >= 1 ? modes + (size_t)(t - 1) * nblk : nullptr;
    LAUNCH(K_EBLK, st,
           launch_enc_block<F>(u, v, codes + (size_t)t * HW,
                               t > 0 ? rprev : nullptr, rcur, pp, bio, log2tab,
                               modes_t, qd_row_off, pre_nl, qd, row_ll, ovf, st));
    bio.codes = codes + (size_t)t * HW;
    bio.orig[0] = u + (size_t)t * HW;
    bio.orig[1] = v + (size_t)t * HW;
    bio.prevrec = t > 0 ? reinterpret_cast<const int2*>(rprev) : nullptr;
    bio.rec = reinterpret_cast<int2*>(rcur);
    bio.ticket = ticket + 2 * t;
    bio.tag_base = (uint32_t)t * (uint32_t)bs_ntask(nby);
    bio.qd_row_off = qd_row_off + (size_t)t * H;
    bio.pre_nl = pre_nl + (size_t)t * cplane;
    bio.row_ll = row_ll + (size_t)t * H;
    bio.frame_tag = (uint32_t)t + 1u;
    LAUNCH(K_BSC, st, (launch_bs_chain<true, F>(bio, nsm, st)));
    if (bio.stamps && t == 1) print_chain_stamps(bio, st);
    if (cls_stats) print_cls_stats(bio, t, st);
    if (recon)
      LAUNCH(K_AUX, st,
             (recon_pairs_kernel<<<1184, 256, 0, st>>>(
                  reinterpret_cast<const int2*>(rcur), H, W, Wp, t,
                  (int64_t)H * W * T, recon),
              cudaGetLastError()));
    return VFCP_OK;
  }

  int end(bool* overflowed) override {
    int h_ovf = 0;
    CK(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *overflowed = h_ovf != 0;
    return VFCP_OK;
  }
};

template <typename F>
int encode_fast(const vfcp_params* p, const F* u, const F* v,
                const uint8_t* codes, const int64_t* qd_row_off, uint16_t* qd,
                uint8_t* modes, int32_t* row_ll, int64_t* recon,
                cudaStream_t st, bool* overflowed, HostOut* ho) {
  EncFrames<F> ef(p, u, v, codes, qd_row_off, qd, modes, row_ll, recon, st);
  int rc = ef.begin(true);
  if (rc) return rc;
  for (int t = 0; t < p->T; t++) {
    if ((rc = ef.frame(t))) return rc;
    if ((rc = ho->frame(t, qd, st))) return rc;
  }
  return ef.end(overflowed);
}

// Per-frame copies of the float64 output to (pinned) host memory on a side
// stream, each gated by an event after the frame's last kernel, so the
// transfers of frame t overlap the decode of frames > t.
struct DecHostOut {
  double* hu = nullptr;
  double* hv = nullptr;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  int init(int T) {
    if (!hu) return VFCP_OK;
    CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    ev.resize(T);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return VFCP_OK;
  }
  int frame(int t, int64_t HW, const double* du, const double* dv, cudaStream_t st) {
    if (!hu) return VFCP_OK;
    CK(cudaEventRecord(ev[t], st));
    CK(cudaStreamWaitEvent(side, ev[t], 0));
    CK(cudaMemcpyAsync(hu + t * HW, du + t * HW, sizeof(double) * HW,
                       cudaMemcpyDeviceToHost, side));
    CK(cudaMemcpyAsync(hv + t * HW, dv + t * HW, sizeof(double) * HW,
                       cudaMemcpyDeviceToHost, side));
    return VFCP_OK;
  }
  int finish() {
    if (!side) return VFCP_OK;
    CK(cudaStreamSynchronize(side));
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(side);
    side = nullptr;
    return VFCP_OK;
  }
  ~DecHostOut() { finish(); }
};

int decode_fast(const vfcp_params* p, const uint8_t* codes, const uint16_t* qd,
                const int64_t* ll, const uint8_t* modes,
                const int64_t* qd_row_off, const int64_t* ll_row_off,
                double* out_u, double* out_v, int64_t* fix_u, int64_t* fix_v,
                cudaStream_t st, DecHostOut* ho) {
  // per frame: dec_block_kernel (dec_block.cu: symbols, ll values, SL and
  // KNOWN blocks, block classes and edges) then the block-scan chain with
  // the interior pass (bscan.cuh), which writes recon(t) and the output
  const int H = p->H, W = p->W, T = p->T;
  const int64_t HW = (int64_t)H * W;
  const int nchunks = (W + 31) / 32, Wp = 32 * nchunks;
  const int nby = (H + 31) / 32;
  const int64_t nblk = (int64_t)nchunks * nby;
  const int64_t plane = (int64_t)H * Wp, cplane = (int64_t)H * nchunks;
  const int nsm = nsm_of();
  Scratch sc(st);
  int32_t *pre_nl, *pre_ll, *a, *out, *rec;
  uint32_t* pins;
  int* ticket;
  CK(sc.get(&pre_nl, (size_t)T * cplane));
  CK(sc.get(&pre_ll, (size_t)T * cplane));
  CK(sc.get(&a, (size_t)2 * plane));      // A / Z of swept blocks
  CK(sc.get(&out, (size_t)2 * plane));    // Z of swept blocks
  CK(sc.get(&rec, (size_t)4 * plane));    // recon ping-pong, (u, v) pairs
  CK(sc.get(&pins, (size_t)2 * cplane));
  // blocks the fast block kernel (dec_block.cu) hands to the general one
  // (the fast kernel stays on this stream: run beside the previous frame's
  // chain it takes the chain warps' issue slots and the whole call slows down)
  int *blist, *bcount;
  int32_t* etab_dev;
  CK(sc.get(&blist, (size_t)nblk));
  CK(sc.get(&bcount, (size_t)T));
  CK(sc.get(&etab_dev, 32));
  CK(cudaMemsetAsync(bcount, 0, sizeof(int) * T, st));
  CK(sc.get(&ticket, (size_t)2 * T));   // per frame: chain / interior
  CK(cudaMemsetAsync(ticket, 0, sizeof(int) * 2 * T, st));
  LAUNCH(K_SCAN, st,
         launch_chunk_prefix<uint16_t>(codes, qd, qd_row_off, (int64_t)T * H,
                                       W, nchunks, p->tau, pre_nl, pre_ll,
                                       st));
  const Ladder lad = make_ladder(p->tau);
  BScanIO bio;
  {
    int rc = bscan_setup(sc, lad, H, W, p->radius, st, &bio);
    if (rc) return rc;
  }
  CK(cudaMemcpyAsync(etab_dev, bio.e_tab, sizeof(int32_t) * 32,
                     cudaMemcpyHostToDevice, st));
  bio.a[0] = a; bio.a[1] = a + plane;
  bio.a_w[0] = a; bio.a_w[1] = a + plane;
  bio.out[0] = out; bio.out[1] = out + plane;
  bio.pin[0] = pins; bio.pin[1] = pins + cplane;
  bio.qd = const_cast<uint16_t*>(qd);
  bio.cpitch = W;
  bio.inv_S = 1.0 / p->scale;
  // the interior pass's vector form: 16-byte rows, float64 output only
  bio.vec4 = (W & 3) == 0 && !fix_u && !fix_v &&
             (((uintptr_t)out_u | (uintptr_t)out_v) & 15) == 0;
  const bool split = dec_block_split<uint16_t>(codes, prep_params(p, 0, lad)) &&
                     ((W * (int64_t)H) & 3) == 0;
  for (int t = 0; t < T; t++) {
    const PrepParams pp = prep_params(p, t, lad);
    int32_t* rprev = rec + 2 * plane * ((t + 1) & 1);
    int32_t* rcur = rec + 2 * plane * (t & 1);
    if (split)
      LAUNCH(K_DBLK, st,
             launch_dec_block_fast<uint16_t>(
                 codes + (size_t)t * HW, qd,
                 t >= 1 ? modes + (size_t)(t - 1) * nblk : nullptr, t > 0,
                 qd_row_off, pre_nl, pp, bio, etab_dev, blist, bcount + t, st));
    LAUNCH(K_DBLK, st,
           launch_dec_block<uint16_t>(
               codes + (size_t)t * HW, qd, ll,
               t >= 1 ? modes + (size_t)(t - 1) * nblk : nullptr,
               t > 0 ? rprev : nullptr, rcur, qd_row_off, ll_row_off, pre_nl,
               pre_ll, pp, bio, pins, pins + cplane, out_u, out_v, fix_u,
               fix_v, bio.inv_S, split ? blist : nullptr, bcount + t, nsm, st));
    bio.codes = codes + (size_t)t * HW;
    bio.prevrec = t > 0 ? reinterpret_cast<const int2*>(rprev) : nullptr;
    bio.rec = reinterpret_cast<int2*>(rcur);
    bio.ticket = ticket + 2 * t;
    bio.tag_base = (uint32_t)t * (uint32_t)bs_ntask(nby);
    bio.qd_row_off = qd_row_off + (size_t)t * H;
    bio.pre_nl = pre_nl + (size_t)t * cplane;
    bio.f64[0] = out_u + (size_t)t * HW;
    bio.f64[1] = out_v + (size_t)t * HW;
    bio.fix[0] = fix_u ? fix_u + (size_t)t * HW : nullptr;
    bio.fix[1] = fix_v ? fix_v + (size_t)t * HW : nullptr;
    bio.frame_tag = (uint32_t)t + 1u;
    bio.pin[0] = pins; bio.pin[1] = pins + cplane;
    LAUNCH(K_BSC, st, launch_bs_chain<false>(bio, nsm, st));
    {
      const int rh = ho->frame(t, HW, out_u, out_v, st);
      if (rh) return rh;
    }
  }
  return VFCP_OK;
}

int encode_common(const vfcp_params* p, const void* u, const void* v,
                  int dtype, const uint8_t* codes, const int64_t* qd_row_off,
                  void* qd, uint8_t* modes, double* scores, int32_t* row_ll,
                  int64_t* recon, HostOut* ho, cudaStream_t st) {
  if (fast_ok(p) && !scores && !getenv("VFCP_SLOW_PATH")) {
    bool ovf = false;
    int rc2 = ho->init(p->T);
    if (rc2) return rc2;
    rc2 = dtype == VFCP_F32
              ? encode_fast<float>(p, (const float*)u, (const float*)v,
                                   codes, qd_row_off, (uint16_t*)qd,
                                   modes, row_ll, recon, st, &ovf, ho)
              : encode_fast<double>(p, (const double*)u, (const double*)v,
                                    codes, qd_row_off, (uint16_t*)qd,
                                    modes, row_ll, recon, st, &ovf, ho);
    if (rc2) return rc2;
    rc2 = ho->finish();
    if (rc2 || !ovf) return rc2;
    // an R0 did not fit int32: redo the field with the generic kernels
  }
  const bool nf = narrow_frames(p->tau), ns = narrow_symbols(p->radius);
  int rc = VFCP_OK;
#define ENC(F, I, SYM)                                                      \
  rc = encode_impl<F, I, SYM>(p, (const F*)u, (const F*)v, codes,          \
                              qd_row_off, (SYM*)qd, modes, scores, row_ll,  \
                              recon, st)
  if (dtype == VFCP_F32) {
    if (nf) { if (ns) ENC(float, int32_t, uint16_t); else ENC(float, int32_t, uint32_t); }
    else { if (ns) ENC(float, int64_t, uint16_t); else ENC(float, int64_t, uint32_t); }
  } else {
    if (nf) { if (ns) ENC(double, int32_t, uint16_t); else ENC(double, int32_t, uint32_t); }
    else { if (ns) ENC(double, int64_t, uint16_t); else ENC(double, int64_t, uint32_t); }
  }
#undef ENC
  if (rc || !ho->host_qd) return rc;
  // generic path: the whole stream at the end
  const int64_t n = ho->frame_off[p->T] - ho->frame_off[0];
  if (n > 0) {
    CK(cudaMemcpyAsync(ho->host_qd, qd, sizeof(uint16_t) * n,
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return VFCP_OK;
}

}  // namespace

extern "C" {

const char* vfcp_last_error(void) { return g_err.c_str(); }
}  // extern "C"

int vfcp_record_error(int code, const char* msg) { return fail(code, msg); }

extern "C" {
int vfcp_version(void) { return 1; }

int64_t vfcp_launch_count(void) { return g_prof.launches; }

int vfcp_prof_enable(int on) {
  for (auto& e : g_prof.ev) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  g_prof.ev.clear();
  g_prof.on = on != 0;
  return VFCP_OK;
}

int vfcp_prof_collect(double* ms, int64_t* counts, int ncls) {
  for (int c = 0; c < ncls; c++) { ms[c] = 0.0; counts[c] = 0; }
  for (auto& e : g_prof.ev) {
    CK(cudaEventSynchronize(e.second.second));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e.second.first, e.second.second));
    if (e.first < ncls) { ms[e.first] += t; counts[e.first] += 1; }
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  g_prof.ev.clear();
  return VFCP_OK;
}

int vfcp_value_range(const void* u, const void* v, int dtype, int64_t n,
                     double* out3, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return fail(VFCP_EINVAL, "empty field");
  int dev = 0, nsm = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int nb = nsm * 8;
  Scratch sc(st);
  double* part;
  CK(sc.get(&part, 3 * (size_t)nb));
  if (dtype == VFCP_F32)
    LAUNCH(K_RANGE, st, launch_range((const float*)u, (const float*)v, n, part, nb, st));
  else
    LAUNCH(K_RANGE, st, launch_range((const double*)u, (const double*)v, n, part, nb, st));
  std::vector<double> h(3 * (size_t)nb);
  CK(cudaMemcpyAsync(h.data(), part, sizeof(double) * 3 * nb,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double lo = h[0], hi = h[1], ma = h[2];
  for (int b = 1; b < nb; b++) {
    lo = std::fmin(lo, h[3 * b]);
    hi = std::fmax(hi, h[3 * b + 1]);
    ma = std::fmax(ma, h[3 * b + 2]);
  }
  out3[0] = lo; out3[1] = hi; out3[2] = ma;
  return VFCP_OK;
}

// ---- frame streaming (compress of a field still crossing PCIe)

int vfcp_value_range_part(const void* u, const void* v, int dtype, int64_t n,
                          double* part, int nb, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0 || nb <= 0) return fail(VFCP_EINVAL, "empty field");
  if (dtype == VFCP_F32)
    LAUNCH(K_RANGE, st, launch_range((const float*)u, (const float*)v, n, part, nb, st));
  else
    LAUNCH(K_RANGE, st, launch_range((const double*)u, (const double*)v, n, part, nb, st));
  return VFCP_OK;
}

int vfcp_analyze_slab(const vfcp_params* p, const void* u, const void* v,
                      int dtype, int t0, int t1, uint8_t* codes,
                      uint32_t* ld_words, uint16_t* mask, int32_t* row_n31,
                      uint64_t* list, int64_t cap, unsigned long long* count,
                      int* ovf, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (t0 < 0 || t1 > p->T || t0 >= t1)
    return fail(VFCP_EINVAL, "vfcp_analyze_slab: bad frame range");
  if (p->tau <= 0 || cap <= 0)
    return fail(VFCP_EINVAL, "vfcp_analyze_slab: needs tau' > 0 and a list");
  cudaStream_t st = (cudaStream_t)stream;
  const int nsm = nsm_of();
  if (dtype == VFCP_F32)
    LAUNCH(K_ANALYZE, st,
           launch_analyze_slab((const float*)u, (const float*)v, p->H, p->W,
                               p->T, t0, t1, p->scale, p->tau, codes, ld_words,
                               mask, row_n31, list, count, ovf,
                               (unsigned long long)cap, nsm, st));
  else
    LAUNCH(K_ANALYZE, st,
           launch_analyze_slab((const double*)u, (const double*)v, p->H, p->W,
                               p->T, t0, t1, p->scale, p->tau, codes, ld_words,
                               mask, row_n31, list, count, ovf,
                               (unsigned long long)cap, nsm, st));
  return VFCP_OK;
}

int vfcp_qd_offsets_upto(const vfcp_params* p, int nframes,
                         const int32_t* row_n31, int64_t* qd_row_off,
                         int64_t* total_dev_to_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (nframes < 1 || nframes > p->T)
    return fail(VFCP_EINVAL, "vfcp_qd_offsets_upto: bad frame count");
  const int64_t nrows = (int64_t)nframes * p->H;
  LAUNCH(K_SCAN, st, launch_row_scan(row_n31, nrows, p->W, 2, qd_row_off, st));
  CK(cudaMemcpyAsync(total_dev_to_host, qd_row_off + nrows, sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  return VFCP_OK;
}

int vfcp_encode_stream_begin(const vfcp_params* p, const void* u,
                             const void* v, int dtype, const uint8_t* codes,
                             const int64_t* qd_row_off, void* qd,
                             uint8_t* modes, int32_t* row_ll, void* stream,
                             void** handle) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!handle) return fail(VFCP_EINVAL, "null handle");
  *handle = nullptr;
  if (!fast_ok(p) || getenv("VFCP_SLOW_PATH"))
    return fail(VFCP_EINVAL,
                "vfcp_encode_stream: configuration outside the block path");
  cudaStream_t st = (cudaStream_t)stream;
  EncFramesBase* ef;
  if (dtype == VFCP_F32)
    ef = new EncFrames<float>(p, (const float*)u, (const float*)v, codes,
                              qd_row_off, (uint16_t*)qd, modes, row_ll,
                              nullptr, st);
  else
    ef = new EncFrames<double>(p, (const double*)u, (const double*)v, codes,
                               qd_row_off, (uint16_t*)qd, modes, row_ll,
                               nullptr, st);
  rc = ef->begin(false);
  if (rc) { delete ef; return rc; }
  *handle = ef;
  return VFCP_OK;
}

int vfcp_encode_stream_frame(void* handle, int t) {
  if (!handle) return fail(VFCP_EINVAL, "null handle");
  return static_cast<EncFramesBase*>(handle)->frame(t);
}

int vfcp_encode_stream_end(void* handle, int* overflowed) {
  if (!handle) return fail(VFCP_EINVAL, "null handle");
  EncFramesBase* ef = static_cast<EncFramesBase*>(handle);
  bool ovf = false;
  const int rc = ef->end(&ovf);
  if (overflowed) *overflowed = ovf ? 1 : 0;
  delete ef;
  return rc;
}

int vfcp_analyze(const vfcp_params* p, const void* u, const void* v,
                 int dtype, uint8_t* codes, uint32_t* ld_words,
                 uint16_t* mask, int32_t* row_n31, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t N = (int64_t)p->H * p->W * p->T;
  CK(cudaMemsetAsync(ld_words, 0, sizeof(uint32_t) * ((N + 31) / 32), st));
  CK(cudaMemsetAsync(row_n31, 0, sizeof(int32_t) * (size_t)p->T * p->H, st));
  // the anchors that need exact work (analyze.cu cube_kernel); a fuller
  // list falls back to the fused kernel
  const unsigned long long cap =
      (unsigned long long)std::min<int64_t>(N, (int64_t)1 << 25);
  Scratch sc(st);
  uint64_t* list;
  unsigned long long* count;
  int* ovf;
  CK(sc.get(&list, (size_t)cap));
  CK(sc.get(&count, 1));
  CK(sc.get(&ovf, 1));
  const int nsm = nsm_of();
  if (dtype == VFCP_F32)
    LAUNCH(K_ANALYZE, st,
           launch_analyze((const float*)u, (const float*)v, p->H, p->W, p->T,
                          p->scale, p->tau, codes, ld_words, mask, row_n31,
                          list, count, ovf, cap, nsm, st));
  else
    LAUNCH(K_ANALYZE, st,
           launch_analyze((const double*)u, (const double*)v, p->H, p->W,
                          p->T, p->scale, p->tau, codes, ld_words, mask,
                          row_n31, list, count, ovf, cap, nsm, st));
  return VFCP_OK;
}

int vfcp_qd_offsets(const vfcp_params* p, const int32_t* row_n31,
                    int64_t* qd_row_off, int64_t* total_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nrows = (int64_t)p->T * p->H;
  LAUNCH(K_SCAN, st, launch_row_scan(row_n31, nrows, p->W, 2, qd_row_off, st));
  CK(cudaMemcpyAsync(total_host, qd_row_off + nrows, sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VFCP_OK;
}

int vfcp_row_offsets(const int32_t* cnt, int64_t nrows, int64_t* off,
                     int64_t* total_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  LAUNCH(K_SCAN, st, launch_row_scan(cnt, nrows, 0, 1, off, st));
  CK(cudaMemcpyAsync(total_host, off + nrows, sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VFCP_OK;
}

int vfcp_encode(const vfcp_params* p, const void* u, const void* v,
                int dtype, const uint8_t* codes, const int64_t* qd_row_off,
                void* qd, uint8_t* modes, double* scores, int32_t* row_ll,
                int64_t* recon, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  HostOut ho;
  return encode_common(p, u, v, dtype, codes, qd_row_off, qd, modes, scores,
                       row_ll, recon, &ho, (cudaStream_t)stream);
}

int vfcp_encode_host(const vfcp_params* p, const void* u, const void* v,
                     int dtype, const uint8_t* codes,
                     const int64_t* qd_row_off, void* qd, uint8_t* modes,
                     int32_t* row_ll, void* host_qd,
                     const int64_t* frame_off, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!narrow_symbols(p->radius))
    return fail(VFCP_EINVAL, "vfcp_encode_host: radius > 32768");
  HostOut ho;
  ho.host_qd = (uint16_t*)host_qd;
  ho.frame_off = frame_off;
  return encode_common(p, u, v, dtype, codes, qd_row_off, qd, modes, nullptr,
                       row_ll, nullptr, &ho, (cudaStream_t)stream);
}

int vfcp_encode_ll(const vfcp_params* p, const void* u, const void* v,
                   int dtype, const uint8_t* codes, const void* qd,
                   const int64_t* qd_row_off, const int32_t* row_ll,
                   const int64_t* ll_row_off, int64_t* ll, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nrows = (int64_t)p->T * p->H;
  const bool ns = narrow_symbols(p->radius);
#define LLW(F, SYM)                                                         \
  LAUNCH(K_LLW, st, launch_ll_write<F, SYM>((const F*)u, (const F*)v, codes,               \
                             (const SYM*)qd, qd_row_off, row_ll,            \
                             ll_row_off, nrows, p->H, p->W, p->scale, ll,   \
                             st))
  if (dtype == VFCP_F32) { if (ns) LLW(float, uint16_t); else LLW(float, uint32_t); }
  else { if (ns) LLW(double, uint16_t); else LLW(double, uint32_t); }
#undef LLW
  return VFCP_OK;
}

int vfcp_decode_prepare(const vfcp_params* p, const uint8_t* codes,
                        const uint8_t* ld, const void* qd, int64_t n_qd,
                        int32_t* row_n31, int64_t* qd_row_off,
                        int32_t* row_ll, int64_t* ll_row_off,
                        int64_t* totals, int* ld_ok, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nrows = (int64_t)p->T * p->H;
  Scratch sc(st);
  int* bad;
  CK(sc.get(&bad, 1));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
  LAUNCH(K_DROWS, st, launch_decode_rows(codes, ld, nrows, p->W, p->tau, row_n31, bad, st));
  LAUNCH(K_SCAN, st, launch_row_scan(row_n31, nrows, p->W, 2, qd_row_off, st));
  int64_t nq = 0;
  int hbad = 0;
  CK(cudaMemcpyAsync(&nq, qd_row_off + nrows, sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  totals[0] = nq;
  *ld_ok = !hbad;
  totals[1] = 0;
  if (nq != n_qd) return VFCP_OK;   // caller raises the length error
  if (narrow_symbols(p->radius))
    LAUNCH(K_DLL, st, launch_decode_ll<uint16_t>((const uint16_t*)qd, qd_row_off, row_n31,
                                  nrows, row_ll, st));
  else
    LAUNCH(K_DLL, st, launch_decode_ll<uint32_t>((const uint32_t*)qd, qd_row_off, row_n31,
                                  nrows, row_ll, st));
  LAUNCH(K_SCAN, st, launch_row_scan(row_ll, nrows, 0, 1, ll_row_off, st));
  CK(cudaMemcpyAsync(totals + 1, ll_row_off + nrows, sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VFCP_OK;
}

static int decode_common(const vfcp_params* p, const uint8_t* codes,
                         const void* qd, int64_t n_qd, const int64_t* ll,
                         int64_t n_ll, const uint8_t* modes,
                         const int64_t* qd_row_off, const int64_t* ll_row_off,
                         double* out_u, double* out_v, int64_t* fix_u,
                         int64_t* fix_v, DecHostOut* ho, cudaStream_t st) {
  if (fast_ok(p) && !getenv("VFCP_SLOW_PATH")) {
    int rc = ho->init(p->T);
    if (rc) return rc;
    rc = decode_fast(p, codes, (const uint16_t*)qd, ll, modes, qd_row_off,
                     ll_row_off, out_u, out_v, fix_u, fix_v, st, ho);
    const int rf = ho->finish();
    return rc ? rc : rf;
  }
  const bool nf = narrow_frames(p->tau), ns = narrow_symbols(p->radius);
  int rc;
#define DEC(I, SYM)                                                          \
  rc = decode_impl<I, SYM>(p, codes, (const SYM*)qd, n_qd, ll, n_ll, modes,   \
                           qd_row_off, ll_row_off, out_u, out_v, fix_u,      \
                           fix_v, st)
  if (nf) { if (ns) DEC(int32_t, uint16_t); else DEC(int32_t, uint32_t); }
  else { if (ns) DEC(int64_t, uint16_t); else DEC(int64_t, uint32_t); }
#undef DEC
  if (rc || !ho->hu) return rc;
  // generic path: the whole output at the end
  const int64_t n = (int64_t)p->H * p->W * p->T;
  CK(cudaMemcpyAsync(ho->hu, out_u, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ho->hv, out_v, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VFCP_OK;
}

int vfcp_decode(const vfcp_params* p, const uint8_t* codes, const void* qd,
                int64_t n_qd, const int64_t* ll, int64_t n_ll,
                const uint8_t* modes,
                const int64_t* qd_row_off, const int64_t* ll_row_off,
                double* out_u, double* out_v, int64_t* fix_u, int64_t* fix_v,
                void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  DecHostOut ho;
  return decode_common(p, codes, qd, n_qd, ll, n_ll, modes, qd_row_off,
                       ll_row_off, out_u, out_v, fix_u, fix_v, &ho,
                       (cudaStream_t)stream);
}

int vfcp_decode_host(const vfcp_params* p, const uint8_t* codes,
                     const void* qd, int64_t n_qd, const int64_t* ll,
                     int64_t n_ll, const uint8_t* modes,
                     const int64_t* qd_row_off, const int64_t* ll_row_off,
                     double* out_u, double* out_v, double* host_u,
                     double* host_v, void* stream) {
  int rc = check_params(p);
  if (rc) return rc;
  if (!host_u || !host_v)
    return fail(VFCP_EINVAL, "vfcp_decode_host: null host buffer");
  DecHostOut ho;
  ho.hu = host_u;
  ho.hv = host_v;
  return decode_common(p, codes, qd, n_qd, ll, n_ll, modes, qd_row_off,
                       ll_row_off, out_u, out_v, nullptr, nullptr, &ho,
                       (cudaStream_t)stream);
}

}  // extern "C"
