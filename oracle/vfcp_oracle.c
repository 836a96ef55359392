/*
 * vfcp_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference `vfcp` hot path
 * (/root/reference/pkg/src/vfcp, numba @njit kernels).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product (paper_2510_25143_b200) never links or calls it.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by running the reference itself
 * (oracle/gen_golden.py -> tests/golden/).
 *
 * Floating point: compiled with -ffp-contract=off and without fast-math so
 * every binary64 op is rounded individually, as numba/LLVM does.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>


#define CODE_LOSSLESS 31
#define K_MAX 30

/* ------------------------------------------------------------------ */
/* predictors.py:25-30  _rha                                          */
static inline int64_t rha(double x) {
    if (x >= 0.0) return (int64_t)floor(x + 0.5);
    return (int64_t)(-floor(-x + 0.5));
}

/* field.py:295-297 round_half_away on x*S, field.py:313-336 to_fixed.
 * dtype 0 = float32, 1 = float64.  Returns max |fixed|. */
int64_t or_to_fixed(const void *src, int dtype, int64_t n, double s,
                    int32_t *out) {
    int64_t m = 0;
    for (int64_t k = 0; k < n; k++) {
        double x = dtype == 0 ? (double)((const float *)src)[k]
                              : ((const double *)src)[k];
        double y = x * s;
        double a = floor(fabs(y) + 0.5);
        double sg = (y > 0.0) ? 1.0 : ((y < 0.0) ? -1.0 : 0.0);
        int64_t q = (int64_t)(sg * a);
        int64_t aq = q < 0 ? -q : q;
        if (aq > m) m = aq;
        out[k] = (int32_t)q; /* callers guarantee |q| < 2^30 */
    }
    return m;
}

/* field.py:69-73 value_range components: min, max, max|x| over both. */
void or_range(const void *u, const void *v, int dtype, int64_t n,
              double *out3) {
    double lo = INFINITY, hi = -INFINITY, ma = 0.0;
    for (int c = 0; c < 2; c++) {
        const void *p = c ? v : u;
        for (int64_t k = 0; k < n; k++) {
            double x = dtype == 0 ? (double)((const float *)p)[k]
                                  : ((const double *)p)[k];
            if (x < lo) lo = x;
            if (x > hi) hi = x;
            double a = fabs(x);
            if (a > ma) ma = a;
        }
    }
    out3[0] = lo; out3[1] = hi; out3[2] = ma;
}

/* ------------------------------------------------------------------ */
/* predicates.py:156-254 _sos_sign (compiled SoS orientation).        */
#define PAD (-(((int64_t)1) << 62))
static int sos_sign(int64_t x0, int64_t y0, int64_t x1, int64_t y1,
                    int64_t x2, int64_t y2, int64_t id0, int64_t id1,
                    int64_t id2) {
    int64_t det = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
    if (det > 0) return 1;
    if (det < 0) return -1;
    int64_t ids[3] = {id0, id1, id2}, xs[3] = {x0, x1, x2},
            ys[3] = {y0, y1, y2};
    int parity = 1;
    for (int i = 1; i < 3; i++) {
        int k = i;
        while (k > 0 && ids[k - 1] > ids[k]) {
            int64_t t;
            t = ids[k - 1]; ids[k - 1] = ids[k]; ids[k] = t;
            t = xs[k - 1]; xs[k - 1] = xs[k]; xs[k] = t;
            t = ys[k - 1]; ys[k - 1] = ys[k]; ys[k] = t;
            parity = -parity;
            k--;
        }
    }
    int64_t best0 = ((int64_t)1) << 62, best1 = 0, best2 = 0, best_coeff = 0;
    for (int c0 = -1; c0 < 2; c0++)
        for (int c1 = -1; c1 < 2; c1++)
            for (int c2 = -1; c2 < 2; c2++) {
                if (c0 == -1 && c1 == -1 && c2 == -1) continue;
                int64_t a0, a1, a2, b0, b1, b2, d0, d1, d2;
                if (c0 == -1) { a0 = xs[0]; a1 = ys[0]; a2 = 1; }
                else if (c0 == 0) { a0 = 1; a1 = 0; a2 = 0; }
                else { a0 = 0; a1 = 1; a2 = 0; }
                if (c1 == -1) { b0 = xs[1]; b1 = ys[1]; b2 = 1; }
                else if (c1 == 0) { b0 = 1; b1 = 0; b2 = 0; }
                else { b0 = 0; b1 = 1; b2 = 0; }
                if (c2 == -1) { d0 = xs[2]; d1 = ys[2]; d2 = 1; }
                else if (c2 == 0) { d0 = 1; d1 = 0; d2 = 0; }
                else { d0 = 0; d1 = 1; d2 = 0; }
                int64_t coeff = a0 * (b1 * d2 - b2 * d1) -
                                a1 * (b0 * d2 - b2 * d0) +
                                a2 * (b0 * d1 - b1 * d0);
                if (coeff == 0) continue;
                int64_t k0 = PAD, k1 = PAD, k2 = PAD;
                int nf = 0;
                if (c0 != -1) { k0 = 2 * ids[0] + c0; nf = 1; }
                if (c1 != -1) {
                    int64_t f = 2 * ids[1] + c1;
                    if (nf == 0) k0 = f; else k1 = f;
                    nf++;
                }
                if (c2 != -1) {
                    int64_t f = 2 * ids[2] + c2;
                    if (nf == 0) k0 = f; else if (nf == 1) k1 = f; else k2 = f;
                    nf++;
                }
                int64_t t;
                if (k1 > k0) { t = k0; k0 = k1; k1 = t; }
                if (k2 > k1) { t = k1; k1 = k2; k2 = t; }
                if (k1 > k0) { t = k0; k0 = k1; k1 = t; }
                int smaller = (k0 < best0) || (k0 == best0 && k1 < best1) ||
                              (k0 == best0 && k1 == best1 && k2 < best2);
                if (smaller) {
                    best0 = k0; best1 = k1; best2 = k2;
                    best_coeff = coeff;
                }
            }
    return best_coeff > 0 ? parity : -parity;
}

/* predicates.py:257-267 _face_cp_sos */
static int face_cp_sos(int64_t ua, int64_t va, int64_t ub, int64_t vb,
                       int64_t uc, int64_t vc, int64_t ida, int64_t idb,
                       int64_t idc) {
    int s = sos_sign(ua, va, ub, vb, uc, vc, ida, idb, idc);
    if (sos_sign(0, 0, ub, vb, uc, vc, -1, idb, idc) != s) return 0;
    if (sos_sign(ua, va, 0, 0, uc, vc, ida, -1, idc) != s) return 0;
    if (sos_sign(ua, va, ub, vb, 0, 0, ida, idb, -1) != s) return 0;
    return 1;
}

/* predicates.py:278-287 (body of _face_scan for one face) */
int or_face_positive(int64_t ua, int64_t va, int64_t ub, int64_t vb,
                     int64_t uc, int64_t vc, int64_t a, int64_t b,
                     int64_t c) {
    int64_t d1 = ua * vb - va * ub;
    int64_t d2 = ub * vc - vb * uc;
    int64_t d3 = uc * va - vc * ua;
    if (d1 != 0 && d2 != 0 && d3 != 0)
        return (d1 > 0 && d2 > 0 && d3 > 0) || (d1 < 0 && d2 < 0 && d3 < 0);
    return face_cp_sos(ua, va, ub, vb, uc, vc, a, b, c);
}

/* ------------------------------------------------------------------ */
/* ebounds.py:101-134 _edge_eb (floor division = Python //).          */
static inline int64_t floordiv(int64_t a, int64_t d) { /* d > 0 */
    int64_t q = a / d;
    if ((a % d != 0) && (a < 0)) q--;
    return q;
}
static inline int64_t i64abs(int64_t x) { return x < 0 ? -x : x; }
static inline int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

int64_t or_edge_eb(int64_t px, int64_t py, int64_t qx, int64_t qy) {
    int64_t dx = qx - px, dy = qy - py;
    int64_t best = i64max(i64abs(px), i64abs(py)) - 1;
    int64_t e1 = i64max(i64abs(qx), i64abs(qy)) - 1;
    if (e1 < best) best = e1;
    for (int which = 0; which < 4; which++) {
        int64_t n, d;
        if (which == 0) { if (dx == 0) continue; n = -px; d = dx; }
        else if (which == 1) { if (dy == 0) continue; n = -py; d = dy; }
        else if (which == 2) { if (dx == dy) continue; n = py - px; d = dx - dy; }
        else { if (dx + dy == 0) continue; n = -(px + py); d = dx + dy; }
        if (d < 0) { n = -n; d = -d; }
        if (0 <= n && n <= d) {
            int64_t a = i64max(i64abs(px * d + n * dx), i64abs(py * d + n * dy));
            int64_t e = floordiv(a - 1, d);
            if (e < best) best = e;
        }
    }
    return best;
}

/* ebounds.py:137-148 _eb_one */
int64_t or_face_eb(int64_t u0, int64_t v0, int64_t u1, int64_t v1,
                   int64_t u2, int64_t v2) {
    int64_t e = or_edge_eb(u0, v0, u1, v1);
    int64_t e1 = or_edge_eb(u1, v1, u2, v2);
    if (e1 < e) e = e1;
    e1 = or_edge_eb(u2, v2, u0, v0);
    if (e1 < e) e = e1;
    if (e < 0) e = 0;
    return e;
}

/* ------------------------------------------------------------------ */
/* mesh.py:91-128 face classes, as (anchor range, offsets).  Class order
 * is the reference's enumeration order; bit c of a face mask = class c.
 * Offsets are (dt, di, dj) of vertices a<b<c from the anchor.          */
static const int CLS_OFF[12][3][3] = {
    {{0, 0, 0}, {0, 1, 0}, {0, 1, 1}}, /* slice_lower */
    {{0, 0, 0}, {0, 0, 1}, {0, 1, 1}}, /* slice_upper */
    {{0, 0, 0}, {0, 0, 1}, {1, 0, 1}}, /* wall_h1 */
    {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}}, /* wall_h2 */
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 0}}, /* wall_v1 */
    {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}}, /* wall_v2 */
    {{0, 0, 0}, {0, 1, 1}, {1, 1, 1}}, /* wall_d1 */
    {{0, 0, 0}, {1, 0, 0}, {1, 1, 1}}, /* wall_d2 */
    {{0, 0, 0}, {0, 1, 0}, {1, 1, 1}}, /* int_lower_a */
    {{0, 0, 0}, {1, 1, 0}, {1, 1, 1}}, /* int_lower_b */
    {{0, 0, 0}, {0, 0, 1}, {1, 1, 1}}, /* int_upper_a */
    {{0, 0, 0}, {1, 0, 1}, {1, 1, 1}}, /* int_upper_b */
};
/* anchor range limits: (t_lim, i_lim, j_lim) meaning anchor t < T - t_lim,
 * i < H - i_lim, j < W - j_lim. */
static const int CLS_LIM[12][3] = {
    {0, 1, 1}, {0, 1, 1},            /* slice: all t, cells */
    {1, 0, 1}, {1, 0, 1},            /* wall_h: t<T-1, j<W-1 */
    {1, 1, 0}, {1, 1, 0},            /* wall_v: t<T-1, i<H-1 */
    {1, 1, 1}, {1, 1, 1},            /* wall_d */
    {1, 1, 1}, {1, 1, 1}, {1, 1, 1}, {1, 1, 1}, /* internal */
};

/* predicates.py:290-301 build_critical_face_set as a 12-bit mask per
 * anchor vertex (mask[anchor] bit c set <=> face of class c positive).
 * ebounds.py:190-206 derive_all -> xi, then codec.py:338 codes.
 * Outputs (any may be NULL): mask u16[N], xi i64[N]. */
void or_analyze_window(int H, int W, int T, const int32_t *u,
                       const int32_t *v, int64_t tau, int ta0, int ta1,
                       uint16_t *mask, int64_t *xi);
void or_analyze(int H, int W, int T, const int32_t *u, const int32_t *v,
                int64_t tau, uint16_t *mask, int64_t *xi) {
    or_analyze_window(H, W, T, u, v, tau, 0, T, mask, xi);
}

/* The same scan restricted to anchors in frames [ta0, ta1) of a window of
 * T frames (window-local ids keep the reference's id order, which is all
 * SoS uses: SURVEY V5).  The xi of a frame-t vertex needs the anchors of
 * frames t-1 and t; the mask of frame t's anchors needs frames t, t+1.
 * Used by the full-size parity driver (tests/parity_full.py). */
void or_analyze_window(int H, int W, int T, const int32_t *u,
                       const int32_t *v, int64_t tau, int ta0, int ta1,
                       uint16_t *mask, int64_t *xi) {
    int64_t hw = (int64_t)H * W, n = hw * T;
    if (mask) memset(mask, 0, sizeof(uint16_t) * n);
    if (xi) for (int64_t k = 0; k < n; k++) xi[k] = tau;
    /* Reference order: all faces of a class, positives zero xi at the end
     * (ebounds.py:203-205); xi scatter-min is order independent. */
    uint8_t *pos_v = NULL;
    if (xi) pos_v = (uint8_t *)calloc((size_t)n, 1);
    for (int c = 0; c < 12; c++) {
        int tl = T - CLS_LIM[c][0], il = H - CLS_LIM[c][1],
            jl = W - CLS_LIM[c][2];
        int64_t oa = CLS_OFF[c][0][0] * hw + CLS_OFF[c][0][1] * W + CLS_OFF[c][0][2];
        int64_t ob = CLS_OFF[c][1][0] * hw + CLS_OFF[c][1][1] * W + CLS_OFF[c][1][2];
        int64_t oc = CLS_OFF[c][2][0] * hw + CLS_OFF[c][2][1] * W + CLS_OFF[c][2][2];
        for (int t = ta0; t < tl && t < ta1; t++)
            for (int i = 0; i < il; i++)
                for (int j = 0; j < jl; j++) {
                    int64_t an = t * hw + (int64_t)i * W + j;
                    int64_t a = an + oa, b = an + ob, cc = an + oc;
                    int64_t ua = u[a], va = v[a], ub = u[b], vb = v[b],
                            uc = u[cc], vc = v[cc];
                    int p = or_face_positive(ua, va, ub, vb, uc, vc, a, b, cc);
                    if (p) {
                        if (mask) mask[an] |= (uint16_t)(1u << c);
                        if (pos_v) { pos_v[a] = 1; pos_v[b] = 1; pos_v[cc] = 1; }
                    }
                    if (xi) {
                        int64_t e = or_face_eb(ua, va, ub, vb, uc, vc);
                        if (e < xi[a]) xi[a] = e;
                        if (e < xi[b]) xi[b] = e;
                        if (e < xi[cc]) xi[cc] = e;
                    }
                }
    }
    if (xi) {
        for (int64_t k = 0; k < n; k++)
            if (pos_v[k]) xi[k] = 0;
        free(pos_v);
    }
}

/* codec.py:80-90 quantize_eb (scalar; test_codec.py:48-58 pins it equal to
 * the vectorised _quantize_eb_vec used by compress). */
int or_quantize_eb(int64_t xi, int64_t tau) {
    if (tau <= 0 || xi <= 0) return CODE_LOSSLESS;
    if (xi >= tau) return 0;
    int64_t m = (tau + xi - 1) / xi;
    uint64_t mm = (uint64_t)(m - 1);
    int k = 0;
    while (mm) { k++; mm >>= 1; }
    if (k > K_MAX || (tau >> k) == 0) return CODE_LOSSLESS;
    return k;
}

void or_codes(const int64_t *xi, int64_t n, int64_t tau, uint8_t *codes,
              uint8_t *lossless) {
    for (int64_t k = 0; k < n; k++) {
        codes[k] = (uint8_t)or_quantize_eb(xi[k], tau);
        if (lossless) lossless[k] = xi[k] == 0;
    }
}

/* ------------------------------------------------------------------ */
/* predictors.py:33-59 _bilinear                                       */
static int64_t bilinear(const int64_t *f, int H, int W, double i_f,
                        double j_f) {
    if (i_f < 0.0) i_f = 0.0;
    else if (i_f > H - 1) i_f = (double)(H - 1);
    if (j_f < 0.0) j_f = 0.0;
    else if (j_f > W - 1) j_f = (double)(W - 1);
    int64_t i0 = (int64_t)floor(i_f), j0 = (int64_t)floor(j_f);
    if (i0 > H - 1) i0 = H - 1;
    if (j0 > W - 1) j0 = W - 1;
    int64_t i1 = i0 + 1 < H - 1 ? i0 + 1 : H - 1;
    int64_t j1 = j0 + 1 < W - 1 ? j0 + 1 : W - 1;
    double a = i_f - (double)i0, b = j_f - (double)j0;
    double val = (1.0 - a) * (1.0 - b) * (double)f[i0 * W + j0];
    val = val + (1.0 - a) * b * (double)f[i0 * W + j1];
    val = val + a * (1.0 - b) * (double)f[i1 * W + j0];
    val = val + a * b * (double)f[i1 * W + j1];
    return rha(val);
}

/* predictors.py:62-73 _lorenzo3d */
static inline int64_t lorenzo3d(const int64_t *cur, const int64_t *prev,
                                int W, int i, int j) {
    int64_t p = 0;
    int64_t k = (int64_t)i * W + j;
    if (i > 0) p += cur[k - W] - prev[k - W];
    if (j > 0) p += cur[k - 1] - prev[k - 1];
    p += prev[k];
    if (i > 0 && j > 0) p += prev[k - W - 1] - cur[k - W - 1];
    return p;
}

/* predictors.py:76-108 _sl_departure */
static void sl_departure(const int64_t *up, const int64_t *vp, int H, int W,
                         int i, int j, double cfl_x, double cfl_y,
                         double d_max, int64_t n_max, double *oi,
                         double *oj) {
    int64_t k = (int64_t)i * W + j;
    double u0 = (double)up[k], v0 = (double)vp[k];
    double dxx = fabs(u0) * cfl_x, dyy = fabs(v0) * cfl_y;
    double d_inf = dxx > dyy ? dxx : dyy; /* max(a, b) */
    if (d_inf <= d_max) {
        double ih = (double)i - 0.5 * v0 * cfl_y;
        double jh = (double)j - 0.5 * u0 * cfl_x;
        double um = (double)bilinear(up, H, W, ih, jh);
        double vm = (double)bilinear(vp, H, W, ih, jh);
        *oi = (double)i - vm * cfl_y;
        *oj = (double)j - um * cfl_x;
        return;
    }
    int64_t n = (int64_t)ceil(d_inf / d_max);
    if (n > n_max) n = n_max;
    double fi = (double)i, fj = (double)j;
    for (int64_t s = 0; s < n; s++) {
        double us = (double)bilinear(up, H, W, fi, fj);
        double vs = (double)bilinear(vp, H, W, fi, fj);
        fi -= vs * cfl_y / (double)n;
        fj -= us * cfl_x / (double)n;
        if (fi < 0.0) fi = 0.0;
        else if (fi > H - 1) fi = (double)(H - 1);
        if (fj < 0.0) fj = 0.0;
        else if (fj > W - 1) fj = (double)(W - 1);
    }
    *oi = fi; *oj = fj;
}

/* Python's max(a, b) returns a unless b > a; NaN-free here. */

/* ------------------------------------------------------------------ */
/* mop.py:68-151 _score_frame.  scores: (nby, nbx, 2) f64.  log2 is libm's
 * (numba lowers math.log2 to it). */
void or_score_frame(int H, int W, const int64_t *uo, const int64_t *vo,
                    const int64_t *up, const int64_t *vp, int64_t tau,
                    int64_t radius, int stride, int bx, int by, double lam,
                    double rmeta, double theta, double cfl_x, double cfl_y,
                    double d_max, int64_t n_max, uint8_t *modes,
                    double *scores) {
    int nby = (H + by - 1) / by, nbx = (W + bx - 1) / bx;
    int64_t hw = (int64_t)H * W;
    int64_t *cu = (int64_t *)malloc(sizeof(int64_t) * hw);
    int64_t *cv = (int64_t *)malloc(sizeof(int64_t) * hw);
    memcpy(cu, uo, sizeof(int64_t) * hw);
    memcpy(cv, vo, sizeof(int64_t) * hw);
    int64_t *hist = (int64_t *)calloc((size_t)radius, sizeof(int64_t));
    int64_t *touched = (int64_t *)malloc(sizeof(int64_t) * 2 * bx * by);
    int64_t two_tau = 2 * tau;
    for (int bi = 0; bi < nby; bi++) {
        int r0 = bi * by, r1 = r0 + by < H ? r0 + by : H;
        for (int bj = 0; bj < nbx; bj++) {
            int c0 = bj * bx, c1 = c0 + bx < W ? c0 + bx : W;
            for (int mode = 0; mode < 2; mode++) {
                int64_t nt = 0, lp = 0, n_ok = 0;
                double acc = 0.0;
                for (int i = r0; i < r1; i++)
                    for (int j = c0; j < c1; j++) {
                        double fi = 0.0, fj = 0.0;
                        if (mode == 1)
                            sl_departure(up, vp, H, W, i, j, cfl_x, cfl_y,
                                         d_max, n_max, &fi, &fj);
                        int sample = ((i - r0) % stride == 0) &&
                                     ((j - c0) % stride == 0);
                        int64_t k = (int64_t)i * W + j;
                        for (int comp = 0; comp < 2; comp++) {
                            int64_t orig = comp == 0 ? uo[k] : vo[k];
                            int64_t pred;
                            if (mode == 1)
                                pred = bilinear(comp == 0 ? up : vp, H, W, fi, fj);
                            else
                                pred = lorenzo3d(comp == 0 ? cu : cv,
                                                 comp == 0 ? up : vp, W, i, j);
                            int64_t r = orig - pred;
                            int64_t idx = rha((double)r / (double)two_tau);
                            int ok = (-radius < idx && idx < radius &&
                                      i64abs(r - idx * two_tau) <= tau);
                            if (mode == 0) {
                                int64_t rec = ok ? pred + idx * two_tau : orig;
                                if (comp == 0) cu[k] = rec; else cv[k] = rec;
                            }
                            if (sample) {
                                if (ok) {
                                    int64_t a = i64abs(idx);
                                    if (hist[a] == 0) touched[nt++] = a;
                                    hist[a] += 1;
                                    n_ok += 1;
                                } else {
                                    lp += 1;
                                }
                            }
                        }
                    }
                double h0 = 0.0;
                if (n_ok > 0) {
                    for (int64_t q = 0; q < nt; q++) {
                        double h = (double)hist[touched[q]];
                        acc += h * log2(h);
                    }
                    h0 = log2((double)n_ok) - acc / (double)n_ok;
                }
                double rate;
                if (n_ok + lp > 0)
                    rate = h0 + lam * (double)lp / (double)(n_ok + lp) + rmeta;
                else
                    rate = rmeta;
                scores[((int64_t)bi * nbx + bj) * 2 + mode] = rate;
                for (int64_t q = 0; q < nt; q++) hist[touched[q]] = 0;
                if (mode == 0)
                    for (int i = r0; i < r1; i++)
                        for (int j = c0; j < c1; j++) {
                            int64_t k = (int64_t)i * W + j;
                            cu[k] = uo[k]; cv[k] = vo[k];
                        }
            }
            double r_lor = scores[((int64_t)bi * nbx + bj) * 2 + 0];
            double r_sl = scores[((int64_t)bi * nbx + bj) * 2 + 1];
            modes[(int64_t)bi * nbx + bj] =
                (r_lor > 0.0 && (r_lor - r_sl) / r_lor > theta) ? 1 : 0;
        }
    }
    free(cu); free(cv); free(hist); free(touched);
}

/* ------------------------------------------------------------------ */
/* codec.py:118-164 _encode_frame.  Returns new positions via pointers. */
void or_encode_frame(int H, int W, const int64_t *uo, const int64_t *vo,
                     const int64_t *up, const int64_t *vp, int64_t *cu,
                     int64_t *cv, const int64_t *eq, const uint8_t *modes,
                     int use_modes, int by, int bx, double cfl_x,
                     double cfl_y, double d_max, int64_t n_max,
                     int64_t radius, int32_t *qd, int64_t *qd_pos,
                     int64_t *ll, int64_t *ll_pos) {
    int nbx = (W + bx - 1) / bx;
    int64_t qp = *qd_pos, lp = *ll_pos;
    for (int i = 0; i < H; i++)
        for (int j = 0; j < W; j++) {
            int64_t k = (int64_t)i * W + j;
            int64_t e = eq[k];
            if (e == 0) {
                cu[k] = uo[k]; cv[k] = vo[k];
                ll[lp] = uo[k]; ll[lp + 1] = vo[k];
                lp += 2;
                continue;
            }
            int sl = use_modes && modes[(int64_t)(i / by) * nbx + j / bx] == 1;
            double fi = 0.0, fj = 0.0;
            if (sl)
                sl_departure(up, vp, H, W, i, j, cfl_x, cfl_y, d_max, n_max,
                             &fi, &fj);
            int64_t two_e = 2 * e;
            for (int comp = 0; comp < 2; comp++) {
                int64_t orig = comp == 0 ? uo[k] : vo[k];
                int64_t pred;
                if (sl)
                    pred = bilinear(comp == 0 ? up : vp, H, W, fi, fj);
                else
                    pred = comp == 0 ? lorenzo3d(cu, up, W, i, j)
                                     : lorenzo3d(cv, vp, W, i, j);
                int64_t r = orig - pred;
                int64_t idx = rha((double)r / (double)two_e);
                int64_t rec;
                if (-radius < idx && idx < radius &&
                    i64abs(r - idx * two_e) <= e) {
                    qd[qp] = (int32_t)(idx + radius);
                    rec = pred + idx * two_e;
                } else {
                    qd[qp] = 0;
                    rec = orig;
                    ll[lp++] = orig;
                }
                qp++;
                if (comp == 0) cu[k] = rec; else cv[k] = rec;
            }
        }
    *qd_pos = qp; *ll_pos = lp;
}

/* codec.py:167-206 _decode_frame */
void or_decode_frame(int H, int W, const int64_t *up, const int64_t *vp,
                     int64_t *cu, int64_t *cv, const int64_t *eq,
                     const uint8_t *modes, int use_modes, int by, int bx,
                     double cfl_x, double cfl_y, double d_max, int64_t n_max,
                     int64_t radius, const int32_t *qd, int64_t *qd_pos,
                     const int64_t *ll, int64_t *ll_pos) {
    int nbx = (W + bx - 1) / bx;
    int64_t qp = *qd_pos, lp = *ll_pos;
    for (int i = 0; i < H; i++)
        for (int j = 0; j < W; j++) {
            int64_t k = (int64_t)i * W + j;
            int64_t e = eq[k];
            if (e == 0) {
                cu[k] = ll[lp]; cv[k] = ll[lp + 1];
                lp += 2;
                continue;
            }
            int sl = use_modes && modes[(int64_t)(i / by) * nbx + j / bx] == 1;
            double fi = 0.0, fj = 0.0;
            if (sl)
                sl_departure(up, vp, H, W, i, j, cfl_x, cfl_y, d_max, n_max,
                             &fi, &fj);
            int64_t two_e = 2 * e;
            for (int comp = 0; comp < 2; comp++) {
                int64_t pred;
                if (sl)
                    pred = bilinear(comp == 0 ? up : vp, H, W, fi, fj);
                else
                    pred = comp == 0 ? lorenzo3d(cu, up, W, i, j)
                                     : lorenzo3d(cv, vp, W, i, j);
                int64_t sym = qd[qp++];
                int64_t rec;
                if (sym == 0) rec = ll[lp++];
                else rec = pred + (sym - radius) * two_e;
                if (comp == 0) cu[k] = rec; else cv[k] = rec;
            }
        }
    *qd_pos = qp; *ll_pos = lp;
}

/* Scalar exports for unit tests of the primitives. */
int64_t or_rha(double x) { return rha(x); }
int64_t or_bilinear(const int64_t *f, int H, int W, double i_f, double j_f) {
    return bilinear(f, H, W, i_f, j_f);
}
void or_sl_departure(const int64_t *up, const int64_t *vp, int H, int W,
                     int i, int j, double cfl_x, double cfl_y, double d_max,
                     int64_t n_max, double *out2) {
    sl_departure(up, vp, H, W, i, j, cfl_x, cfl_y, d_max, n_max, &out2[0],
                 &out2[1]);
}
int or_sos_sign(int64_t x0, int64_t y0, int64_t x1, int64_t y1, int64_t x2,
                int64_t y2, int64_t id0, int64_t id1, int64_t id2) {
    return sos_sign(x0, y0, x1, y1, x2, y2, id0, id1, id2);
}
