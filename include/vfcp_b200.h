/*
 * vfcp_b200.h -- C ABI of the B200-native vfcp hot path.
 *
 * Drop-in boundary for the reference's numba kernel layer
 * (/root/reference/pkg/src/vfcp).  The reference binds these stages as
 * numba @njit functions over caller-allocated numpy arrays that are mutated
 * in place; this library exposes the same stages, coarsened
 * to whole-field / frame-streaming device calls over caller-allocated device
 * buffers.  Plain pointers and sizes only; `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Every call returns 0 on success or a negative
 * VFCP_E* code; vfcp_last_error() gives the message.
 *
 * Device-pointer calls are asynchronous on `stream` unless documented as
 * synchronising (they return host values).
 */
#ifndef VFCP_B200_H
#define VFCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VFCP_OK 0
#define VFCP_EINVAL -1      /* bad argument (reference raises ValueError) */
#define VFCP_ECUDA -2       /* CUDA runtime error */
#define VFCP_ECAPACITY -3   /* output buffer too small */
#define VFCP_ECORRUPT -4    /* archive content inconsistent */

#define VFCP_F32 0
#define VFCP_F64 1

#define VFCP_PRED_MOP 0     /* codec.py:41 PREDICTORS order */
#define VFCP_PRED_LORENZO 1
#define VFCP_PRED_SL 2

/* Codec settings (codec.py:44-68 Config + the archive header fields). */
typedef struct vfcp_params {
  int32_t H, W, T;
  double dx, dy, dt;
  double scale;        /* S, a power of two (field.py:300-310) */
  int64_t tau;         /* tau' = max(0, floor(eps*S - 0.5)) (codec.py:71-77) */
  int32_t predictor;   /* VFCP_PRED_* */
  int32_t bx, by, stride;
  int32_t radius;      /* |idx| < radius; symbols are uint16 iff radius <= 32768 */
  int32_t n_max;
  double lam, theta, d_max;
} vfcp_params;

const char* vfcp_last_error(void);
int vfcp_version(void);

/* Instrumentation: number of kernels this library has launched, and
 * per-kernel-class CUDA-event timings (classes: 0 range, 1 analyze, 2 scan,
 * 3 mop, 4 encode chain, 5 ll write / symbol scatter, 6 decode prep,
 * 7 decode ll, 8 decode chain, 9 aux (frame emit), 10 encode prep).
 * vfcp_prof_collect synchronises on the recorded events. */
int64_t vfcp_launch_count(void);
int vfcp_prof_enable(int on);
int vfcp_prof_collect(double* ms, int64_t* counts, int ncls);

/* field.py:69-73 FieldSeries.value_range and the max|x| of to_fixed
 * (field.py:322).  Synchronising: out3 = {min, max, max|x|} over u and v. */
int vfcp_value_range(const void* u, const void* v, int dtype, int64_t n,
                     double* out3, void* stream);

/* predicates.py:290-301 build_critical_face_set + ebounds.py:190-206
 * derive_all + codec.py:97-115 _quantize_eb_vec, fused.
 *   codes    u8[N]          eb ladder code per vertex (31 = lossless)
 *   ld_words u32[ceil(N/32)] l_d = (xi == 0) as np.packbits bytes
 *   mask     u16[N] or NULL positive-face classes per anchor vertex
 *            (bit c = class c in mesh.py:91-128 order)
 *   row_n31  i32[T*H]        code-31 vertices per frame row
 * u, v are float32 or float64 (dtype) device arrays of N = H*W*T. */
int vfcp_analyze(const vfcp_params* p, const void* u, const void* v,
                 int dtype, uint8_t* codes, uint32_t* ld_words,
                 uint16_t* mask, int32_t* row_n31, void* stream);

/* Exclusive row offsets of the qd symbol stream from row_n31:
 * qd_row_off[r] = 2 * sum_{q<r} (W - row_n31[q]), qd_row_off[T*H] = total.
 * Synchronising: *total_host = number of qd symbols. */
int vfcp_qd_offsets(const vfcp_params* p, const int32_t* row_n31,
                    int64_t* qd_row_off, int64_t* total_host, void* stream);

/* mop.py:154-173 select_modes + codec.py:118-164 _encode_frame over all
 * frames (codec.py:359-376).
 *   qd      u16 (or u32 when radius > 32768) symbols, capacity from
 *           vfcp_qd_offsets
 *   modes   u8[(T-1)*nby*nbx] per-block modes for t >= 1 (1 = SL)
 *   scores  f64[(T-1)*nby*nbx*2] or NULL: MoP rates [lorenzo, sl]
 *   row_ll  i32[T*H] lossless-stream entries per frame row
 *   recon   i64[2*N] or NULL: the encoder's reconstruction (u then v). */
int vfcp_encode(const vfcp_params* p, const void* u, const void* v,
                int dtype, const uint8_t* codes, const int64_t* qd_row_off,
                void* qd, uint8_t* modes, double* scores, int32_t* row_ll,
                int64_t* recon, void* stream);

/* vfcp_encode that also streams the symbol stream to (pinned) host memory
 * while it runs: frame t's symbols qd[frame_off[t] .. frame_off[t+1]) are
 * copied to host_qd on a side stream as soon as frame t is encoded, so the
 * D2H overlaps the later frames (the entropy stage of codec.py:378-387 reads
 * them on the host).  frame_off: host i64[T+1] = qd_row_off[t*H]. */
int vfcp_encode_host(const vfcp_params* p, const void* u, const void* v,
                     int dtype, const uint8_t* codes,
                     const int64_t* qd_row_off, void* qd, uint8_t* modes,
                     int32_t* row_ll, void* host_qd,
                     const int64_t* frame_off, void* stream);

/* ---- frame streaming: compress() of a field that is still crossing PCIe.
 * The reference's compress (codec.py:321-376) is value_range -> to_fixed ->
 * derive_all -> the frame loop; on a host-resident field the steps below let
 * frame t be analysed and encoded as soon as frames <= t + 1 are on the
 * device, while the later frames' H2D copies are in flight.             */

/* field.py:69-73 value_range + choose_scale's max|x| on HOST memory (u, v:
 * host arrays of n values), reduced by nthreads host threads: the scale and a
 * relative eps must be known before the first frame can be converted, i.e.
 * before the data has crossed PCIe.  out3 = {min, max, max|x|}.  Meant for
 * the spans the DMA delivers last (the device reduces the frames that have
 * arrived); a hint the device range (vfcp_value_range_part over every frame)
 * is checked against. */
int vfcp_host_range(const void* u, const void* v, int dtype, int64_t n,
                    int nthreads, double* out3);

/* The launch of vfcp_value_range without its host reduction: nb partial
 * {min, max, max|x|} triples of n values into device part[3 * nb]. */
int vfcp_value_range_part(const void* u, const void* v, int dtype, int64_t n,
                          double* part, int nb, void* stream);

/* vfcp_analyze restricted to the anchors of frames [t0, t1) (predicates.py:
 * 290-301 / ebounds.py:190-206 enumerate faces per anchor vertex; an anchor
 * of frame t touches frames t and t + 1 only).  Reads frames t0 ..
 * min(t1, T-1).  codes / ld_words / mask / row_n31 / *ovf must be zeroed
 * before the first slab; all updates are atomic max / or / first-touch
 * counts, so any partition of [0, T) into slabs leaves vfcp_analyze's
 * arrays.  Frame t's codes are final once the anchors of frames t - 1 and t
 * have run.  list: device u64[cap] scratch, count: device u64, ovf: device
 * int set when a slab's list overflowed (redo the field with vfcp_analyze).
 * Needs tau' > 0. */
int vfcp_analyze_slab(const vfcp_params* p, const void* u, const void* v,
                      int dtype, int t0, int t1, uint8_t* codes,
                      uint32_t* ld_words, uint16_t* mask, int32_t* row_n31,
                      uint64_t* list, int64_t cap, unsigned long long* count,
                      int* ovf, void* stream);

/* vfcp_qd_offsets over the rows of the first nframes frames (their counts
 * final); qd_row_off[nframes * H] also goes to *total (page-locked host
 * memory) asynchronously on `stream`. */
int vfcp_qd_offsets_upto(const vfcp_params* p, int nframes,
                         const int32_t* row_n31, int64_t* qd_row_off,
                         int64_t* total, void* stream);

/* vfcp_encode's frame loop (codec.py:359-376) one frame at a time: begin
 * allocates the scratch (block path only: VFCP_EINVAL otherwise, use
 * vfcp_encode), frame(t) enqueues frame t on the stream given to begin --
 * t = 0, 1, ... in order, each once orig(t), codes(t) and qd_row_off of its
 * rows are final in stream order -- and end synchronises, frees the handle
 * and reports whether an int32 overflow asks for vfcp_encode instead. */
int vfcp_encode_stream_begin(const vfcp_params* p, const void* u,
                             const void* v, int dtype, const uint8_t* codes,
                             const int64_t* qd_row_off, void* qd,
                             uint8_t* modes, int32_t* row_ll, void* stream,
                             void** handle);
int vfcp_encode_stream_frame(void* handle, int t);
int vfcp_encode_stream_end(void* handle, int* overflowed);

/* Exclusive scan of per-row counts: off[r] = sum_{q<r} cnt[q], off[nrows] =
 * total.  Synchronising: *total_host = total. */
int vfcp_row_offsets(const int32_t* cnt, int64_t nrows, int64_t* off,
                     int64_t* total_host, void* stream);

/* The lossless side stream of codec.py:129-131,155-158 in raster order. */
int vfcp_encode_ll(const vfcp_params* p, const void* u, const void* v,
                   int dtype, const uint8_t* codes, const void* qd,
                   const int64_t* qd_row_off, const int32_t* row_ll,
                   const int64_t* ll_row_off, int64_t* ll, void* stream);

/* Decoder stream bookkeeping (codec.py:404-413, 447-450).  Synchronising.
 *   ld       packed l_d bytes or NULL (checked against codes == 31)
 *   totals   host i64[2] = {qd symbols, ll values} the archive must hold
 *   ld_ok    host int: 0 if l_d disagrees with the eb codes. */
int vfcp_decode_prepare(const vfcp_params* p, const uint8_t* codes,
                        const uint8_t* ld, const void* qd, int64_t n_qd,
                        int32_t* row_n31, int64_t* qd_row_off,
                        int32_t* row_ll, int64_t* ll_row_off,
                        int64_t* totals, int* ld_ok, void* stream);

/* codec.py:401-453 decompress_with_stats frame loop (_decode_frame).
 *   qd, ll        the symbol / lossless streams and their lengths
 *   out_u, out_v  f64[N] reconstruction * (1/S)
 *   fix_u, fix_v  i64[N] or NULL: fixed-point reconstruction. */
int vfcp_decode(const vfcp_params* p, const uint8_t* codes, const void* qd,
                int64_t n_qd, const int64_t* ll, int64_t n_ll,
                const uint8_t* modes,
                const int64_t* qd_row_off, const int64_t* ll_row_off,
                double* out_u, double* out_v, int64_t* fix_u, int64_t* fix_v,
                void* stream);
/* vfcp_decode, and each frame's f64 output copied to host_u / host_v
 * (f64[N], page-locked for the copies to overlap the decode of later
 * frames) as soon as the frame is decoded; returns after the copies. */
int vfcp_decode_host(const vfcp_params* p, const uint8_t* codes,
                     const void* qd, int64_t n_qd, const int64_t* ll,
                     int64_t n_ll, const uint8_t* modes,
                     const int64_t* qd_row_off, const int64_t* ll_row_off,
                     double* out_u, double* out_v, double* host_u,
                     double* host_v, void* stream);

/* ---- host entropy backend (huffman.py), byte-identical to the reference */
/* huffman.py:21-48 code_lengths (heapq order, serial tie-break). */
int vfcp_huff_lengths(const int64_t* counts, int32_t alphabet, uint8_t* lens);
/* huffman.py:101-113 encode: symbol histogram over a host array of
 * sym_bytes-wide unsigned symbols. */
int vfcp_huff_count(const void* symbols, int sym_bytes, int64_t n,
                    int32_t alphabet, int64_t* counts);
/* huffman.py:51-76: canonical codes + MSB-first packing into out (zeroed,
 * ceil(bits/8) bytes).  Returns total bits in *bits. */
int vfcp_huff_pack(const void* symbols, int sym_bytes, int64_t n,
                   const uint8_t* lens, int32_t alphabet, uint8_t* out,
                   int64_t out_bytes, int64_t* bits, int threads);
/* huffman.py:116-149 decode into sym_bytes-wide symbols.  Returns
 * VFCP_ECORRUPT if the stream does not consume exactly total_bits. */
int vfcp_huff_unpack(const uint8_t* data, int64_t total_bits,
                     const uint8_t* lens, int32_t alphabet, int64_t n,
                     void* out, int sym_bytes);

/* Device-side entropy stage (huffman.py:16-76 encode): counts of
 * a device symbol array (sym_bytes 1 or 2) added into device u64
 * counts[alphabet]; wbase: the first bin of the shared-memory window (the
 * symbols' mode, e.g. radius - 4096 for the residual stream). */
int vfcp_huff_hist_dev(const void* symbols, int sym_bytes, int64_t n,
                       int32_t alphabet, int32_t wbase,
                       unsigned long long* counts, void* stream);

/* MSB-first canonical-Huffman bits of a device symbol array under the code
 * lengths lens_host (host, from vfcp_huff_lengths) into device out_words
 * (n_words >= ceil(total_bits / 32); zeroed here): the bytes are the
 * reference's _pack_bits output. */
int vfcp_huff_pack_dev(const void* symbols, int sym_bytes, int64_t n,
                       const uint8_t* lens_host, int32_t alphabet,
                       uint32_t* out_words, int64_t n_words, void* stream);

/* huffman.py:79-98 decode on the device: the packed bytes as 32-bit words
 * (device, n_words >= ceil(total_bits / 32) + 2, padding zero) -> n symbols
 * (sym_bytes 1 or 2) in device `out`.  Chunks of the stream are decoded in
 * parallel and resynchronised to the sequential decoder's codeword
 * boundaries.  VFCP_ECORRUPT for a stream the sequential decoder would not
 * consume exactly (the caller then decodes on the host for the reference's
 * exact error). */
int vfcp_huff_unpack_dev(const uint32_t* words, int64_t n_words,
                         int64_t total_bits, const uint8_t* lens_host,
                         int32_t alphabet, int64_t n, void* out,
                         int sym_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
