// Device-side entropy stage: the symbol histogram and the
// MSB-first canonical-Huffman bit packing of huffman.py:16-76 (encode) on
// the GPU.  The code lengths stay on the host (vfcp_huff_lengths restates the
// reference's heap order exactly); the packed bytes are identical to the
// reference's _pack_bits output.
//
//   vfcp_huff_hist_dev   counts[alphabet] (+=) of a device symbol array:
//                        per-CTA shared-memory window of HW_BINS bins around
//                        `wbase` (the symbols' mode) with warp-aggregated
//                        atomics, global atomics outside the window
//   vfcp_huff_pack_dev   per chunk of HP_CHUNK symbols: bits of the chunk
//                        (pass 1), exclusive scan over chunks (CUB), then
//                        every thread appends the canonical codewords of
//                        its HP_PER symbols to a 64-bit MSB-first buffer and
//                        emits 32-bit big-endian words: plain stores for the
//                        words it owns, atomicOr for the (at most two) words
//                        it shares with its neighbours
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vfcp_b200.h"

namespace vfcp {

constexpr int HW_BINS = 8192;
constexpr int HP_T = 256;
constexpr int HP_PER = 64;
constexpr int HP_CHUNK = HP_T * HP_PER;

template <typename S>
__global__ void __launch_bounds__(256)
huff_hist_kernel(const S* __restrict__ sym, int64_t n, int wbase,
                 unsigned long long* __restrict__ counts) {
  __shared__ unsigned int h[HW_BINS];
  for (int k = threadIdx.x; k < HW_BINS; k += blockDim.x) h[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // 16 bytes of symbols per thread and step (the eight / sixteen match
  // operations of a step are independent, so their latencies overlap)
  constexpr int VPT = 16 / (int)sizeof(S);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * VPT;
  const bool aligned = ((uintptr_t)sym & 15) == 0;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x * VPT; i0 < n; i0 += stride) {
    const int64_t i = i0 + (int64_t)threadIdx.x * VPT;   // warp-uniform loop bound
    int sv[VPT];
    if (aligned && i + VPT <= n) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(sym + i));
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < VPT; k++)
        sv[k] = sizeof(S) == 2 ? (int)((w[k >> 1] >> (16 * (k & 1))) & 0xffffu)
                               : (int)((w[k >> 2] >> (8 * (k & 3))) & 0xffu);
    } else {
#pragma unroll
      for (int k = 0; k < VPT; k++) sv[k] = i + k < n ? (int)sym[i + k] : -1;
    }
#pragma unroll
    for (int k = 0; k < VPT; k++) {
      const int s = sv[k];
      const unsigned grp = __match_any_sync(0xffffffffu, s);
      const bool leader = s >= 0 && (grp & ((1u << lane) - 1u)) == 0;
      if (leader) {
        const int w = s - wbase;
        if ((unsigned)w < (unsigned)HW_BINS) atomicAdd(&h[w], (unsigned)__popc(grp));
        else atomicAdd(&counts[s], (unsigned long long)__popc(grp));
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < HW_BINS; k += blockDim.x)
    if (h[k]) atomicAdd(&counts[wbase + k], (unsigned long long)h[k]);
}

// pass 1: bits per chunk
template <typename S>
__global__ void __launch_bounds__(HP_T)
huff_bits_kernel(const S* __restrict__ sym, int64_t n,
                 const uint8_t* __restrict__ lens,
                 unsigned long long* __restrict__ chunk_bits) {
  typedef cub::BlockReduce<unsigned long long, HP_T> BR;
  __shared__ typename BR::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * HP_CHUNK;
  unsigned long long b = 0;
  for (int k = threadIdx.x; k < HP_CHUNK; k += HP_T) {
    const int64_t i = base + k;
    if (i < n) b += __ldg(lens + sym[i]);
  }
  const unsigned long long tot = BR(tmp).Sum(b);
  if (threadIdx.x == 0) chunk_bits[blockIdx.x] = tot;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) {
  return __byte_perm(x, 0, 0x0123);
}

// pass 2: pack (out: 32-bit words, zeroed)
template <typename S>
__global__ void __launch_bounds__(HP_T)
huff_pack_kernel(const S* __restrict__ sym, int64_t n,
                 const uint8_t* __restrict__ lens,
                 const unsigned long long* __restrict__ codes,
                 const unsigned long long* __restrict__ chunk_off,
                 uint32_t* __restrict__ out) {
  typedef cub::BlockScan<unsigned long long, HP_T> BS;
  __shared__ typename BS::TempStorage tmp;
  // the CTA's symbols staged in shared memory with coalesced 16-byte loads,
  // one padded row per thread (its HP_PER consecutive symbols), read back
  // 16 bytes at a time without bank conflicts
  constexpr int ROWB = HP_PER * (int)sizeof(S);
  constexpr int PADB = ROWB + 16;
  constexpr int V = 16 / (int)sizeof(S);
  __shared__ __align__(16) unsigned char ss[HP_T * PADB];
  const int64_t cbase = (int64_t)blockIdx.x * HP_CHUNK;
  const int count = (int)min((int64_t)HP_CHUNK, n - cbase);
  if (count == HP_CHUNK && ((uintptr_t)(sym + cbase) & 15) == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(sym + cbase);
    for (int q = threadIdx.x; q < HP_CHUNK * (int)sizeof(S) / 16; q += HP_T)
      *reinterpret_cast<uint4*>(ss + (q / (ROWB / 16)) * PADB + (q % (ROWB / 16)) * 16) =
          __ldg(src + q);
  } else {
    for (int e = threadIdx.x; e < count; e += HP_T)
      reinterpret_cast<S*>(ss + (e / HP_PER) * PADB)[e % HP_PER] = sym[cbase + e];
  }
  __syncthreads();
  const unsigned char* row = ss + threadIdx.x * PADB;
  const int cnt = max(0, min(HP_PER, count - (int)threadIdx.x * HP_PER));
  auto sym_at = [&](const uint4& q, int i) -> int {   // i-th symbol of a piece
    const uint32_t wd = i < V / 4 ? q.x : i < V / 2 ? q.y : i < 3 * V / 4 ? q.z : q.w;
    const int sh = (i % (V / 4)) * 8 * (int)sizeof(S);
    return (int)((wd >> sh) & (sizeof(S) == 1 ? 0xffu : 0xffffu));
  };
  unsigned long long mine = 0;
  for (int k0 = 0; k0 < cnt; k0 += V) {
    const uint4 q = *reinterpret_cast<const uint4*>(row + k0 * (int)sizeof(S));
#pragma unroll
    for (int i = 0; i < V; i++)
      if (k0 + i < cnt) mine += __ldg(lens + sym_at(q, i));
  }
  unsigned long long off;
  BS(tmp).ExclusiveSum(mine, off);
  if (cnt == 0 || mine == 0) return;
  const unsigned long long p0 = chunk_off[blockIdx.x] + off;
  int64_t wi = (int64_t)(p0 >> 5);          // word being filled
  int nb = (int)(p0 & 31);                  // bits of it before ours (zero)
  unsigned long long buf = 0;               // MSB-first, nb bits valid
  bool first_word = true;
  auto emit_full = [&]() {
    while (nb >= 32) {
      const uint32_t w = bswap32((uint32_t)(buf >> 32));
      if (first_word) atomicOr(out + wi, w);
      else out[wi] = w;
      first_word = false;
      buf <<= 32;
      nb -= 32;
      wi++;
    }
  };
  auto append = [&](unsigned long long c, int L) {   // L <= 32, nb < 32
    buf |= c << (64 - nb - L);
    nb += L;
    emit_full();
  };
  for (int k0 = 0; k0 < cnt; k0 += V) {
    const uint4 q = *reinterpret_cast<const uint4*>(row + k0 * (int)sizeof(S));
#pragma unroll
    for (int i = 0; i < V; i++) {
      if (k0 + i >= cnt) break;
      const int s = sym_at(q, i);
      const int L = __ldg(lens + s);
      const unsigned long long c = __ldg(codes + s);
      if (L > 32) {
        append(c >> 32, L - 32);
        append(c & 0xffffffffull, 32);
      } else if (L > 0) {
        append(c, L);
      }
    }
  }
  if (nb > 0) atomicOr(out + wi, bswap32((uint32_t)(buf >> 32)));
}

// ------------------------------------------------------------- decode
// huffman.py:79-98 (_unpack_bits) in parallel: the bitstream is cut into
// chunks of HD_CB bits; a thread decodes its chunk from a start position
// until the first codeword boundary at or past the chunk end (its exit).
// The true start of chunk k+1 is the exit of chunk k decoded from its true
// start; starting from the chunk boundaries and re-decoding every chunk
// whose start moved converges quickly (Huffman codes resynchronise within a
// few codewords), and reproduces the sequential decoder's codeword
// boundaries exactly.  Then the per-chunk counts are scanned and every chunk
// writes its symbols.
constexpr int HD_CB = 1024;      // bits per chunk
constexpr int HD_LB = 12;        // lookup-table bits

struct HuffDecTables {
  const uint32_t* lut;           // [1 << lb]: (symbol << 8) | length, 0: long
  const uint32_t* symtab;        // symbols by (length, symbol)
  int64_t first_code[64];
  int64_t count_at[64];
  int64_t offset_at[64];
  int lb, max_len;
};

// 64 bits of the big-endian stream from bit p (words: bswapped 32-bit)
__device__ __forceinline__ unsigned long long hd_window(const uint32_t* w,
                                                        int64_t p) {
  const int64_t wi = p >> 5;
  const int o = (int)(p & 31);
  const unsigned long long a = ((unsigned long long)bswap32(__ldg(w + wi)) << 32) |
                               bswap32(__ldg(w + wi + 1));
  if (o == 0) return a;
  return (a << o) | (bswap32(__ldg(w + wi + 2)) >> (32 - o));
}

// one codeword at p: returns its length (0: invalid) and the symbol
__device__ __forceinline__ int hd_step(const HuffDecTables& t, const uint32_t* lut,
                                       const uint32_t* w, int64_t p,
                                       uint32_t* sym) {
  const unsigned long long win = hd_window(w, p);
  const uint32_t e = lut[win >> (64 - t.lb)];
  if (e) {
    *sym = e >> 8;
    return (int)(e & 255u);
  }
  for (int L = t.lb + 1; L <= t.max_len; L++) {
    if (t.count_at[L] == 0) continue;
    const int64_t d = (int64_t)(win >> (64 - L)) - t.first_code[L];
    if (d >= 0 && d < t.count_at[L]) {
      *sym = __ldg(t.symtab + t.offset_at[L] + d);
      return L;
    }
  }
  return 0;
}

// A decoding cursor over one chunk: a 64-bit window of the stream held in
// registers and refilled when fewer than 32 of its bits are left (the
// table needs lb <= 12 valid bits), so a short codeword costs a shared-
// memory lookup and two shifts, not three global loads.
struct HdCursor {
  unsigned long long buf;
  int avail;
  int64_t p;
  // next codeword: its length (0: invalid) and symbol
  __device__ __forceinline__ int next(const HuffDecTables& t, const uint32_t* lut,
                                      const uint32_t* w, uint32_t* sym) {
    if (avail < 32) {
      buf = hd_window(w, p);
      avail = 64;
    }
    const uint32_t e = lut[buf >> (64 - t.lb)];
    int L;
    if (e) {
      *sym = e >> 8;
      L = (int)(e & 255u);
    } else {
      L = hd_step(t, lut, w, p, sym);   // long codeword: table walk
      if (L == 0) return 0;
    }
    p += L;
    buf <<= L;   // L <= 60
    avail -= L;  // < 32 (even negative) forces a refill
    return L;
  }
};

// chunk k starts at its boundary and is decoded in the first pass
__global__ void huff_init_kernel(int64_t nchunk, int64_t* __restrict__ start,
                                 int* __restrict__ dirty) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nchunk) {
    start[k] = k * (int64_t)HD_CB;
    dirty[k] = 1;
  }
}

// sync pass: chunks whose start moved are decoded to their exit
__global__ void __launch_bounds__(256)
huff_sync_kernel(HuffDecTables t, const uint32_t* __restrict__ w,
                 int64_t total_bits, int64_t nchunk,
                 int64_t* __restrict__ start, int64_t* __restrict__ exitp,
                 int32_t* __restrict__ count, int* __restrict__ dirty,
                 int* __restrict__ changed, int* __restrict__ bad) {
  __shared__ uint32_t lut[1 << HD_LB];
  for (int k = threadIdx.x; k < (1 << t.lb); k += blockDim.x) lut[k] = t.lut[k];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nchunk) return;
  if (!dirty[k]) return;
  dirty[k] = 0;
  const int64_t end = min((k + 1) * (int64_t)HD_CB, total_bits);
  HdCursor cur{0ull, 0, start[k]};
  int32_t c = 0;
  while (cur.p < end) {
    uint32_t sym;
    if (cur.next(t, lut, w, &sym) == 0) { atomicOr(bad, 1); break; }
    c++;
  }
  const int64_t p = cur.p;
  exitp[k] = p;
  count[k] = c;
  if (k + 1 < nchunk && start[k + 1] != p) {
    start[k + 1] = p;
    dirty[k + 1] = 1;
    atomicOr(changed, 1);
  }
}

// symbols of chunk k from its true start to out[off[k]...]; once the
// output position is 8-byte aligned, symbols are gathered in a 64-bit
// register and stored 8 bytes at a time
template <typename S>
__global__ void __launch_bounds__(256)
huff_write_kernel(HuffDecTables t, const uint32_t* __restrict__ w,
                  int64_t total_bits, int64_t nchunk,
                  const int64_t* __restrict__ start,
                  const long long* __restrict__ off, S* __restrict__ out) {
  __shared__ uint32_t lut[1 << HD_LB];
  for (int k = threadIdx.x; k < (1 << t.lb); k += blockDim.x) lut[k] = t.lut[k];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nchunk) return;
  constexpr int V = 8 / sizeof(S);
  const int64_t end = min((k + 1) * (int64_t)HD_CB, total_bits);
  HdCursor cur{0ull, 0, start[k]};
  int64_t o = off[k];
  uint32_t sym;
  while (cur.p < end && ((uintptr_t)(out + o) & 7) != 0) {
    if (cur.next(t, lut, w, &sym) == 0) return;
    out[o++] = (S)sym;
  }
  unsigned long long acc = 0;
  int nv = 0;
  while (cur.p < end) {
    if (cur.next(t, lut, w, &sym) == 0) break;
    acc |= (unsigned long long)sym << (8 * sizeof(S) * nv);
    if (++nv == V) {
      *reinterpret_cast<unsigned long long*>(out + o) = acc;
      o += V;
      acc = 0;
      nv = 0;
    }
  }
  for (int i = 0; i < nv; i++) out[o + i] = (S)(acc >> (8 * sizeof(S) * i));
}

}  // namespace vfcp

using namespace vfcp;

// capi.cu: the library's last-error message
int vfcp_record_error(int code, const char* msg);

namespace {
int hfail(int code, const std::string& m) {
  return vfcp_record_error(code, m.c_str());
}
#define HCK(x)                                                              \
  do {                                                                      \
    cudaError_t _e = (x);                                                   \
    if (_e != cudaSuccess) return hfail(VFCP_ECUDA, cudaGetErrorString(_e)); \
  } while (0)
}  // namespace

extern "C" {

int vfcp_huff_hist_dev(const void* symbols, int sym_bytes, int64_t n,
                       int32_t alphabet, int32_t wbase,
                       unsigned long long* counts, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return VFCP_OK;
  if (sym_bytes != 1 && sym_bytes != 2) return hfail(VFCP_EINVAL, "symbol width");
  // the window must lie inside the alphabet (a small alphabet is covered by
  // a window at 0: bins past it stay empty)
  if (wbase < 0 || (alphabet >= HW_BINS && wbase + HW_BINS > alphabet) ||
      (alphabet < HW_BINS))
    wbase = alphabet >= HW_BINS ? std::min(std::max(wbase, 0), alphabet - HW_BINS) : 0;
  int dev = 0, nsm = 148;
  HCK(cudaGetDevice(&dev));
  HCK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t blocks = std::min<int64_t>((n + 2047) / 2048, (int64_t)nsm * 8);
  if (sym_bytes == 2)
    huff_hist_kernel<uint16_t><<<(unsigned)blocks, 256, 0, st>>>(
        (const uint16_t*)symbols, n, wbase, counts);
  else
    huff_hist_kernel<uint8_t><<<(unsigned)blocks, 256, 0, st>>>(
        (const uint8_t*)symbols, n, wbase, counts);
  HCK(cudaGetLastError());
  return VFCP_OK;
}

int vfcp_huff_pack_dev(const void* symbols, int sym_bytes, int64_t n,
                       const uint8_t* lens_host, int32_t alphabet,
                       uint32_t* out_words, int64_t n_words, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (sym_bytes != 1 && sym_bytes != 2) return hfail(VFCP_EINVAL, "symbol width");
  HCK(cudaMemsetAsync(out_words, 0, sizeof(uint32_t) * (size_t)n_words, st));
  if (n <= 0) return VFCP_OK;
  // canonical codes by ascending (length, symbol) (huffman.py:51-62)
  std::vector<unsigned long long> codes(alphabet, 0);
  {
    std::vector<int> order;
    for (int s = 0; s < alphabet; s++)
      if (lens_host[s]) order.push_back(s);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return lens_host[a] < lens_host[b];
    });
    unsigned long long code = 0;
    int prev = 0;
    for (int s : order) {
      code <<= (lens_host[s] - prev);
      prev = lens_host[s];
      codes[s] = code;
      code++;
    }
  }
  const int64_t nchunk = (n + HP_CHUNK - 1) / HP_CHUNK;
  uint8_t* d_lens = nullptr;
  unsigned long long *d_codes = nullptr, *d_bits = nullptr, *d_off = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  HCK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_bits, d_off, (int)nchunk, st));
  HCK(cudaMallocAsync(&d_lens, alphabet, st));
  HCK(cudaMallocAsync(&d_codes, sizeof(unsigned long long) * alphabet, st));
  HCK(cudaMallocAsync(&d_bits, sizeof(unsigned long long) * nchunk, st));
  HCK(cudaMallocAsync(&d_off, sizeof(unsigned long long) * nchunk, st));
  HCK(cudaMallocAsync(&d_tmp, tmp_bytes + 16, st));
  HCK(cudaMemcpyAsync(d_lens, lens_host, alphabet, cudaMemcpyHostToDevice, st));
  HCK(cudaMemcpyAsync(d_codes, codes.data(), sizeof(unsigned long long) * alphabet,
                      cudaMemcpyHostToDevice, st));
  if (sym_bytes == 2) {
    huff_bits_kernel<uint16_t><<<(unsigned)nchunk, HP_T, 0, st>>>(
        (const uint16_t*)symbols, n, d_lens, d_bits);
  } else {
    huff_bits_kernel<uint8_t><<<(unsigned)nchunk, HP_T, 0, st>>>(
        (const uint8_t*)symbols, n, d_lens, d_bits);
  }
  HCK(cudaGetLastError());
  HCK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_bits, d_off, (int)nchunk, st));
  if (sym_bytes == 2) {
    huff_pack_kernel<uint16_t><<<(unsigned)nchunk, HP_T, 0, st>>>(
        (const uint16_t*)symbols, n, d_lens, d_codes, d_off, out_words);
  } else {
    huff_pack_kernel<uint8_t><<<(unsigned)nchunk, HP_T, 0, st>>>(
        (const uint8_t*)symbols, n, d_lens, d_codes, d_off, out_words);
  }
  HCK(cudaGetLastError());
  cudaFreeAsync(d_lens, st);
  cudaFreeAsync(d_codes, st);
  cudaFreeAsync(d_bits, st);
  cudaFreeAsync(d_off, st);
  cudaFreeAsync(d_tmp, st);
  return VFCP_OK;
}

int vfcp_huff_unpack_dev(const uint32_t* words, int64_t n_words,
                         int64_t total_bits, const uint8_t* lens_host,
                         int32_t alphabet, int64_t n, void* out,
                         int sym_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) return VFCP_OK;
  if (sym_bytes != 1 && sym_bytes != 2) return hfail(VFCP_EINVAL, "symbol width");
  // the window reads two words past any bit position inside the stream
  if (n_words < (total_bits + 31) / 32 + 2)
    return hfail(VFCP_ECAPACITY, "vfcp_huff_unpack_dev: words need 2 words of padding");
  int max_len = 0;
  for (int s = 0; s < alphabet; s++) max_len = std::max<int>(max_len, lens_host[s]);
  if (max_len == 0 || max_len > 60) return hfail(VFCP_ECORRUPT, "corrupt entropy stream");
  std::vector<int32_t> order;
  for (int s = 0; s < alphabet; s++)
    if (lens_host[s]) order.push_back(s);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return lens_host[a] < lens_host[b]; });
  HuffDecTables t;
  memset(&t, 0, sizeof(t));
  {
    unsigned long long code = 0;
    int64_t idx = 0;
    for (int s : order) t.count_at[lens_host[s]]++;
    for (int L = 1; L <= max_len; L++) {
      code <<= 1;
      t.first_code[L] = (int64_t)code;
      t.offset_at[L] = idx;
      code += (unsigned long long)t.count_at[L];
      idx += t.count_at[L];
    }
  }
  t.lb = std::min(max_len, HD_LB);
  t.max_len = max_len;
  std::vector<uint32_t> lut((size_t)1 << t.lb, 0), symtab(order.size());
  for (size_t q = 0; q < order.size(); q++) symtab[q] = (uint32_t)order[q];
  for (int L = 1; L <= t.lb; L++)
    for (int64_t q = 0; q < t.count_at[L]; q++) {
      const uint64_t c = (uint64_t)t.first_code[L] + (uint64_t)q;
      const uint32_t sym = (uint32_t)order[t.offset_at[L] + q];
      const uint64_t lo = c << (t.lb - L), hi = (c + 1) << (t.lb - L);
      for (uint64_t x = lo; x < hi; x++) lut[x] = (sym << 8) | (uint32_t)L;
    }
  const int64_t nchunk = (total_bits + HD_CB - 1) / HD_CB;
  if (nchunk == 0) return hfail(VFCP_ECORRUPT, "corrupt entropy stream");
  uint32_t *d_lut = nullptr, *d_sym = nullptr;
  int64_t *d_start = nullptr, *d_exit = nullptr;
  int32_t* d_count = nullptr;
  long long* d_off = nullptr;
  int *d_dirty = nullptr, *d_flags = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_bytes = 0;
  HCK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_count, d_off, (int)nchunk, st));
  HCK(cudaMallocAsync(&d_lut, sizeof(uint32_t) * lut.size(), st));
  HCK(cudaMallocAsync(&d_sym, sizeof(uint32_t) * std::max<size_t>(1, symtab.size()), st));
  HCK(cudaMallocAsync(&d_start, sizeof(int64_t) * nchunk, st));
  HCK(cudaMallocAsync(&d_exit, sizeof(int64_t) * nchunk, st));
  HCK(cudaMallocAsync(&d_count, sizeof(int32_t) * nchunk, st));
  HCK(cudaMallocAsync(&d_off, sizeof(long long) * (nchunk + 1), st));
  HCK(cudaMallocAsync(&d_dirty, sizeof(int) * nchunk, st));
  HCK(cudaMallocAsync(&d_flags, sizeof(int) * 2, st));
  HCK(cudaMallocAsync(&d_tmp, tmp_bytes + 16, st));
  HCK(cudaMemcpyAsync(d_lut, lut.data(), sizeof(uint32_t) * lut.size(),
                      cudaMemcpyHostToDevice, st));
  HCK(cudaMemcpyAsync(d_sym, symtab.data(), sizeof(uint32_t) * symtab.size(),
                      cudaMemcpyHostToDevice, st));
  huff_init_kernel<<<(unsigned)((nchunk + 255) / 256), 256, 0, st>>>(nchunk, d_start,
                                                                   d_dirty);
  HCK(cudaGetLastError());
  t.lut = d_lut;
  t.symtab = d_sym;
  HCK(cudaMemsetAsync(d_flags, 0, sizeof(int) * 2, st));
  const unsigned grid = (unsigned)((nchunk + 255) / 256);
  int rc = VFCP_OK;
  int h[2] = {0, 0};
  for (int it = 0; it < 64; it++) {
    HCK(cudaMemsetAsync(d_flags, 0, sizeof(int), st));   // changed
    huff_sync_kernel<<<grid, 256, 0, st>>>(t, words, total_bits, nchunk, d_start,
                                           d_exit, d_count, d_dirty, d_flags,
                                           d_flags + 1);
    HCK(cudaGetLastError());
    HCK(cudaMemcpyAsync(h, d_flags, sizeof(int) * 2, cudaMemcpyDeviceToHost, st));
    HCK(cudaStreamSynchronize(st));
    if (h[1] || !h[0]) break;
  }
  long long total = 0;
  int64_t last_exit = -1;
  if (!h[1] && !h[0]) {
    HCK(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_count, d_off, (int)nchunk, st));
    int32_t lc = 0;
    long long lo = 0;
    HCK(cudaMemcpyAsync(&lo, d_off + nchunk - 1, sizeof(long long), cudaMemcpyDeviceToHost, st));
    HCK(cudaMemcpyAsync(&lc, d_count + nchunk - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HCK(cudaMemcpyAsync(&last_exit, d_exit + nchunk - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HCK(cudaStreamSynchronize(st));
    total = lo + lc;
  }
  if (h[1] || h[0] || total != n || last_exit != total_bits) {
    // invalid code, no convergence or a length mismatch: the caller decodes
    // on the host (the reference's exact error behaviour)
    rc = hfail(VFCP_ECORRUPT, "corrupt entropy stream");
  } else if (sym_bytes == 2) {
    huff_write_kernel<uint16_t><<<grid, 256, 0, st>>>(t, words, total_bits, nchunk,
                                                      d_start, d_off, (uint16_t*)out);
  } else {
    huff_write_kernel<uint8_t><<<grid, 256, 0, st>>>(t, words, total_bits, nchunk,
                                                     d_start, d_off, (uint8_t*)out);
  }
  cudaFreeAsync(d_lut, st);
  cudaFreeAsync(d_sym, st);
  cudaFreeAsync(d_start, st);
  cudaFreeAsync(d_exit, st);
  cudaFreeAsync(d_count, st);
  cudaFreeAsync(d_off, st);
  cudaFreeAsync(d_dirty, st);
  cudaFreeAsync(d_flags, st);
  cudaFreeAsync(d_tmp, st);
  if (rc) return rc;
  HCK(cudaGetLastError());
  return VFCP_OK;
}

}  // extern "C"
