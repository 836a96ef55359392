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
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;   // warp-uniform loop bound
    const bool ok = i < n;
    const int s = ok ? (int)sym[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, s);
    const bool leader = ok && (grp & ((1u << lane) - 1u)) == 0;
    if (leader) {
      const int w = s - wbase;
      if ((unsigned)w < (unsigned)HW_BINS) atomicAdd(&h[w], (unsigned)__popc(grp));
      else atomicAdd(&counts[s], (unsigned long long)__popc(grp));
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
  const int64_t first = (int64_t)blockIdx.x * HP_CHUNK + (int64_t)threadIdx.x * HP_PER;
  const int cnt = (int)max((int64_t)0, min((int64_t)HP_PER, n - first));
  unsigned long long mine = 0;
  for (int k = 0; k < cnt; k++) mine += __ldg(lens + sym[first + k]);
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
  for (int k = 0; k < cnt; k++) {
    const int s = (int)sym[first + k];
    const int L = __ldg(lens + s);
    const unsigned long long c = __ldg(codes + s);
    if (L > 32) {
      append(c >> 32, L - 32);
      append(c & 0xffffffffull, 32);
    } else if (L > 0) {
      append(c, L);
    }
  }
  if (nb > 0) atomicOr(out + wi, bswap32((uint32_t)(buf >> 32)));
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
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)nsm * 8);
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

}  // extern "C"
