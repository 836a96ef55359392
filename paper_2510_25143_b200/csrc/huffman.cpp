// Host entropy backend: canonical Huffman, byte-identical to huffman.py.
//
//   vfcp_huff_lengths  huffman.py:21-48  code_lengths (heap order by
//                      (count, serial); merged nodes get serials
//                      present[-1]+1, +2, ...)
//   vfcp_huff_pack     huffman.py:51-76  canonical codes (ascending
//                      (length, symbol)) + MSB-first bit packing
//   vfcp_huff_unpack   huffman.py:79-98,116-149 decode
//
// The reference keeps this stage on the host; so does this build (it is
// timed and reported separately from the device pipeline).  Packing is
// multi-threaded over symbol chunks with exact bit offsets.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vfcp_b200.h"

namespace {
constexpr int MAX_CODE_LEN = 60;

inline uint32_t sym_at(const void* s, int sym_bytes, int64_t k) {
  switch (sym_bytes) {
    case 1: return ((const uint8_t*)s)[k];
    case 2: return ((const uint16_t*)s)[k];
    case 4: return ((const uint32_t*)s)[k];
    default: return (uint32_t)((const int64_t*)s)[k];
  }
}

void canonical(const uint8_t* lens, int32_t alphabet,
               std::vector<uint64_t>& codes) {
  std::vector<int32_t> order;
  for (int32_t s = 0; s < alphabet; s++)
    if (lens[s]) order.push_back(s);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return lens[a] < lens[b]; });
  codes.assign(alphabet, 0);
  uint64_t code = 0;
  int prev = 0;
  for (int32_t s : order) {
    code <<= (lens[s] - prev);
    prev = lens[s];
    codes[s] = code;
    code += 1;
  }
}
}  // namespace

extern "C" {

int vfcp_huff_lengths(const int64_t* counts, int32_t alphabet,
                      uint8_t* lens) {
  std::memset(lens, 0, (size_t)alphabet);
  std::vector<int32_t> present;
  for (int32_t s = 0; s < alphabet; s++)
    if (counts[s]) present.push_back(s);
  if (present.empty()) return VFCP_OK;
  if (present.size() == 1) {
    lens[present[0]] = 1;
    return VFCP_OK;
  }
  // nodes: leaves 0..P-1, merges appended; parent links give the depths
  const size_t P = present.size();
  std::vector<int64_t> parent(2 * P, -1);
  typedef std::pair<std::pair<int64_t, int64_t>, int64_t> Item;  // ((w, serial), node)
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  for (size_t q = 0; q < P; q++)
    heap.push({{counts[present[q]], (int64_t)present[q]}, (int64_t)q});
  int64_t serial = (int64_t)present.back() + 1;
  int64_t next = (int64_t)P;
  while (heap.size() > 1) {
    Item a = heap.top(); heap.pop();
    Item b = heap.top(); heap.pop();
    parent[a.second] = next;
    parent[b.second] = next;
    heap.push({{a.first.first + b.first.first, serial}, next});
    serial++;
    next++;
  }
  std::vector<int> depth(next, 0);
  for (int64_t n = next - 2; n >= 0; n--) depth[n] = depth[parent[n]] + 1;
  int mx = 0;
  for (size_t q = 0; q < P; q++) mx = std::max(mx, depth[q]);
  if (mx > MAX_CODE_LEN) return VFCP_EINVAL;
  for (size_t q = 0; q < P; q++) lens[present[q]] = (uint8_t)depth[q];
  return VFCP_OK;
}

int vfcp_huff_count(const void* symbols, int sym_bytes, int64_t n,
                    int32_t alphabet, int64_t* counts) {
  std::memset(counts, 0, sizeof(int64_t) * (size_t)alphabet);
  for (int64_t k = 0; k < n; k++) {
    uint32_t s = sym_at(symbols, sym_bytes, k);
    if (s >= (uint32_t)alphabet) return VFCP_EINVAL;
    counts[s]++;
  }
  return VFCP_OK;
}

int vfcp_huff_pack(const void* symbols, int sym_bytes, int64_t n,
                   const uint8_t* lens, int32_t alphabet, uint8_t* out,
                   int64_t out_bytes, int64_t* bits_out, int threads) {
  std::vector<uint64_t> codes;
  canonical(lens, alphabet, codes);
  if (threads < 1) threads = 1;
  if (n < (int64_t)threads * 65536) threads = 1;
  std::vector<int64_t> start(threads + 1), bits(threads + 1, 0);
  for (int t = 0; t <= threads; t++) start[t] = n * t / threads;
  auto count = [&](int t) {
    int64_t b = 0;
    for (int64_t k = start[t]; k < start[t + 1]; k++)
      b += lens[sym_at(symbols, sym_bytes, k)];
    bits[t + 1] = b;
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < threads; t++) th.emplace_back(count, t);
    count(0);
    for (auto& x : th) x.join();
  }
  for (int t = 0; t < threads; t++) bits[t + 1] += bits[t];
  const int64_t total = bits[threads];
  if ((total + 7) / 8 > out_bytes) return VFCP_ECAPACITY;
  std::memset(out, 0, (size_t)((total + 7) / 8));
  auto pack = [&](int t) {
    int64_t pos = bits[t];
    // bit accumulator, MSB-first; flushes whole bytes
    uint64_t acc = 0;
    int nacc = 0;
    // leading partial byte shared with the previous chunk
    int lead = (int)(pos & 7);
    int64_t byte = pos >> 3;
    acc = 0;
    nacc = lead;  // pretend the first `lead` bits are zeros
    bool first = true;
    auto flush_byte = [&](uint8_t b) {
      if (first && lead) __atomic_fetch_or(out + byte, b, __ATOMIC_RELAXED);
      else out[byte] = b;
      first = false;
      byte++;
    };
    for (int64_t k = start[t]; k < start[t + 1]; k++) {
      uint32_t s = sym_at(symbols, sym_bytes, k);
      int L = lens[s];
      uint64_t c = codes[s];
      if (nacc + L > 64) {
        // split: emit the high part first
        int hi = 64 - nacc;
        acc = (acc << hi) | (c >> (L - hi));
        nacc = 64;
        while (nacc >= 8) { flush_byte((uint8_t)(acc >> (nacc - 8))); nacc -= 8; }
        L -= hi;
        c &= (L == 64) ? ~0ull : ((1ull << L) - 1);
      }
      acc = (L == 64) ? c : ((acc << L) | c);
      nacc += L;
      while (nacc >= 8) { flush_byte((uint8_t)(acc >> (nacc - 8))); nacc -= 8; }
    }
    if (nacc > 0) {
      uint8_t b = (uint8_t)((acc << (8 - nacc)) & 0xFF);
      // trailing partial byte may be shared with the next chunk
      __atomic_fetch_or(out + byte, b, __ATOMIC_RELAXED);
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < threads; t++) th.emplace_back(pack, t);
    pack(0);
    for (auto& x : th) x.join();
  }
  *bits_out = total;
  return VFCP_OK;
}

int vfcp_huff_unpack(const uint8_t* data, int64_t total_bits,
                     const uint8_t* lens, int32_t alphabet, int64_t n,
                     void* out, int sym_bytes) {
  if (n == 0) return VFCP_OK;
  int max_len = 0;
  for (int32_t s = 0; s < alphabet; s++) max_len = std::max<int>(max_len, lens[s]);
  if (max_len == 0) return VFCP_ECORRUPT;
  std::vector<int32_t> order;
  for (int32_t s = 0; s < alphabet; s++)
    if (lens[s]) order.push_back(s);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return lens[a] < lens[b]; });
  std::vector<int64_t> count_at(max_len + 1, 0), offset_at(max_len + 1, 0);
  std::vector<uint64_t> first_code(max_len + 1, 0);
  for (int32_t s : order) count_at[lens[s]]++;
  uint64_t code = 0;
  int64_t idx = 0;
  for (int L = 1; L <= max_len; L++) {
    code <<= 1;
    first_code[L] = code;
    offset_at[L] = idx;
    code += (uint64_t)count_at[L];
    idx += count_at[L];
  }
  // LUT over the next LB bits: (symbol << 8) | length, 0 = slow path
  const int LB = std::min(max_len, 12);
  std::vector<uint32_t> lut((size_t)1 << LB, 0);
  for (int L = 1; L <= LB; L++)
    for (int64_t q = 0; q < count_at[L]; q++) {
      uint64_t c = first_code[L] + (uint64_t)q;
      uint32_t sym = (uint32_t)order[offset_at[L] + q];
      uint64_t lo = c << (LB - L), hi = (c + 1) << (LB - L);
      for (uint64_t x = lo; x < hi; x++) lut[x] = (sym << 8) | (uint32_t)L;
    }
  const int64_t nbytes = (total_bits + 7) / 8;
  auto peek = [&](int64_t pos, int nb) -> uint64_t {
    // nb <= 57 bits starting at bit pos (zeros past the end)
    int64_t b = pos >> 3;
    uint64_t w = 0;
    for (int q = 0; q < 8; q++) {
      w <<= 8;
      if (b + q < nbytes) w |= data[b + q];
    }
    w <<= (pos & 7);
    return w >> (64 - nb);
  };
  int64_t pos = 0;
  for (int64_t k = 0; k < n; k++) {
    uint32_t sym;
    uint64_t e = lut[peek(pos, LB)];
    if (e) {
      sym = e >> 8;
      pos += (int)(e & 0xFF);
    } else {
      uint64_t c = 0;
      int L = 0;
      while (true) {
        if (pos >= nbytes * 8) return VFCP_ECORRUPT;
        int bit = (data[pos >> 3] >> (7 - (pos & 7))) & 1;
        pos++;
        c = (c << 1) | (uint64_t)bit;
        L++;
        if (L > max_len) return VFCP_ECORRUPT;
        if (count_at[L] > 0) {
          int64_t d = (int64_t)c - (int64_t)first_code[L];
          if (d >= 0 && d < count_at[L]) {
            sym = (uint32_t)order[offset_at[L] + d];
            break;
          }
        }
      }
    }
    if (pos > total_bits) return VFCP_ECORRUPT;
    switch (sym_bytes) {
      case 1: ((uint8_t*)out)[k] = (uint8_t)sym; break;
      case 2: ((uint16_t*)out)[k] = (uint16_t)sym; break;
      case 4: ((uint32_t*)out)[k] = sym; break;
      default: ((int64_t*)out)[k] = sym; break;
    }
  }
  if (pos != total_bits) return VFCP_ECORRUPT;
  return VFCP_OK;
}

}  // extern "C"
