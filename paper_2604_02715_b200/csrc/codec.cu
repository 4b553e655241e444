// Exponent-Huffman codec: multi-threaded host encoder (bit-identical to
// xpg codec.py:235-272) and the sm_100a decoder kernel (codec.py:275-330).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "codec.cuh"
#include "codec_dev.cuh"
#include "ptx_sm100.cuh"
#include "launch_count.h"

namespace xpgb {

bool codec_canonical_codes(const uint8_t* lengths, uint32_t* codes) {
  // canonical order (length, symbol) ascending, as HuffmanTable.from_lengths (codec.py:152-173)
  double kraft = 0.0;
  int present = 0;
  for (int s = 0; s < kCodecSymbols; ++s) {
    codes[s] = 0;
    if (lengths[s] > kCodecMaxLen) return false;
    if (lengths[s]) {
      kraft += 1.0 / (double)(1ull << lengths[s]);
      ++present;
    }
  }
  if (!present || kraft > 1.0 + 1e-12) return false;
  uint64_t code = 0;
  int prev = 0;
  for (int l = 1; l <= kCodecMaxLen; ++l)
    for (int s = 0; s < kCodecSymbols; ++s)
      if (lengths[s] == l) {
        code <<= (l - prev);
        codes[s] = (uint32_t)code;
        code += 1;
        prev = l;
      }
  return true;
}

void codec_histogram(const uint8_t* data, size_t bytes, uint64_t* counts, int threads) {
  const size_t n = bytes / 2;
  threads = std::max(1, std::min(threads, (int)std::max<size_t>(1, n / (1 << 20))));
  std::vector<std::vector<uint64_t>> part(threads, std::vector<uint64_t>(kCodecSymbols, 0));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const size_t a = n * t / threads, b = n * (t + 1) / threads;
      const uint16_t* w = reinterpret_cast<const uint16_t*>(data);
      uint64_t* c = part[t].data();
      for (size_t i = a; i < b; ++i) ++c[(w[i] >> 7) & 0xFF];
    });
  for (auto& th : pool) th.join();
  for (int s = 0; s < kCodecSymbols; ++s) {
    uint64_t v = 0;
    for (int t = 0; t < threads; ++t) v += part[t][s];
    counts[s] = v;
  }
}

size_t codec_bits_bound(size_t n, const uint8_t* lengths) {
  int mx = 0;
  for (int s = 0; s < kCodecSymbols; ++s) mx = std::max<int>(mx, lengths[s]);
  return (n * (size_t)mx + 7) / 8;
}

bool codec_encode(const uint16_t* words, size_t n, const uint8_t* lengths, const uint32_t* codes, uint8_t* sm_out,
                  uint8_t* bits_out, size_t bits_cap, size_t* bits_len, uint64_t* bit_count, uint32_t* index_out,
                  int chunk, int* missing) {
  uint64_t acc = 0;
  int nacc = 0;
  size_t out = 0;
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint16_t w = words[i];
    const int e = (w >> 7) & 0xFF;
    const int l = lengths[e];
    if (!l) {
      if (missing) *missing = e;
      return false;
    }
    if (index_out && chunk > 0 && (i % (size_t)chunk) == 0) index_out[i / chunk] = (uint32_t)total;
    sm_out[i] = (uint8_t)(((w >> 8) & 0x80) | (w & 0x7F));
    acc = (acc << l) | codes[e];
    nacc += l;
    total += l;
    while (nacc >= 8) {
      nacc -= 8;
      if (out < bits_cap) bits_out[out] = (uint8_t)(acc >> nacc);
      ++out;
    }
    acc &= (nacc ? ((1ull << nacc) - 1) : 0ull);
  }
  if (nacc) {
    if (out < bits_cap) bits_out[out] = (uint8_t)(acc << (8 - nacc));
    ++out;
  }
  *bits_len = out;
  *bit_count = total;
  if (missing) *missing = -1;
  return out <= bits_cap && total < (1ull << 32);
}

// Sequential host scan of a stream: rebuilds the chunk index and validates it the way
// decompress() does (codec.py:304-327).  Returns 0, 1 = truncated, 2 = invalid code.
int codec_build_index(const uint8_t* bits, size_t bits_len, size_t n, const uint8_t* lengths, int chunk,
                      uint32_t* index_out, size_t* consumed_bits) {
  int count[kCodecMaxLen + 1] = {0};
  uint32_t first_code[kCodecMaxLen + 1] = {0};
  for (int s = 0; s < kCodecSymbols; ++s)
    if (lengths[s]) ++count[lengths[s]];
  uint32_t code = 0;
  int prev = 0, maxlen = 0;
  for (int l = 1; l <= kCodecMaxLen; ++l)
    if (count[l]) {
      code <<= (l - prev);
      first_code[l] = code;
      code += count[l];
      prev = l;
      maxlen = l;
    }
  const uint64_t total_bits = (uint64_t)bits_len * 8;
  uint64_t pos = 0;
  for (size_t i = 0; i < n; ++i) {
    if (index_out && (i % (size_t)chunk) == 0) index_out[i / chunk] = (uint32_t)pos;
    uint32_t c = 0;
    int l = 0;
    for (;;) {
      if (pos >= total_bits) return 1;
      c = (c << 1) | ((bits[pos >> 3] >> (7 - (pos & 7))) & 1);
      ++pos;
      ++l;
      if (l > maxlen) return 2;
      if (count[l] && c - first_code[l] < (uint32_t)count[l]) break;
    }
  }
  if (consumed_bits) *consumed_bits = pos;
  return 0;
}

// ----------------------------------------------------------------------------- GPU decoder

struct DecodeParams {
  DecodeTensor t[kMaxDecodeTensors];  // tensors of one launch, each n values
  int ntensors;
  uint64_t n;
  int chunk;
  const DecTables* tabs;  // prebuilt by k_build_tables
};



// Eight (sign/mantissa, exponent) byte pairs -> bf16 words by byte permutes:
// x = [e1 s1 e0 s0] per 16-bit lane -> (s >> 7) << 15 | e << 7 | (s & 0x7F).
__device__ __forceinline__ uint32_t pack_words(uint32_t sm4, uint32_t ex4, uint32_t sel) {
  const uint32_t x = __byte_perm(sm4, ex4, sel);
  return ((x >> 1) & 0x7F807F80u) | (x & 0x007F007Fu) | ((x << 8) & 0x80008000u);
}

// Bitstream words for one chunk, the next one always in flight.  (16-byte loads with a
// second in flight measured slower: 726 vs 951 GB/s.)
struct WordScalar {
  const uint32_t* wp;
  uint32_t nxt;
  __device__ __forceinline__ void init(const uint32_t* p) {
    wp = p;
    nxt = *wp++;
  }
  __device__ __forceinline__ uint32_t pop() {
    const uint32_t r = nxt;
    nxt = *wp++;
    return bswap32(r);
  }
};

template <bool FAST, class R>
__device__ __forceinline__ void decode_chunk(R& q, uint64_t win, int avail, const uint8_t* __restrict__ sm,
                                             uint16_t* __restrict__ out, uint64_t v0, uint64_t v1, const uint32_t* lut3, const uint8_t* lmeta,
                                             int ml, const int* count, const uint32_t* first_code,
                                             const int* first_rank, const uint8_t* sorted_sym);


__global__ void __launch_bounds__(256) k_build_tables(const CodecTable table, DecTables* out) {
  __shared__ uint32_t lut3[1 << kMultiBits];
  __shared__ uint8_t lmeta[1 << kMultiBits];
  __shared__ uint32_t first_code[kCodecMaxLen + 1];
  __shared__ int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  __shared__ uint8_t sorted_sym[kCodecSymbols];
  __shared__ int maxlen;
  const int tid = threadIdx.x;
  if (tid <= kCodecMaxLen) count[tid] = 0;
  __syncthreads();
  if (tid < kCodecSymbols && table.len[tid]) atomicAdd(&count[table.len[tid]], 1);
  __syncthreads();
  if (tid == 0) {
    uint32_t code = 0;
    int prev = 0, rank = 0, ml = 0;
    for (int l = 1; l <= kCodecMaxLen; ++l) {
      first_rank[l] = rank;
      first_code[l] = 0;
      if (count[l]) {
        code <<= (l - prev);
        first_code[l] = code;
        code += count[l];
        prev = l;
        rank += count[l];
        ml = l;
      }
    }
    maxlen = ml;
  }
  __syncthreads();
  if (tid < kCodecSymbols) {
    const int l = table.len[tid];
    if (l) {
      int r = 0;
      for (int s = 0; s < tid; ++s) r += (table.len[s] == l);
      sorted_sym[first_rank[l] + r] = (uint8_t)tid;
    }
  }
  __syncthreads();
  const int ml = maxlen;
  // whole codes at the head of every 11-bit pattern: a code is whole when its length
  // fits the known bits (a prefix code is decided by its own bits only)
  for (int i = tid; i < (1 << kMultiBits); i += blockDim.x) {
    const uint64_t w = (uint64_t)i << (64 - kMultiBits);
    uint32_t syms = 0;
    int tot = 0, c = 0;
    while (c < 4) {
      int sym;
      const int l = canon_decode(w << tot, ml, count, first_code, first_rank, sorted_sym, &sym);
      if (!l || tot + l > kMultiBits) break;
      syms |= (uint32_t)sym << (8 * c);
      tot += l;
      ++c;
    }
    lut3[i] = syms;
    lmeta[i] = (uint8_t)(c | (tot << 3));
  }
  __syncthreads();

  for (int i = tid; i < (1 << kMultiBits); i += blockDim.x) {
    out->lut3[i] = lut3[i];
    out->lmeta[i] = lmeta[i];
  }
  // pair table: every 12-bit pattern -> the first two whole codes it starts with, already in
  // bf16 position for k_exp_decode2: e0 << 7 and e1 << 23 (the exponent fields of a pair of
  // bf16 words), their total length in bits 0..3 (0: the pair does not fit in 12 bits), and
  // the first code's own length in bits 16..20 (0: longer than 12 bits).  Every metadata bit
  // sits where the final select keeps the sign/mantissa plane, so one LOP3 drops it.
  for (int i = tid; i < (1 << kPairBits); i += blockDim.x) {
    const uint64_t w = (uint64_t)i << (64 - kPairBits);
    int s0 = 0, s1 = 0;
    const int l0 = canon_decode(w, ml, count, first_code, first_rank, sorted_sym, &s0);
    uint32_t e = 0;
    if (l0 && l0 <= kPairBits) {
      e = ((uint32_t)s0 << 7) | ((uint32_t)l0 << 16);
      const int l1 = canon_decode(w << l0, ml, count, first_code, first_rank, sorted_sym, &s1);
      if (l1 && l0 + l1 <= kPairBits) e |= ((uint32_t)s1 << 23) | (uint32_t)(l0 + l1);
    }
    out->pair[i] = e;
  }
  if (tid <= kCodecMaxLen) {
    out->first_code[tid] = first_code[tid];
    out->count[tid] = count[tid];
    out->first_rank[tid] = first_rank[tid];
  }
  if (tid < kCodecSymbols) out->sorted_sym[tid] = sorted_sym[tid];
  if (tid == 0) out->maxlen = maxlen;
}

// One thread decodes one chunk (`chunk` values) starting at index[c]: a 64-bit
// MSB-first window and a multi-symbol table -- every 11-bit pattern maps to the
// up-to-4 whole codewords it starts with (exponents average ~2.6 bits, so one
// lookup usually yields 3-4 values); the symbols sit in one 32-bit table and the
// count/length in a byte table beside it.  Codes longer than the table, and a chunk's
// last values (never decode past the chunk), take the canonical first-code search.
// The tables are 10 KB of shared memory so decode blocks still fit beside a resident
// GEMM CTA; the next bitstream word is always in flight.  Output words are
// (sign << 15) | (exponent << 7) | mantissa, 16 per 32-byte store.
__global__ void __launch_bounds__(256) k_exp_decode(const __grid_constant__ DecodeParams p) {
  __shared__ uint32_t lut3[1 << kMultiBits];
  __shared__ __align__(16) uint8_t lmeta[1 << kMultiBits];
  __shared__ uint32_t first_code[kCodecMaxLen + 1];
  __shared__ int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  __shared__ uint8_t sorted_sym[kCodecSymbols];
  const int tid = threadIdx.x;
  {
    const DecTables* t = p.tabs;
    const uint4* src = reinterpret_cast<const uint4*>(t->lut3);
    uint4* dst = reinterpret_cast<uint4*>(lut3);
    for (int i = tid; i < (1 << kMultiBits) / 4; i += blockDim.x) dst[i] = src[i];
    for (int i = tid; i < (1 << kMultiBits) / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(lmeta)[i] = reinterpret_cast<const uint4*>(t->lmeta)[i];
    if (tid <= kCodecMaxLen) {
      first_code[tid] = t->first_code[tid];
      count[tid] = t->count[tid];
      first_rank[tid] = t->first_rank[tid];
    }
    if (tid < kCodecSymbols) sorted_sym[tid] = t->sorted_sym[tid];
  }
  const int ml = p.tabs->maxlen;
  __syncthreads();

  const uint64_t n = p.n;
  const uint64_t cpt = (n + p.chunk - 1) / p.chunk;  // chunks per tensor
  const uint64_t n_chunks = cpt * (uint64_t)p.ntensors;
  for (uint64_t gc = blockIdx.x * (uint64_t)blockDim.x + tid; gc < n_chunks; gc += (uint64_t)gridDim.x * blockDim.x) {
    const int ti = (int)(gc / cpt);
    const uint64_t c = gc - (uint64_t)ti * cpt;
    const DecodeTensor& d = p.t[ti];
    const uint8_t* __restrict__ sm = d.sm;
    uint16_t* __restrict__ out = d.out;
    const uint64_t v0 = c * p.chunk;
    const uint64_t v1 = (v0 + p.chunk < n) ? v0 + p.chunk : n;
    const uint32_t bitpos = d.index[c] - d.bit_base;
    const uint32_t w = bitpos >> 5, sh = bitpos & 31;
    uint64_t win = (((uint64_t)bswap32(d.bits[w]) << 32) | bswap32(d.bits[w + 1])) << sh;
    int avail = 64 - (int)sh;
    WordScalar q;
    q.init(d.bits + w + 2);
    decode_chunk<true>(q, win, avail, sm, out, v0, v1, lut3, lmeta, ml, count, first_code, first_rank, sorted_sym);
  }
}

template <bool FAST, class R>
__device__ __forceinline__ void decode_chunk(R& q, uint64_t win, int avail, const uint8_t* __restrict__ sm,
                                             uint16_t* __restrict__ out, uint64_t v0, uint64_t v1, const uint32_t* lut3, const uint8_t* lmeta,
                                             int ml, const int* count, const uint32_t* first_code,
                                             const int* first_rank, const uint8_t* sorted_sym) {
  // exponent bytes decoded but not yet written: b0 = values 0..7 of the group, b1 = 8..15,
  // b2 = the spill of a multi-symbol lookup past the group
  uint64_t b0 = 0, b1 = 0, b2 = 0;
  int np = 0;
  const bool wide = ((reinterpret_cast<uintptr_t>(out + v0) | reinterpret_cast<uintptr_t>(sm + v0)) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(out + v0) & 31) == 0;
  for (uint64_t v = v0; v < v1; v += 16) {
    const int cnt = (int)((v1 - v) < 16 ? (v1 - v) : 16);
    uint4 smv = make_uint4(0, 0, 0, 0);
    if (cnt == 16 && wide) smv = *reinterpret_cast<const uint4*>(sm + v);
    if (FAST && cnt == 16 && wide) {
      // a whole group: two halves of 8 exponent bytes, each a 64-bit register filled at
      // byte 8*np; a multi-symbol lookup that crosses the half spills into `carry`.  A
      // lookup may run up to 2 symbols past the chunk (never written): they come from
      // the next chunk's bits or the stream's 8-byte look-ahead padding.
      uint64_t h[2];
      uint64_t cur = b0, carry = 0;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        // one lookup: the fast path needs kMultiBits valid bits, the canonical path (codes
        // longer than the table) refills to >= 32 first
        auto step = [&]() {
          const uint32_t ix = (uint32_t)(win >> (64 - kMultiBits));
          const uint32_t e = lut3[ix];
          const uint32_t mt = lmeta[ix];
          int k = mt & 7, l;
          uint64_t bytes;
          if (__builtin_expect(k == 0, 0)) {
            if (avail < 32) {
              win |= (uint64_t)q.pop() << (32 - avail);
              avail += 32;
            }
            int sym = 0;
            l = canon_decode(win, ml, count, first_code, first_rank, sorted_sym, &sym);
            bytes = (uint32_t)sym;
            k = 1;
          } else {
            l = (int)(mt >> 3);
            bytes = e;
          }
          win <<= l;
          avail -= l;
          const int sh = 8 * np;
          cur |= bytes << sh;
          carry |= np > 4 ? bytes >> (64 - sh) : 0ull;
          np += k;
        };
        while (np < 8) {
          // one refill per up to three lookups: after it avail >= 32, the first lookup
          // leaves >= 21 bits, and each further one runs while kMultiBits remain
          if (avail < 32) {
            win |= (uint64_t)q.pop() << (32 - avail);
            avail += 32;
          }
          step();
          if (np < 8 && avail >= kMultiBits) step();
          if (np < 8 && avail >= kMultiBits) step();
        }
        h[half] = cur;
        cur = carry;
        carry = 0;
        np -= 8;
      }
      b0 = cur;
      const uint32_t e0 = (uint32_t)h[0], e1 = (uint32_t)(h[0] >> 32), e2 = (uint32_t)h[1], e3 = (uint32_t)(h[1] >> 32);
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + v),
                   "r"(pack_words(smv.x, e0, 0x5140u)), "r"(pack_words(smv.x, e0, 0x7362u)),
                   "r"(pack_words(smv.y, e1, 0x5140u)), "r"(pack_words(smv.y, e1, 0x7362u)),
                   "r"(pack_words(smv.z, e2, 0x5140u)), "r"(pack_words(smv.z, e2, 0x7362u)),
                   "r"(pack_words(smv.w, e3, 0x5140u)), "r"(pack_words(smv.w, e3, 0x7362u))
                   : "memory");
      continue;
    }
    while (np < cnt) {
      if (avail < 32) {
        win |= (uint64_t)q.pop() << (32 - avail);
        avail += 32;
      }
      const uint32_t ix = (uint32_t)(win >> (64 - kMultiBits));
      const uint32_t e = lut3[ix];
      const uint32_t mt = lmeta[ix];
      int k = mt & 7, l;
      uint64_t bytes;
      if (k == 0 || k > (int)(v1 - v) - np) {
        int sym = 0;
        l = canon_decode(win, ml, count, first_code, first_rank, sorted_sym, &sym);
        bytes = (uint32_t)sym;
        k = 1;
      } else {
        l = (int)(mt >> 3);
        bytes = e;
      }
      win <<= l;
      avail -= l;
      if (np < 8) {
        b0 |= bytes << (8 * np);
        if (np > 4) b1 |= bytes >> (64 - 8 * np);
      } else {
        const int q = np - 8;
        b1 |= bytes << (8 * q);
        if (q > 4) b2 |= bytes >> (64 - 8 * q);
      }
      np += k;
    }
    if (cnt == 16 && wide) {
      // one 32-byte store per 16 values: a whole sector per thread (the warp's threads
      // write 32 different chunks, so narrower stores cost proportionally more wavefronts)
      const uint32_t e0 = (uint32_t)b0, e1 = (uint32_t)(b0 >> 32), e2 = (uint32_t)b1, e3 = (uint32_t)(b1 >> 32);
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + v),
                   "r"(pack_words(smv.x, e0, 0x5140u)), "r"(pack_words(smv.x, e0, 0x7362u)),
                   "r"(pack_words(smv.y, e1, 0x5140u)), "r"(pack_words(smv.y, e1, 0x7362u)),
                   "r"(pack_words(smv.z, e2, 0x5140u)), "r"(pack_words(smv.z, e2, 0x7362u)),
                   "r"(pack_words(smv.w, e3, 0x5140u)), "r"(pack_words(smv.w, e3, 0x7362u))
                   : "memory");
    } else {
      for (int j = 0; j < cnt; ++j) {
        const uint32_t sym = (uint32_t)((j < 8 ? b0 >> (8 * j) : b1 >> (8 * (j - 8)))) & 0xFFu;
        const uint32_t sb = sm[v + j];
        out[v + j] = (uint16_t)(((sb & 0x80u) << 8) | (sym << 7) | (sb & 0x7Fu));
      }
    }
    b0 = b2;
    b1 = 0;
    b2 = 0;
    np -= cnt;
  }
}


// ---------------------------------------------------------------- decoder v2 (pair table)
//
// One thread per chunk as k_exp_decode, but built around a 12-bit *pair* table whose entry is
// already the exponent half of two bf16 words (e0 << 7 | e1 << 23, metadata in the bits the
// sign/mantissa plane owns).  Per pair of values: one window extract, one table load, one
// length add, one byte permute that duplicates the two sign/mantissa bytes into their 16-bit
// lanes, and one LOP3 select (mask 0x807F807F) -- instead of variable-count symbol insertion.
// 99.7% of pairs of synthetic N(0, 0.02) exponents fit 12 bits; the rest take a per-symbol
// path (the entry's single-code length, or the canonical first-code search for codes > 12
// bits).  Window: 64 bits, bit position p; the stream refills one 32-bit word every second
// pair when p >= 32, so a lookup always has 12 valid bits (p <= 43 at the odd pair).
// One chunk [v0, v1) of one tensor with the pair table (k_exp_decode2's per-thread loop).
template <class W>
__device__ __forceinline__ void decode_chunk_v2(W& w, const uint8_t* __restrict__ sm, uint16_t* __restrict__ out,
                                                uint64_t v0, uint64_t v1, const uint32_t* pair, const CanonTabs& ct) {
    const bool fast = ((v1 - v0) & 15) == 0 &&
                      ((reinterpret_cast<uintptr_t>(out + v0) & 31) | (reinterpret_cast<uintptr_t>(sm + v0) & 15)) == 0;
    if (fast) {
      uint4 nsm = *reinterpret_cast<const uint4*>(sm + v0);
      for (uint64_t v = v0; v < v1; v += 16) {
        const uint4 smv = nsm;
        if (v + 16 < v1) nsm = *reinterpret_cast<const uint4*>(sm + v + 16);  // one group ahead
        const uint32_t smw[4] = {smv.x, smv.y, smv.z, smv.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((j & 1) == 0) w.refill();
          uint32_t e = pair[w.peek12()];
          const int len = (int)(e & 15u);
          if (__builtin_expect(len == 0, 0)) e = pair_slow(w, pair, ct);
          else w.p += len;
          const uint32_t dup = __byte_perm(smw[j >> 1], 0, (j & 1) ? 0x3322u : 0x1100u);
          o[j] = (dup & 0x807F807Fu) | (e & 0x7F807F80u);
        }
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + v), "r"(o[0]), "r"(o[1]),
                     "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                     : "memory");
      }
    } else {
      // ragged or unaligned chunk: one symbol and one 2-byte store at a time
      for (uint64_t v = v0; v < v1; ++v) {
        w.refill();
        const uint32_t sym = symbol_slow(w, pair[w.peek12()], ct);
        const uint32_t sb = sm[v];
        out[v] = (uint16_t)(((sb & 0x80u) << 8) | (sym << 7) | (sb & 0x7Fu));
      }
    }
}

template <class W, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_exp_decode2(const __grid_constant__ DecodeParams p) {
  __shared__ uint32_t pair[1 << kPairBits];
  __shared__ uint32_t first_code[kCodecMaxLen + 1];
  __shared__ int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  __shared__ uint8_t sorted_sym[kCodecSymbols];
  const int tid = threadIdx.x;
  {
    const DecTables* t = p.tabs;
    const uint4* src = reinterpret_cast<const uint4*>(t->pair);
    uint4* dst = reinterpret_cast<uint4*>(pair);
    for (int i = tid; i < (1 << kPairBits) / 4; i += blockDim.x) dst[i] = src[i];
    if (tid <= kCodecMaxLen) {
      first_code[tid] = t->first_code[tid];
      count[tid] = t->count[tid];
      first_rank[tid] = t->first_rank[tid];
    }
    if (tid < kCodecSymbols) sorted_sym[tid] = t->sorted_sym[tid];
  }
  const CanonTabs ct{count, first_code, first_rank, sorted_sym, p.tabs->maxlen};
  __syncthreads();

  const uint64_t n = p.n;
  const uint64_t cpt = (n + p.chunk - 1) / p.chunk;  // chunks per tensor
  const uint64_t n_chunks = cpt * (uint64_t)p.ntensors;
  for (uint64_t gc = blockIdx.x * (uint64_t)blockDim.x + tid; gc < n_chunks; gc += (uint64_t)gridDim.x * blockDim.x) {
    const int ti = (int)(gc / cpt);
    const uint64_t c = gc - (uint64_t)ti * cpt;
    const DecodeTensor& d = p.t[ti];
    const uint8_t* __restrict__ sm = d.sm;
    uint16_t* __restrict__ out = d.out;
    const uint64_t v0 = c * p.chunk;
    const uint64_t v1 = (v0 + p.chunk < n) ? v0 + p.chunk : n;
    const uint32_t bitpos = d.index[c] - d.bit_base;
    W w;
    w.init(d.bits, bitpos);
    decode_chunk_v2(w, sm, out, v0, v1, pair, ct);
  }
}


// Decoder v6: the pair decoder of k_exp_decode2 with (a) one contiguous run of chunks per
// thread -- a tensor's stream is contiguous, so the window enters it once per run instead of
// once per chunk -- and (b) the stream fed through a per-thread shared-memory ring by cp.async
// (SWindow, codec_dev.cuh) instead of one-word-ahead global loads, which ncu put under ~25%
// of v2's stall samples (long scoreboard on the popped word).
constexpr int kRun6Bytes = 128;  // SWindow ring per thread
__global__ void __launch_bounds__(256) k_exp_decode6(const __grid_constant__ DecodeParams p) {
  __shared__ uint32_t pair[1 << kPairBits];
  __shared__ uint32_t first_code[kCodecMaxLen + 1];
  __shared__ int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  __shared__ uint8_t sorted_sym[kCodecSymbols];
  extern __shared__ __align__(16) uint8_t ring6[];  // 256 x kRun6Bytes
  const int tid = threadIdx.x;
  {
    const DecTables* t = p.tabs;
    const uint4* src = reinterpret_cast<const uint4*>(t->pair);
    uint4* dst = reinterpret_cast<uint4*>(pair);
    for (int i = tid; i < (1 << kPairBits) / 4; i += blockDim.x) dst[i] = src[i];
    if (tid <= kCodecMaxLen) {
      first_code[tid] = t->first_code[tid];
      count[tid] = t->count[tid];
      first_rank[tid] = t->first_rank[tid];
    }
    if (tid < kCodecSymbols) sorted_sym[tid] = t->sorted_sym[tid];
  }
  const CanonTabs ct{count, first_code, first_rank, sorted_sym, p.tabs->maxlen};
  __syncthreads();

  const uint64_t n = p.n;
  const uint64_t cpt = (n + p.chunk - 1) / p.chunk;  // chunks per tensor
  const uint64_t threads = (uint64_t)gridDim.x * blockDim.x;
  // runs of R consecutive chunks, never across tensors: about one run per thread
  const uint64_t R = (cpt * (uint64_t)p.ntensors + threads - 1) / threads;
  const uint64_t rpt = (cpt + R - 1) / R;  // runs per tensor
  const uint32_t ring = smem_u32(ring6 + tid * kRun6Bytes);
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < rpt * (uint64_t)p.ntensors; g += threads) {
    const int ti = (int)(g / rpt);
    const uint64_t c0 = (g - (uint64_t)ti * rpt) * R;
    const uint64_t c1 = c0 + R < cpt ? c0 + R : cpt;
    const DecodeTensor& d = p.t[ti];
    const uint8_t* __restrict__ sm = d.sm;
    uint16_t* __restrict__ out = d.out;
    const uint64_t v0 = c0 * p.chunk;
    const uint64_t v1 = (c1 * p.chunk < n) ? c1 * p.chunk : n;
    SWindow w;
    w.init(d.bits, d.index[c0] - d.bit_base, ring, (uint32_t)(tid & 7));
    const bool aligned = ((reinterpret_cast<uintptr_t>(out + v0) & 31) | (reinterpret_cast<uintptr_t>(sm + v0) & 15)) == 0;
    const uint64_t vf = aligned ? v0 + ((v1 - v0) & ~15ull) : v0;  // whole groups on the fast path
    if (vf > v0) {
      uint4 nsm = *reinterpret_cast<const uint4*>(sm + v0);
      for (uint64_t v = v0; v < vf; v += 16) {
        const uint4 smv = nsm;
        if (v + 16 < vf) nsm = *reinterpret_cast<const uint4*>(sm + v + 16);  // one group ahead
        const uint32_t smw[4] = {smv.x, smv.y, smv.z, smv.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((j & 1) == 0) w.refill();
          uint32_t e = pair[w.peek12()];
          const int len = (int)(e & 15u);
          if (__builtin_expect(len == 0, 0)) e = pair_slow(w, pair, ct);
          else w.p += len;
          const uint32_t dup = __byte_perm(smw[j >> 1], 0, (j & 1) ? 0x3322u : 0x1100u);
          o[j] = (dup & 0x807F807Fu) | (e & 0x7F807F80u);
        }
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + v), "r"(o[0]), "r"(o[1]),
                     "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                     : "memory");
      }
    }
    for (uint64_t v = vf; v < v1; ++v) {  // ragged tail / unaligned run: one symbol at a time
      w.refill();
      const uint32_t sym = symbol_slow(w, pair[w.peek12()], ct);
      const uint32_t sb = sm[v];
      out[v] = (uint16_t)(((sb & 0x80u) << 8) | (sym << 7) | (sb & 0x7Fu));
    }
  }
}


// Decoder v7: tile-staged.  A CTA takes a tile of up to 256 consecutive chunks of one tensor
// (64K values at chunk 256).  (A) One thread bulk-copies the tile's bitstream -- one
// contiguous byte range between two chunk-index entries -- into shared memory with the TMA
// engine.  (B) Thread t decodes chunk t from shared memory only (stream words and the pair
// table are LDS; no global load sits on the decode chain) into exponent bytes, stored in a
// swizzled per-chunk row.  (C) The CTA merges exponents with the sign/mantissa plane in one
// coalesced sweep: consecutive lanes read consecutive 16-byte pieces of the plane and write
// consecutive 32-byte pieces of bf16 output.  v2 issued per-lane loads and stores 256 B apart
// (one chunk per lane) and stalled on them (ncu: long scoreboard on the stream word first).
// Tiles whose stream exceeds the staging buffer, and each tensor's last tile (its stream end
// is not known to the kernel), decode chunk by chunk from global memory as v2 does.
constexpr int kTile7 = 256;  // chunks per tile = threads per CTA
__host__ __device__ constexpr int bits7_cap(int chunk) { return chunk >= 256 ? 28 * 1024 : 16 * 1024; }
__host__ __device__ constexpr int smem7_bytes(int chunk) {
  return bits7_cap(chunk) + kTile7 * chunk + (1 << kPairBits) * 4 + 64;
}

__device__ __forceinline__ uint32_t exp_pair_bytes(uint32_t ea, uint32_t eb) {
  // pair-table words (e0 << 7 | e1 << 23 | meta) -> [e0a e1a e0b e1b]
  return __byte_perm(ea >> 7, eb >> 7, 0x6420);
}

// Window over a stream staged in shared memory (word addresses, one word in flight).
struct LWindow {
  uint64_t win;
  int p;
  uint32_t nxt;
  uint32_t addr;  // smem address of the next word to load
  __device__ __forceinline__ void init(uint32_t word_addr, uint32_t bit_in_word) {
    uint32_t a, b;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(word_addr));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(b) : "r"(word_addr + 4));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nxt) : "r"(word_addr + 8));
    win = ((uint64_t)bswap32(a) << 32) | bswap32(b);
    addr = word_addr + 12;
    p = (int)bit_in_word;
  }
  __device__ __forceinline__ void refill() {
    if (p >= 32) {
      win = (win << 32) | bswap32(nxt);
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nxt) : "r"(addr));
      addr += 4;
      p -= 32;
    }
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

__global__ void __launch_bounds__(kTile7) k_exp_decode7(const __grid_constant__ DecodeParams p) {
  __shared__ uint32_t first_code[kCodecMaxLen + 1];
  __shared__ int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  __shared__ uint8_t sorted_sym[kCodecSymbols];
  __shared__ __align__(8) uint64_t bar;
  extern __shared__ __align__(16) uint8_t sm7[];
  const int chunk = p.chunk;
  const int cap = bits7_cap(chunk);
  uint8_t* tbits = sm7;                          // staged stream bytes of the tile
  uint8_t* tex = sm7 + cap;                      // exponent bytes: [chunk t][chunk] swizzled by 16 B
  uint32_t* pair = reinterpret_cast<uint32_t*>(tex + kTile7 * chunk);
  const int tid = threadIdx.x;
  {
    const DecTables* t = p.tabs;
    const uint4* src = reinterpret_cast<const uint4*>(t->pair);
    uint4* dst = reinterpret_cast<uint4*>(pair);
    for (int i = tid; i < (1 << kPairBits) / 4; i += blockDim.x) dst[i] = src[i];
    if (tid <= kCodecMaxLen) {
      first_code[tid] = t->first_code[tid];
      count[tid] = t->count[tid];
      first_rank[tid] = t->first_rank[tid];
    }
    if (tid < kCodecSymbols) sorted_sym[tid] = t->sorted_sym[tid];
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
    }
  }
  const CanonTabs ct{count, first_code, first_rank, sorted_sym, p.tabs->maxlen};
  __syncthreads();

  const uint64_t n = p.n;
  const uint64_t cpt = (n + chunk - 1) / chunk;
  const uint64_t tpt = (cpt + kTile7 - 1) / kTile7;  // tiles per tensor
  const uint64_t n_tiles = tpt * (uint64_t)p.ntensors;
  const int upc = chunk / 16;  // 16-byte units per chunk row of tex
  // a tile is staged when it is full, not the tensor's last (its stream end is known), aligned,
  // and its stream fits the buffer; returns the byte range to copy
  auto plan = [&](uint64_t tile, const uint8_t** g0, uint32_t* bytes) -> bool {
    const int ti = (int)(tile / tpt);
    const uint64_t c0 = (tile - (uint64_t)ti * tpt) * kTile7, c1 = c0 + kTile7;
    const DecodeTensor& d = p.t[ti];
    if (c1 >= cpt) return false;
    const uint32_t b0 = d.index[c0] - d.bit_base, b1 = d.index[c1] - d.bit_base;
    const uint64_t v0 = c0 * chunk;
    if (((reinterpret_cast<uintptr_t>(d.out + v0) & 31) | (reinterpret_cast<uintptr_t>(d.sm + v0) & 15) |
         (reinterpret_cast<uintptr_t>(d.bits) & 15)) != 0)
      return false;
    *g0 = reinterpret_cast<const uint8_t*>(d.bits) + ((b0 >> 3) & ~15u);
    // through the tile's last bit + 16 bytes (the window reads up to 96 bits past its position)
    *bytes = ((((b1 + 7) >> 3) + 16 + 15) & ~15u) - ((b0 >> 3) & ~15u);
    return *bytes <= (uint32_t)cap;
  };
  __shared__ int s_staged;
  uint32_t phase = 0;
  uint64_t prefetched = ~0ull;  // tile whose stream thread 0 already put in flight
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int ti = (int)(tile / tpt);
    const uint64_t j = tile - (uint64_t)ti * tpt;
    const DecodeTensor& d = p.t[ti];
    const uint64_t c0 = j * kTile7, c1 = (c0 + kTile7 < cpt) ? c0 + kTile7 : cpt;
    const uint64_t v0 = c0 * chunk, v1 = (c1 * chunk < n) ? c1 * chunk : n;
    const uint32_t my_bit = (c0 + tid < c1) ? d.index[c0 + tid] - d.bit_base : 0u;  // issued early
    if (tid == 0) {
      const uint8_t* g0 = nullptr;
      uint32_t bytes = 0;
      const bool st = plan(tile, &g0, &bytes);
      if (st && prefetched != tile) {
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_load_1d(tbits, g0, bytes, &bar);
      }
      s_staged = st ? 1 : 0;
    }
    __syncthreads();
    if (!s_staged) {
      // chunk by chunk from global memory (k_exp_decode2's loop)
      const uint64_t c = c0 + tid;
      if (c < c1) {
        Window w;
        w.init(d.bits, my_bit);
        const uint64_t a = c * chunk, b = (a + chunk < n) ? a + chunk : n;
        decode_chunk_v2(w, d.sm, d.out, a, b, pair, ct);
      }
      __syncthreads();  // s_staged is rewritten for the next tile
      continue;
    }
    const uint32_t base_bit = ((d.index[c0] - d.bit_base) >> 3 & ~15u) * 8;
    mbar_wait(&bar, phase);  // (A) the tile's stream is in tbits
    phase ^= 1;
    // (B) chunk tid: exponent bytes into its tex row
    {
      const uint32_t bit = my_bit - base_bit;
      LWindow w;
      w.init(smem_u32(tbits) + (bit >> 5) * 4, bit & 31);
      const uint32_t row = smem_u32(tex + tid * chunk);
      const uint32_t swz = (uint32_t)(tid & (upc - 1));
#pragma unroll 1
      for (int u = 0; u < upc; ++u) {
        uint32_t e[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if ((q & 1) == 0) w.refill();
          uint32_t x = pair[w.peek12()];
          const int len = (int)(x & 15u);
          if (__builtin_expect(len == 0, 0)) x = pair_slow(w, pair, ct);
          else w.p += len;
          e[q] = x;
        }
        const uint32_t o0 = exp_pair_bytes(e[0], e[1]), o1 = exp_pair_bytes(e[2], e[3]);
        const uint32_t o2 = exp_pair_bytes(e[4], e[5]), o3 = exp_pair_bytes(e[6], e[7]);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((((uint32_t)u) ^ swz) << 4)), "r"(o0),
                     "r"(o1), "r"(o2), "r"(o3)
                     : "memory");
      }
    }
    __syncthreads();
    // tbits is free: put the next tile's stream in flight under this tile's merge
    if (tid == 0) {
      const uint64_t nxt = tile + gridDim.x;
      const uint8_t* g0 = nullptr;
      uint32_t bytes = 0;
      if (nxt < n_tiles && plan(nxt, &g0, &bytes)) {
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_load_1d(tbits, g0, bytes, &bar);
        prefetched = nxt;
      }
    }
    // (C) coalesced merge with the sign/mantissa plane, 4 units per thread in flight
    const uint32_t units = (uint32_t)((v1 - v0) / 16);  // a multiple of 4 * kTile7 on staged tiles
    const uint4* smp = reinterpret_cast<const uint4*>(d.sm + v0);
    for (uint32_t i0 = tid; i0 < units; i0 += 4 * kTile7) {
      uint4 smv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) smv[r] = __ldg(smp + i0 + r * kTile7);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t i = i0 + r * kTile7;
        const uint32_t cc = i / upc, uu = i % upc;
        uint4 ex;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(ex.x), "=r"(ex.y), "=r"(ex.z), "=r"(ex.w)
                     : "r"(smem_u32(tex + cc * chunk) + ((uu ^ (cc & (upc - 1))) << 4)));
        uint16_t* o = d.out + v0 + 16 * (uint64_t)i;
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o),
                     "r"(pack_words(smv[r].x, ex.x, 0x5140u)), "r"(pack_words(smv[r].x, ex.x, 0x7362u)),
                     "r"(pack_words(smv[r].y, ex.y, 0x5140u)), "r"(pack_words(smv[r].y, ex.y, 0x7362u)),
                     "r"(pack_words(smv[r].z, ex.z, 0x5140u)), "r"(pack_words(smv[r].z, ex.z, 0x7362u)),
                     "r"(pack_words(smv[r].w, ex.w, 0x5140u)), "r"(pack_words(smv[r].w, ex.w, 0x7362u))
                     : "memory");
      }
    }
    __syncthreads();  // tex is reused by the next tile
  }
}

void launch_exp_decode(const uint8_t* sm, const uint32_t* bits, const uint32_t* index, uint64_t n, int chunk,
                       const CodecTable& table, uint16_t* out, cudaStream_t s, uint32_t bit_base) {
  DecodeTensor t{sm, bits, index, out, bit_base};
  launch_exp_decode_multi(&t, 1, n, chunk, table, s);
}

// Device tables per (device, codec table), built once on first use (synchronously, so a
// decode on any stream may read them) and kept for the process.
static const DecTables* decode_tables(const CodecTable& table, cudaStream_t s) {
  struct Entry {
    int dev;
    CodecTable t;
    DecTables* d;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.dev == dev && memcmp(e.t.len, table.len, sizeof(table.len)) == 0) return e.d;
  DecTables* d = nullptr;
  if (cudaMalloc(&d, sizeof(DecTables)) != cudaSuccess) return nullptr;
  k_build_tables<<<1, 256, 0, s>>>(table, d);
  note_launch();
  if (cudaStreamSynchronize(s) != cudaSuccess) return nullptr;
  cache.push_back(Entry{dev, table, d});
  return d;
}

void prepare_decode_tables(const CodecTable& table, cudaStream_t s) { decode_tables(table, s); }

const DecTables* codec_device_tables(const CodecTable& table, cudaStream_t s) { return decode_tables(table, s); }

void launch_exp_decode_multi(const DecodeTensor* tensors, int ntensors, uint64_t n, int chunk, const CodecTable& table,
                             cudaStream_t s) {
  if (n == 0 || ntensors <= 0) return;
  DecodeParams p;
  p.ntensors = ntensors;
  p.n = n;
  p.chunk = chunk;
  p.tabs = decode_tables(table, s);
  if (!p.tabs) return;  // the caller's CKLAUNCH reports the CUDA error
  for (int i = 0; i < ntensors; ++i) p.t[i] = tensors[i];
  const uint64_t n_chunks = ((n + chunk - 1) / chunk) * (uint64_t)ntensors;
  // one resident wave, grid-striding over the chunks: a second partial wave left the
  // tail idle (chunk 256: 1265 GB/s at 5 blocks/SM vs 1107 at 8)
  static const int resident = [] {
    int dev = 0, sms = 148, per_sm = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode, 256, 0);
    return std::max(1, sms * std::max(1, per_sm));
  }();
  // XPGB_DECODER=1: the round-1 multi-symbol decoder; 3: the pair decoder fed from a 16-byte
  // stream queue (QWindow); 4 / 5: 2 / 3 stream words in flight; 6: contiguous chunk runs per
  // thread fed through a shared-memory ring (k_exp_decode6); 7: tile-staged (k_exp_decode7);
  // default 2 (A/B only)
  static const int ver = [] {
    const char* e = getenv("XPGB_DECODER");
    return e ? atoi(e) : 2;
  }();
  if (ver == 1) {
    const uint64_t blocks = std::min<uint64_t>((n_chunks + 255) / 256, (uint64_t)resident);
    k_exp_decode<<<(unsigned)blocks, 256, 0, s>>>(p);
  } else {
    static const int resident2 = [] {
      int dev = 0, sms = 148, per_sm = 4;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode2<Window>, 256, 0);
      return std::max(1, sms * std::max(1, per_sm));
    }();
    const uint64_t blocks = std::min<uint64_t>((n_chunks + 255) / 256, (uint64_t)resident2);
    if (ver == 7 && chunk % 16 == 0 && chunk <= 256 && (chunk & (chunk - 1)) == 0) {
      static int resident7[2] = {0, 0};  // chunk 256 / below
      const int ci = chunk >= 256 ? 0 : 1;
      if (!resident7[ci]) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_exp_decode7, cudaFuncAttributeMaxDynamicSharedMemorySize, smem7_bytes(256));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode7, kTile7, smem7_bytes(chunk));
        resident7[ci] = std::max(1, sms * std::max(1, per_sm));
      }
      const uint64_t tiles = ((n + (uint64_t)chunk * kTile7 - 1) / ((uint64_t)chunk * kTile7)) * ntensors;
      const uint64_t b7 = std::min<uint64_t>(tiles, (uint64_t)resident7[ci]);
      k_exp_decode7<<<(unsigned)b7, kTile7, smem7_bytes(chunk), s>>>(p);
    } else if (ver == 6) {
      static const int resident6 = [] {
        int dev = 0, sms = 148, per_sm = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_exp_decode6, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * kRun6Bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode6, 256, 256 * kRun6Bytes);
        return std::max(1, sms * std::max(1, per_sm));
      }();
      const uint64_t b6 = std::min<uint64_t>((n_chunks + 255) / 256, (uint64_t)resident6);
      k_exp_decode6<<<(unsigned)b6, 256, 256 * kRun6Bytes, s>>>(p);
    } else if (ver == 3) k_exp_decode2<QWindow><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (ver == 4) k_exp_decode2<WindowD<2>><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (ver == 5) k_exp_decode2<WindowD<3>><<<(unsigned)blocks, 256, 0, s>>>(p);
    else if (ver == 8 || ver == 9) {  // register-capped for 6 / 8 resident CTAs per SM (occupancy A/B)
      static int res8[2] = {0, 0};
      const int vi = ver - 8;
      if (!res8[vi]) {
        int dev = 0, sms = 148, per_sm = 4;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (vi == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode2<Window, 6>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exp_decode2<Window, 8>, 256, 0);
        res8[vi] = std::max(1, sms * std::max(1, per_sm));
      }
      const uint64_t b8 = std::min<uint64_t>((n_chunks + 255) / 256, (uint64_t)res8[vi]);
      if (vi == 0) k_exp_decode2<Window, 6><<<(unsigned)b8, 256, 0, s>>>(p);
      else k_exp_decode2<Window, 8><<<(unsigned)b8, 256, 0, s>>>(p);
    }
    else k_exp_decode2<Window><<<(unsigned)blocks, 256, 0, s>>>(p);
  }
  note_launch();
}

}  // namespace xpgb
