// Device-side exponent-Huffman decode primitives shared by the standalone decoder
// (codec.cu) and the decode-into-GEMM kernel (moe_gemm_dec.cu).
#pragma once
#include <cstdint>

#include "codec.cuh"

namespace xpgb {

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

constexpr int kMultiBits = 11;

__device__ __forceinline__ int canon_decode(uint64_t win, int ml, const int* count, const uint32_t* first_code,
                                            const int* first_rank, const uint8_t* sorted_sym, int* sym) {
  for (int l = 1; l <= ml; ++l) {
    const uint32_t code = (uint32_t)(win >> (64 - l));
    if (count[l] && code - first_code[l] < (uint32_t)count[l]) {
      *sym = sorted_sym[first_rank[l] + (code - first_code[l])];
      return l;
    }
  }
  return 0;  // invalid code: the host index scan rejects such streams before they get here
}

// Decode tables of one codec table, built once by k_build_tables and copied into every
// decoder CTA's shared memory (building them per CTA cost ~20 us per launch -- most of a
// small tensor's decode).
constexpr int kPairBits = 12;
struct DecTables {
  uint32_t lut3[1 << kMultiBits];  // up to 4 symbols (4 x 8 b)
  uint8_t lmeta[1 << kMultiBits];  // count | total length << 3
  uint32_t pair[1 << kPairBits];   // k_exp_decode2's pair table (see there)
  uint32_t first_code[kCodecMaxLen + 1];
  int count[kCodecMaxLen + 1], first_rank[kCodecMaxLen + 1];
  uint8_t sorted_sym[kCodecSymbols];
  int maxlen;
};

struct Window {
  uint64_t win;  // bits [0, 64) of the stream from the current word, MSB first
  int p;         // bits already consumed from the top of `win`
  uint32_t nxt;  // next stream word (raw, in flight)
  const uint32_t* wp;
  __device__ __forceinline__ void init(const uint32_t* bits, uint32_t bitpos) {
    wp = bits + (bitpos >> 5);
    win = ((uint64_t)bswap32(wp[0]) << 32) | bswap32(wp[1]);
    nxt = wp[2];
    wp += 3;
    p = (int)(bitpos & 31);
  }
  __device__ __forceinline__ void refill() {
    if (p >= 32) {
      win = (win << 32) | bswap32(nxt);
      nxt = *wp++;
      p -= 32;
    }
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

// Stream window fed from a 16-byte register queue: a word is popped per 32 bits consumed and
// a new 16-byte load is issued every 4 words, so the next load is ~4 words (~24 values)
// ahead of use -- the decoder is latency-bound (ncu: long-scoreboard stalls on the one-word-ahead
// Window), and the decode-into-GEMM kernel has only 8 decoder warps per SM to hide it with.
struct QWindow {
  uint64_t win;
  int p;
  int qi;            // next word of `cur` to pop (0..3)
  uint4 cur, nxt;
  const uint4* qp;   // next 16-byte block to load
  __device__ __forceinline__ uint32_t pop() {
    const uint32_t r = qi == 0 ? cur.x : qi == 1 ? cur.y : qi == 2 ? cur.z : cur.w;
    if (++qi == 4) {
      cur = nxt;
      nxt = __ldg(qp++);
      qi = 0;
    }
    return r;
  }
  __device__ __forceinline__ void init(const uint32_t* bits, uint32_t bitpos) {
    const uint32_t* w0 = bits + (bitpos >> 5);
    const uintptr_t a = reinterpret_cast<uintptr_t>(w0);
    const uint4* b = reinterpret_cast<const uint4*>(a & ~uintptr_t(15));
    cur = __ldg(b);
    nxt = __ldg(b + 1);
    qp = b + 2;
    qi = (int)((a >> 2) & 3);
    const uint32_t hi = bswap32(pop());
    const uint32_t lo = bswap32(pop());
    win = ((uint64_t)hi << 32) | lo;
    p = (int)(bitpos & 31);
  }
  __device__ __forceinline__ void refill() {
    if (p >= 32) {
      win = (win << 32) | bswap32(pop());
      p -= 32;
    }
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

// Window with D stream words in flight (D = 1 is Window): ncu of the one-word-ahead decoder
// puts ~25% of its stall samples on the byte swap of the word it just popped (the load
// issued only ~6 values earlier); each extra word in flight costs one register move.
template <int D>
struct WindowD {
  uint64_t win;
  int p;
  uint32_t q[D];  // next D stream words (raw), q[0] first
  const uint32_t* wp;
  __device__ __forceinline__ void init(const uint32_t* bits, uint32_t bitpos) {
    wp = bits + (bitpos >> 5);
    win = ((uint64_t)bswap32(wp[0]) << 32) | bswap32(wp[1]);
#pragma unroll
    for (int i = 0; i < D; ++i) q[i] = wp[2 + i];
    wp += 2 + D;
    p = (int)(bitpos & 31);
  }
  __device__ __forceinline__ void refill() {
    if (p >= 32) {
      win = (win << 32) | bswap32(q[0]);
#pragma unroll
      for (int i = 0; i + 1 < D; ++i) q[i] = q[i + 1];
      q[D - 1] = *wp++;
      p -= 32;
    }
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// Stream window of one decoder thread, fed through shared memory.  In the decode-into-GEMM
// kernel a decoder thread reads its own tensor row's stream -- 256 threads, 256 streams far
// apart -- and with ~200 KB of the SM in shared memory the L1 cannot hold a line per stream: word-by-word global loads missed to
// L2 on nearly every refill (measured: the fused GEMM ran ~8x slower than the standalone
// decoder).  Here the stream is copied ahead with cp.async (LDGSTS, bypassing L1) into a
// per-thread ring of two 64-byte blocks; the window pops words from it with LDS.  A block is
// refetched as soon as the window leaves it, so the copy runs ~64 bytes (~200 values) ahead.
// The ring's 16-byte chunks are XOR-swizzled by the thread index to spread banks.
struct SWindow {
  uint64_t win;
  int p;
  uint32_t nxt;     // next stream word (raw)
  uint32_t wi;      // ring word (0..31) that follows nxt
  uint32_t base;    // smem address of this thread's ring
  uint32_t sw;      // chunk swizzle (thread & 7)
  const uint8_t* g; // global address of the next block to fetch
  __device__ __forceinline__ uint32_t word(uint32_t w) const {
    return lds32(base + ((((w >> 2) ^ sw)) << 4) + ((w & 3) << 2));
  }
  __device__ __forceinline__ void fetch(uint32_t slot) {  // 64 bytes into ring words [16 slot, 16 slot + 16)
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) cp_async16(base + (((slot * 4 + i) ^ sw) << 4), g + 16 * i);
    cp_async_commit();
    g += 64;
  }
  __device__ __forceinline__ void init(const uint32_t* bits, uint32_t bitpos, uint32_t ring, uint32_t swz) {
    base = ring;
    sw = swz;
    const uintptr_t a = reinterpret_cast<uintptr_t>(bits + (bitpos >> 5));
    g = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(15));
    const uint32_t w0 = (uint32_t)((a >> 2) & 3);
    fetch(0);
    fetch(1);
    cp_async_wait1();
    win = ((uint64_t)bswap32(word(w0)) << 32) | bswap32(word(w0 + 1));
    nxt = word(w0 + 2);
    wi = w0 + 3;
    p = (int)(bitpos & 31);
  }
  __device__ __forceinline__ uint32_t pop() {
    const uint32_t r = nxt;
    if ((wi & 15) == 0) {  // entering the other block: the one just left is free
      fetch(((wi >> 4) ^ 1) & 1);
      cp_async_wait1();
    }
    nxt = word(wi);
    wi = (wi + 1) & 31;
    return r;
  }
  __device__ __forceinline__ void refill() {
    if (p >= 32) {
      win = (win << 32) | bswap32(pop());
      p -= 32;
    }
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

struct CanonTabs {
  const int* count;
  const uint32_t* first_code;
  const int* first_rank;
  const uint8_t* sorted_sym;
  int ml;
};

// One exponent symbol the slow way (p < 32 on entry, so >= 32 bits are valid).
template <class W>
__device__ __forceinline__ uint32_t symbol_slow(W& w, uint32_t ent, const CanonTabs& ct) {
  int l = (int)((ent >> 16) & 31);
  uint32_t sym = (ent >> 7) & 0xFFu;
  if (!l) {
    int s = 0;
    l = canon_decode(w.win << w.p, ct.ml, ct.count, ct.first_code, ct.first_rank, ct.sorted_sym, &s);
    sym = (uint32_t)s;
  }
  w.p += l;
  return sym;
}

// A pair that does not fit the table: two single symbols; leaves p < 32.
template <class W>
__device__ __forceinline__ uint32_t pair_slow(W& w, const uint32_t* __restrict__ pair, const CanonTabs& ct) {
  w.refill();
  const uint32_t a = symbol_slow(w, pair[w.peek12()], ct);
  w.refill();
  const uint32_t b = symbol_slow(w, pair[w.peek12()], ct);
  w.refill();
  return (a << 7) | (b << 23);
}

}  // namespace xpgb
