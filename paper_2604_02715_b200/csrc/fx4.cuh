// FX4: a fixed-width exponent format for the compressed *device* tier (a B200 addition; the
// reference's device tier is exponent-Huffman, codec.py:235-272).
//
// Huffman exponents (~2.6 bits) are the smallest encoding, but decoding them is a serial
// dependency chain per stream (window shift -> table load -> length -> next shift), and a GEMM
// that expands weights on the fly cannot hide that chain with enough warps (moe_gemm_dec.cu,
// profiles/r2_fused_*.jsonl).  FX4 stores each exponent as a 4-bit offset from a per-tensor
// base, so every value's code sits at a fixed bit position: a 16-byte load carries 32 codes
// and decoding is a table lookup per pair with no dependency between pairs.  The price is
// bytes: 12.1 bits per value instead of 10.7 (ratio 0.758 vs 0.662), which is why the planner
// uses it only where the step is SM-bound rather than link-bound.
//
// Record of one tensor of n values (n % 256 == 0), every part 16-byte aligned:
//   sm    n bytes           sign/mantissa plane ((w >> 8) & 0x80 | w & 0x7F), as the Huffman record
//   nib   n / 2 bytes       value i's code in byte i/2, low nibble for even i: exponent - base,
//                           15 = escape (exponent outside [base, base + 14])
//   idx   ns + 1 uint32     escapes before each 256-value segment (ns = n / 256), exclusive prefix
//   esc   total bytes       exponent bytes of the escaped values, in value order (+16 slack)
// The base is chosen per tensor to cover the most values (15-wide window of the histogram),
// at most kFxMaxBase: decoders add it to four codes in one 32-bit add, so base + 15 must fit a byte.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace xpgb {

constexpr int kFxSeg = 256;  // values per escape-index segment
constexpr int kFxMaxBase = 240;  // base + 15 <= 255

struct FxLayout {
  uint64_t n, nib, idx, esc, total;  // byte offsets (sm at 0) and record size
};

inline uint64_t fx_round16(uint64_t x) { return (x + 15) & ~15ull; }

inline FxLayout fx_layout(uint64_t n, uint64_t n_esc) {
  FxLayout l;
  l.n = n;
  l.nib = fx_round16(n);
  l.idx = l.nib + fx_round16(n / 2);
  l.esc = l.idx + fx_round16(4 * (n / kFxSeg + 1));
  l.total = l.esc + fx_round16(n_esc) + 16;
  return l;
}

// Encode one bf16 tensor already in device memory into `rec` (device, fx_layout(n, esc).total
// bytes).  Two passes: histogram + escape counts, then the write; returns the escape count and
// base through the pointers.  Synchronises `s` (device-tier staging is setup, not the hot path).
// scratch: >= (n / 256 + 1) * 4 + 1024 bytes of device memory.
void fx4_count(const uint16_t* raw, uint64_t n, uint32_t* scratch, int* base, uint64_t* n_esc, cudaStream_t s);
void fx4_encode(const uint16_t* raw, uint64_t n, int base, uint32_t* scratch, uint8_t* rec, cudaStream_t s);
// Expand a record into bf16 (the non-fused paths: prefill-sized groups, external compute).
void launch_fx4_decode(const uint8_t* rec, uint64_t n, int base, uint16_t* out, cudaStream_t s);

}  // namespace xpgb
