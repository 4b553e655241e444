// Exponent-only canonical Huffman codec for bf16 (bit-compatible with xpg codec.py).
//
// Stream convention (codec.py:1-10, 235-272): one table per model over the 256
// exponent byte values; canonical codes assigned in (length, symbol) order;
// codewords packed MSB-first; the last byte is zero-padded.  The sign/mantissa
// plane is one raw byte per value ((w >> 8) & 0x80 | w & 0x7F).
//
// B200 addition: a chunk index — the bit offset at which every block of
// `chunk` values starts — so thousands of GPU threads can decode one tensor's
// sequential stream in parallel.  It is side metadata; the stream bytes are
// exactly the reference's.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace xpgb {

constexpr int kCodecSymbols = 256;
constexpr int kCodecMaxLen = 32;
constexpr int kLutBits = 12;

struct CodecTable {
  uint8_t len[kCodecSymbols];
};

// Canonical code of every symbol from its length (0 = absent).  Returns false
// if the lengths violate Kraft or exceed 32.
bool codec_canonical_codes(const uint8_t* lengths, uint32_t* codes);

// Exponent histogram of a bf16 byte buffer (multi-threaded).
void codec_histogram(const uint8_t* data, size_t bytes, uint64_t* counts, int threads);

// Encode one tensor: returns false (and sets *missing) when an exponent has no codeword.
// sm_out: n bytes; bits_out: capacity `bits_cap` bytes; index_out: ceil(n/chunk) entries.
bool codec_encode(const uint16_t* words, size_t n, const uint8_t* lengths, const uint32_t* codes, uint8_t* sm_out,
                  uint8_t* bits_out, size_t bits_cap, size_t* bits_len, uint64_t* bit_count, uint32_t* index_out,
                  int chunk, int* missing);

// Host scan: chunk index + validation (0 ok, 1 truncated, 2 invalid code).
int codec_build_index(const uint8_t* bits, size_t bits_len, size_t n, const uint8_t* lengths, int chunk,
                      uint32_t* index_out, size_t* consumed_bits);

// Upper bound of the stream bytes of n values under `lengths`.
size_t codec_bits_bound(size_t n, const uint8_t* lengths);

// One tensor of a multi-tensor decode launch: stream pointers (index entries minus
// bit_base give bit offsets into `bits`) and the destination of its n values.
struct DecodeTensor {
  const uint8_t* sm;
  const uint32_t* bits;
  const uint32_t* index;
  uint16_t* out;
  uint32_t bit_base;
};
constexpr int kMaxDecodeTensors = 64;
// Builds (once per device and table) the decode tables every decoder launch copies into
// shared memory; launch_exp_decode* build them lazily, a context builds them up front.
void prepare_decode_tables(const CodecTable& table, cudaStream_t s);
// The prebuilt device tables (codec_dev.cuh) of `table`, built on first use.
struct DecTables;
const DecTables* codec_device_tables(const CodecTable& table, cudaStream_t s);

// GPU decode: bits must be readable as 32-bit words up to round_up(bits_len, 4) + 8 bytes.
// bit_base is subtracted from every index entry (decoding one staged piece of a stream).
void launch_exp_decode(const uint8_t* sm, const uint32_t* bits, const uint32_t* index, uint64_t n, int chunk,
                       const CodecTable& table, uint16_t* out, cudaStream_t s, uint32_t bit_base = 0);
// Up to kMaxDecodeTensors tensors of n values each in one launch (one staged run of
// consecutive records, or consecutive device-tier records of a layer).
void launch_exp_decode_multi(const DecodeTensor* tensors, int ntensors, uint64_t n, int chunk, const CodecTable& table,
                             cudaStream_t s);
constexpr uint64_t kStagePieceBytes = 64ull << 20;  // max bytes of one staged record piece
constexpr int kMaxStageBufs = 16;                   // staging buffers per kind (ring of pieces)

}  // namespace xpgb
