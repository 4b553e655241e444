// Device-side data structures shared by the MoE kernels and the runtime.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace xpgb {

constexpr int kBM = 128;        // UMMA M: weight rows per tile
constexpr int kBK = 64;         // K elements per stage (one 128-B swizzle atom of bf16)
constexpr int kBoxRowsB = 16;   // activation rows per TMA box
constexpr int kMaxExperts = 1024;
constexpr int kMaxTopK = 32;

// Device page-table entry: -1 = unmapped, else (block0 << 2) | state.
__host__ __device__ inline int32_t pt_entry(int32_t block0, int32_t state) { return (block0 << 2) | state; }
__host__ __device__ inline int32_t pt_state(int32_t e) { return e < 0 ? 0 : (e & 3); }
__host__ __device__ inline int32_t pt_block0(int32_t e) { return e < 0 ? -1 : (e >> 2); }

// Fault word (first fault wins): bit0 set | kind << 1 | state << 3 | expert << 8 | layer << 32.
__host__ __device__ inline long long fault_pack(int layer, int expert, int kind, int state) {
  return 1LL | ((long long)kind << 1) | ((long long)state << 3) | ((long long)expert << 8) |
         ((long long)layer << 32);
}

// Routing + expert-major permutation of one layer (written by k_route_plan).
struct PlanView {
  int32_t* topk;     // [T][kk] routed ids (1-based, ascending)
  int32_t* pos;      // [T][kk] row of the (token, slot) pair in expert-major order, -1 if not local
  int32_t* offsets;  // [E+1] row ranges per local expert
};

// Activations reach the tensor cores as two bf16 planes, x = hi + lo with hi = bf16_rn(x)
// and lo = bf16_rn(x - hi): every activation row buffer (expert-major x rows, h rows) holds
// the hi rows, then the lo rows `lo_rows` rows later.  A contraction issues one MMA per plane
// into the same fp32 accumulator, so the weights (exact bf16, as the reference widens them,
// model.py:130-139) meet activations carried to ~2^-17 relative instead of bf16's 2^-9 --
// the reference computes x and h in float32 (pipeline.py:180-208).  At decode the GEMMs are
// HBM-bound on the weights, so the second MMA costs no time.
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  *hi = __float2bfloat16_rn(v);
  *lo = __float2bfloat16_rn(v - __bfloat162float(*hi));
}

// K blocks [kb0, kb1) of split s of S over KB blocks of kBK: boundaries on multiples of 4
// blocks (256 values) when KB allows, so a split starts on a codec chunk boundary and the
// decode-into-GEMM kernel sums exactly the same K ranges as k_moe_gemm (bit-identical).
__host__ __device__ inline void split_kb(int s, int S, int KB, int* kb0, int* kb1) {
  if (KB % 4 == 0) {
    const int n = KB / 4;
    *kb0 = (s * n / S) * 4;
    *kb1 = ((s + 1) * n / S) * 4;
  } else {
    *kb0 = s * KB / S;
    *kb1 = (s + 1) * KB / S;
  }
}

// A device-tier expert tensor read in place by the decode-into-GEMM kernel
// (moe_gemm_dec.cu): its exponent-Huffman record (sign/mantissa plane, bitstream, chunk
// index; index entries minus bit_base are bit offsets into `bits`).
// FX4 records (fx4.cuh) reuse the fields: bits = the nibble plane, index = the escape index,
// bit_base = the tensor's base exponent, esc = the escape bytes.
struct DecRec {
  const uint8_t* sm;
  const uint32_t* bits;
  const uint32_t* index;
  uint32_t bit_base;
  uint32_t fmt;  // 0 exponent-Huffman, 1 FX4
  const uint8_t* esc;
  const CUtensorMap* maps;  // FX4: 2-D maps of the sign/mantissa plane [rows][K] and nibbles [rows][K/2]
};

// Arguments of one grouped-GEMM launch (gate/up or down) of one layer.
struct GemmParams {
  const int32_t* offsets;  // [E+1]
  const int32_t* pt;       // [E] device page-table entries of (layer, kind)
  long long* fault;
  long long act_lo_rows;   // rows between the hi and lo planes of the activation operand (x or h)
  long long h_lo_rows;     // rows between the hi and lo planes of hbuf (the gate/up output)
  __nv_bfloat16* hbuf;     // gate/up output  [2][h_lo_rows][F] bf16 (hi plane, lo plane)
  float* part;             // down output     [splits][rows][H] fp32
  long long split_stride;  // elements between split planes of `part`
  int layer, e_first, E, F, H, splits;
  int E_routed;       // groups [0, E_routed) are paged experts (slot table); [E_routed, E) shared experts
  int shared_block0;  // block of this layer's first shared expert in the shared-weights maps
  // per group of the launch: groups whose record pointer is set run in the decode-into-GEMM
  // kernel and are skipped by k_moe_gemm (nullptr: no fused groups)
  const DecRec* dec;
  uint32_t dec_fmt_mask;  // bit f: records of format f are read in place by k_moe_gemm_dec in this layer
  // gate/up -> down overlap of the decode-into-GEMM kernels (nullptr: off): the gate/up launch
  // counts each group's finished units here and lets the down launch start early (programmatic
  // dependent launch); the down launch waits per group for all of that group's gate/up units
  int* unit_done;
  int unit_bn;  // token-tile width of the gate/up launch whose units unit_done counts (k_moe_gemm)
  int act_lo;   // 1: the activations' lo plane is multiplied too (fp32-like); 0: the hi plane only
                // (bf16 activations, half the MMAs; xpgb_set_activation_planes) -- 1-CTA kernels
};

// ---- launchers (moe_kernels.cu)
void launch_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int32_t* out,
                  cudaStream_t s);
// Route + count + scan + positions for `layer_count` layers.  Up to kPlanSingleCtaPairs
// (token, slot) pairs per layer: one fused CTA per layer; above: route+count over
// token blocks, then scan+place over pair blocks (scratch: 2*layer_count*E int32).
// Views for layer i live at topk/pos + i*T*kk and offsets + i*(E+1).
constexpr int kPlanSingleCtaPairs = 128;
// S shared experts per layer join every token of [sh0, sh1) after its routed slots (ids
// L+1..L+S, groups E..E+S-1; other tokens get id 0 / pos -1 there): plan rows are
// [T][kk+S], offsets [E+S+1].
void launch_route_plan(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int e_first, int E,
                       int S, int sh0, int sh1, int32_t* topk, int32_t* pos, int32_t* offsets, int32_t* scratch,
                       const long long* fault, cudaStream_t s);
// xp: hi plane; its lo plane starts lo_rows rows later.
void launch_gather(const float* x, const int32_t* pos, const long long* fault, __nv_bfloat16* xp, long long lo_rows,
                   int T, int kk, int H, cudaStream_t s);
// map_ws: the shared experts' weights (read for groups >= p.E_routed).
// lean: one stage fewer so exponent-decoder CTAs co-reside (paged runs with a compressed tier)
void launch_gate_up(const CUtensorMap& map_w, const CUtensorMap& map_x, const CUtensorMap& map_ws,
                    const GemmParams& p, int bn, int grid, cudaStream_t s, bool lean = false);
void launch_down(const CUtensorMap& map_w, const CUtensorMap& map_h, const CUtensorMap& map_ws,
                 const GemmParams& p, int bn, int grid, cudaStream_t s, bool lean = false);
// y_t = ordered weighted sum of the token's kk expert rows (the first kr scaled by
// inv_k, the rest -- shared experts -- by 1); optionally also writes bf16(y_t) to
// the next layer's expert-major rows (fused gather).
// accumulate: y_t starts from its current value (a later pass adds shared experts).
void launch_combine(const float* part, const int32_t* pos, const long long* fault, float* y, int T, int kk, int kr,
                    int H, int splits, long long split_stride, float inv_k, const int32_t* next_pos,
                    __nv_bfloat16* xp, long long lo_rows, cudaStream_t s, bool accumulate = false);
void launch_shared_plan(int32_t* pos, int32_t* off, int T, int S, cudaStream_t s);
void launch_reduce_rows(const float* part, const long long* fault, float* out, int n_rows, int H, int splits,
                        long long split_stride, cudaStream_t s);
void set_gemm_attrs();
// CTA-pair (cta_group::2) grouped GEMM for prefill-sized expert groups (moe_gemm_pair.cu):
// 256 token rows x 256 weight rows per pair, unsplit (down writes split plane 0).
bool pair_gemm_supported(int H, int F);
void set_pair_gemm_attrs();
// split: the token rows' lo plane is a second MMA per K step (as the 1-CTA kernel always
// does); false takes bf16 activations only (2x the tensor throughput at prefill, per-layer
// rel-L2 ~3e-3 instead of ~1e-6; XPGB_FAST_PREFILL=1).
// Decode-into-GEMM (moe_gemm_dec.cu): the groups g with p.dec[g].sm set, weights expanded
// from their compressed records into the UMMA tiles on-chip.  Needs K % chunk == 0 for both
// projections (a split starts on a chunk boundary) and H % 256 == 0.
struct CodecTable;
bool gemm_dec_supported(int H, int F, int chunk);
void set_gemm_dec_attrs();
void launch_gemm_dec(bool gate_up, const CUtensorMap& map_b, const GemmParams& p, const CodecTable& table, int chunk,
                     int bn, int grid, cudaStream_t s, bool fx4 = false);
void launch_gemm_pair(bool gate_up, const CUtensorMap& map_x, const CUtensorMap& map_w, const CUtensorMap& map_ws,
                      const GemmParams& p, int num_sms, cudaStream_t s, bool split = true);

}  // namespace xpgb
