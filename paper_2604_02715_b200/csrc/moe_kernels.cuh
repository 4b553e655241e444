// Device-side data structures shared by the MoE kernels and the runtime.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace xpgb {

constexpr int kBM = 128;         // UMMA M: weight rows per tile
constexpr int kBK = 64;          // K elements per stage (one 128-B swizzle atom of bf16)
constexpr int kBoxRowsB = 16;    // activation rows per TMA box
constexpr int kMaxExperts = 1024;
constexpr int kMaxTopK = 32;

// Device page-table entry: -1 = unmapped, else (block0 << 2) | state.
__host__ __device__ inline int32_t pt_entry(int32_t block0, int32_t state) { return (block0 << 2) | state; }
__host__ __device__ inline int32_t pt_state(int32_t e) { return e < 0 ? 0 : (e & 3); }
__host__ __device__ inline int32_t pt_block0(int32_t e) { return e < 0 ? -1 : (e >> 2); }

// Fault word layout (first fault wins): 1 | kind<<1 | state<<3 | expert<<5 | layer<<16 ... packed in int64.
__host__ __device__ inline long long fault_pack(int layer, int expert, int kind, int state) {
  return 1LL | ((long long)kind << 1) | ((long long)state << 3) | ((long long)expert << 8) |
         ((long long)layer << 32);
}

// One unit of grouped-GEMM work.
struct __align__(16) GemmUnit {
  int32_t expert;     // local expert index (0-based in the context's shard)
  int32_t m0;         // first weight row of the tile
  int32_t row_begin;  // first activation row (expert-major pair order)
  int32_t n_and_split;  // n_rows | split << 16
};

// Per-layer forward workspace (device pointers), owned by the runtime.
struct LayerWork {
  int32_t* topk;        // [T][kk] routed ids (1-based), this layer
  int32_t* pos;         // [T][kk] row of the (token, slot) pair in expert-major order, -1 if not local
  int32_t* offsets;     // [E+1]
  int32_t* slot_gu;     // [E] 0-based block of GATE_UP page, -1 if not read
  int32_t* slot_dn;     // [E]
  GemmUnit* units1;     // gate/up units
  GemmUnit* units2;     // down units
  int32_t* counters;    // [0] = n_units1, [1] = n_units2, [2] = n_pairs
  __nv_bfloat16* xp;    // [cap_rows][H] gathered bf16 rows
  __nv_bfloat16* hbuf;  // [cap_rows][F] SwiGLU activations
  float* part;          // [splits][cap_rows][H] down partials
  long long* fault;     // fault word
};

// ---- launchers (moe_kernels.cu) ----
void launch_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int32_t* out,
                  cudaStream_t s);
void launch_plan(const LayerWork& w, const int32_t* pt_table_gu, const int32_t* pt_table_dn, int layer, int T,
                 int kk, int e_first, int e_count, int F, int H, int bn1, int bn2, int splits, cudaStream_t s);
void launch_plan_rows(const LayerWork& w, const int32_t* offsets_in, const int32_t* pt_table_gu,
                      const int32_t* pt_table_dn, int layer, int e_first, int e_count, int F, int H, int bn1,
                      int bn2, int splits, cudaStream_t s);
void launch_gather(const LayerWork& w, const float* x, int T, int kk, int H, cudaStream_t s);
void launch_gate_up(const CUtensorMap& map_w, const CUtensorMap& map_x, const LayerWork& w, int F, int H,
                    int bn, int grid, cudaStream_t s);
void launch_down(const CUtensorMap& map_w, const CUtensorMap& map_h, const LayerWork& w, int F, int H, int bn,
                 int splits, int cap_rows, int grid, cudaStream_t s);
void launch_combine(const LayerWork& w, float* y, int T, int kk, int H, int splits, int cap_rows, float inv_k,
                    cudaStream_t s);
void launch_reduce_rows(const LayerWork& w, float* out, int n_rows, int H, int splits, int cap_rows,
                        cudaStream_t s);
int gemm_smem_bytes(int which, int bn);
void set_gemm_attrs();

}  // namespace xpgb
