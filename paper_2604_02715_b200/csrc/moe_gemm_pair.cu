// Grouped expert GEMM for prefill-sized expert groups on CTA pairs (cta_group::2).
//
// The decode kernel (k_moe_gemm, moe_kernels.cu) is swap-AB: weights are the
// UMMA A operand and an expert's few token rows are B.  Once an expert holds
// hundreds of rows the contraction is compute-bound and the tile shape decides
// how many operand bytes each MMA flop costs.  Here two SMs of a TPC cooperate
// on one 256 x 256 output tile:
//
//   A (M = 256 token rows)   : each CTA stages its own 128 rows   (16 KB / 64-K step)
//   B (N = 256 weight rows)  : each CTA stages half, 128 rows     (16 KB / 64-K step)
//   D (fp32, TMEM)           : each CTA holds its 128 rows x 256 columns
//
// so a CTA moves 32 KB of operands per 2*128*256*64 flops -- 1.5x fewer than the
// 1-CTA gate/up tile and 2x fewer than the 1-CTA down tile.  gate/up pairs the
// two halves of B as [128 gate rows | the matching 128 up rows]: every TMEM lane
// then holds g and u of the same feature, and the SwiGLU epilogue is lane-local.
//
// Roles per CTA (192 threads): warp 0 = TMA producer (both CTAs, each loads its
// halves; transaction bytes land on the leader's "full" barrier), warp 1 = TMEM
// allocator (both) + MMA issuer (leader only; commits multicast to both CTAs),
// warps 2..5 = epilogue (both; they release an accumulator stage by arriving on
// the leader's "tempty" barrier at cluster scope).
//
// Units are (expert, 256-row token tile, weight tile); weight tiles are grouped
// 8 at a time so the pairs in flight share a few weight tiles and a few token
// tiles in L2.  The prologue repeats the page-table residency check of the
// decode kernel (paging.py:228-237).
#include <cuda_bf16.h>

#include "launch_count.h"
#include "moe_kernels.cuh"
#include "ptx_sm100.cuh"

namespace xpgb {

namespace {

constexpr int kPairRows = 128;                       // rows per CTA of A and of B
constexpr int kPairTile = kPairRows * kBK * 2;       // one 128-row x 64-K bf16 tile (16 KB)
constexpr int kPairAcc = 256;                        // TMEM columns per accumulator stage
constexpr int kWeightGroup = 8;                      // weight tiles per rasterization group
constexpr int kPairTab = (3 * kMaxExperts + 8) * 4;

// SPLIT: the token tile comes as its hi and lo bf16 planes (moe_kernels.cuh: split_bf16),
// two MMAs per K step; otherwise bf16 activations only.
template <bool SPLIT>
struct PairCfg {
  static constexpr int STAGE = (SPLIT ? 3 : 2) * kPairTile;  // A hi (+ A lo) + B half
  static constexpr int STAGES = SPLIT ? 4 : 6;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256 + kPairTab;
  static_assert(SMEM <= 227 * 1024, "pair GEMM stages exceed 227 KB");
};

// Offset arithmetic on the shared pointer itself: a round trip through uintptr_t loses the
// address space, and every table read through the result becomes a generic LD instead of LDS.
__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return p + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(p)) & 1023u)) & 1023u);
}

__device__ __forceinline__ float silu_pair(float g) { return g * (1.0f / (1.0f + __expf(-g))); }

struct PairUnit {
  int e, tt, wt;
};

__device__ __forceinline__ PairUnit pair_unit(int u, const int* s_up, const int* s_off, int E, int MT) {
  int lo = 0, hi = E;  // largest e with s_up[e] <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_up[mid] <= u) lo = mid; else hi = mid;
  }
  const int n = s_off[lo + 1] - s_off[lo];
  const int TT = (n + 2 * kPairRows - 1) / (2 * kPairRows);
  const int l = u - s_up[lo];
  const int blk = l / (kWeightGroup * TT);
  const int in = l - blk * kWeightGroup * TT;
  const int gsz = min(kWeightGroup, MT - blk * kWeightGroup);
  PairUnit r;
  r.e = lo;
  r.tt = in / gsz;
  r.wt = blk * kWeightGroup + in % gsz;
  return r;
}

}  // namespace

template <bool GU, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_moe_gemm_pair(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                    const __grid_constant__ CUtensorMap map_ws, GemmParams p) {
  using PC = PairCfg<SPLIT>;
  constexpr int kPairStages = PC::STAGES;
  constexpr int kPairStageBytes = PC::STAGE;
  constexpr int kBOff = (SPLIT ? 2 : 1) * kPairTile;  // B half after the token plane(s)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPairStages * kPairStageBytes);
  uint64_t* empty = full + kPairStages;
  uint64_t* tfull = empty + kPairStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_off = reinterpret_cast<int*>(smem + kPairStages * kPairStageBytes + 256);
  int* s_up = s_off + kMaxExperts + 1;
  int* s_slot = s_up + kMaxExperts + 1;
  int* s_flag = s_slot + kMaxExperts;

  const int E = p.E;
  const int MT = GU ? (p.F + kPairRows - 1) / kPairRows : (p.H + 2 * kPairRows - 1) / (2 * kPairRows);
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  // ---- prologue (identical in both CTAs: same global inputs, same decisions)
  if (threadIdx.x == 0) *s_flag = 0;
  for (int e = threadIdx.x; e <= E; e += blockDim.x) s_off[e] = p.offsets[e];
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    bool bad = false;
    if (lane == 0) s_up[0] = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      int u = 0;
      if (e < E) {
        const int n = s_off[e + 1] - s_off[e];
        if (n > 0) {
          u = ((n + 2 * kPairRows - 1) / (2 * kPairRows)) * MT;
          if (e < p.E_routed) {
            const int32_t ent = p.pt[e];
            if (pt_state(ent) != 2) {
              if (rank == 0)
                atomicCAS((unsigned long long*)p.fault, 0ull,
                          (unsigned long long)fault_pack(p.layer, p.e_first + e + 1, GU ? 1 : 2, pt_state(ent)));
              bad = true;
            }
            s_slot[e] = pt_block0(ent);
          } else {
            s_slot[e] = p.shared_block0 + (e - p.E_routed);
          }
        }
      }
      int x = u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (e < E) s_up[e + 1] = carry + x;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) *s_flag = 1;
  }
  __syncthreads();
  const int n_units = s_up[E];
  if (*s_flag || pair >= n_units) return;  // both CTAs of the pair take the same exit

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_x);
    tma_prefetch_desc(&map_w);
    if (E > p.E_routed) tma_prefetch_desc(&map_ws);
    for (int s = 0; s < kPairStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 128); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<2 * kPairAcc>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's barriers exist before any cross-CTA arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int K = GU ? p.H : p.F;
  const int KB = (K + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_last();  // weight tiles are re-read by every token tile
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < n_units; u += npairs) {
        const PairUnit un = pair_unit(u, s_up, s_off, E, MT);
        const int xrow = s_off[un.e] + un.tt * 2 * kPairRows + (int)rank * kPairRows;
        const int wrow = GU ? s_slot[un.e] * 2 * p.F + un.wt * kPairRows + (int)rank * p.F
                            : s_slot[un.e] * p.H + un.wt * 2 * kPairRows + (int)rank * kPairRows;
        const CUtensorMap* mw = un.e < p.E_routed ? &map_w : &map_ws;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kPairStageBytes;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * kPairStageBytes);
          tma_load_2d_pair(sa, &map_x, &full[stage], kb * kBK, xrow, pol_x);
          if (SPLIT) tma_load_2d_pair(sa + kPairTile, &map_x, &full[stage], kb * kBK, xrow + (int)p.act_lo_rows, pol_x);
          tma_load_2d_pair(sa + kBOff, mw, &full[stage], kb * kBK, wrow, pol_w);
          if (++stage == kPairStages) { stage = 0; phase ^= 1; }
        }
      }
      // drain: every multicast release of this CTA's stages has landed before exit
      for (int i = 0; i < kPairStages; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == kPairStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(2 * kPairRows, kPairAcc);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = pair; u < n_units; u += npairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_par = (it >> 1) & 1;
        mbar_wait_cluster(&tempty[acc], acc_par ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * kPairAcc;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_base = smem_u32(smem + stage * kPairStageBytes);
            const uint32_t b_base = a_base + kBOff;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t bdesc = sdesc_k_sw128(b_base + 32 * k);
              umma_bf16_pair(d0, sdesc_k_sw128(a_base + 32 * k), bdesc, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if (SPLIT) umma_bf16_pair(d0, sdesc_k_sw128(a_base + kPairTile + 32 * k), bdesc, idesc, 1u);
            }
            umma_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kPairStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int u = pair; u < n_units; u += npairs, ++it) {
      const PairUnit un = pair_unit(u, s_up, s_off, E, MT);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_par);
      tc_fence_after();
      const int n = s_off[un.e + 1] - s_off[un.e];
      const int r = (int)rank * kPairRows + q * 32 + (int)lane;  // row inside the 256-row token tile
      const bool valid = un.tt * 2 * kPairRows + r < n;
      const long long row = (long long)s_off[un.e] + un.tt * 2 * kPairRows + r;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * kPairAcc;
      if (GU) {
        const int f0 = un.wt * kPairRows;
        __nv_bfloat16* hrow = p.hbuf + row * p.F + f0;
        for (int c0 = 0; c0 < kPairRows; c0 += 16) {
          float g[16], v[16];
          tmem_ld16(tbase + c0, g);
          tmem_ld16(tbase + kPairRows + c0, v);
          if (valid && f0 + c0 + 16 <= p.F) {
            __nv_bfloat16 hi[16], lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) split_bf16(silu_pair(g[i]) * v[i], &hi[i], &lo[i]);
            uint4* dst = reinterpret_cast<uint4*>(hrow + c0);
            dst[0] = reinterpret_cast<const uint4*>(hi)[0];
            dst[1] = reinterpret_cast<const uint4*>(hi)[1];
            // the lo plane (read only by a split down projection; every row's h is stored
            // split, so paths can mix)
            uint4* dlo = reinterpret_cast<uint4*>(hrow + c0 + (size_t)p.h_lo_rows * p.F);
            dlo[0] = reinterpret_cast<const uint4*>(lo)[0];
            dlo[1] = reinterpret_cast<const uint4*>(lo)[1];
          }
        }
      } else {
        const int f0 = un.wt * 2 * kPairRows;
        float* orow = p.part + row * p.H + f0;  // split 0 (the pair kernel runs unsplit)
        for (int c0 = 0; c0 < kPairAcc; c0 += 16) {
          float v[16];
          tmem_ld16(tbase + c0, v);
          if (valid && f0 + c0 + 16 <= p.H) {
            float4* dst = reinterpret_cast<float4*>(orow + c0);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA may overwrite this stage
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<2 * kPairAcc>(tmem);
}

bool pair_gemm_supported(int H, int F) { return H % (2 * kPairRows) == 0 && F % kPairRows == 0; }

void set_pair_gemm_attrs() {
  cudaFuncSetAttribute(k_moe_gemm_pair<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<true>::SMEM);
  cudaFuncSetAttribute(k_moe_gemm_pair<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<true>::SMEM);
  cudaFuncSetAttribute(k_moe_gemm_pair<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       PairCfg<false>::SMEM);
  cudaFuncSetAttribute(k_moe_gemm_pair<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       PairCfg<false>::SMEM);
}

void launch_gemm_pair(bool gate_up, const CUtensorMap& map_x, const CUtensorMap& map_w, const CUtensorMap& map_ws,
                      const GemmParams& p, int num_sms, cudaStream_t s, bool split) {
  const int grid = (num_sms / 2) * 2;
  if (split) {
    if (gate_up)
      k_moe_gemm_pair<true, true><<<grid, 192, PairCfg<true>::SMEM, s>>>(map_x, map_w, map_ws, p);
    else
      k_moe_gemm_pair<false, true><<<grid, 192, PairCfg<true>::SMEM, s>>>(map_x, map_w, map_ws, p);
  } else {
    if (gate_up)
      k_moe_gemm_pair<true, false><<<grid, 192, PairCfg<false>::SMEM, s>>>(map_x, map_w, map_ws, p);
    else
      k_moe_gemm_pair<false, false><<<grid, 192, PairCfg<false>::SMEM, s>>>(map_x, map_w, map_ws, p);
  }
  note_launch();
}

}  // namespace xpgb
