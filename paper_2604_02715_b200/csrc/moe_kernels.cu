// MoE layer kernels for sm_100a:
//   k_route      hash router top-k (bit-exact with xpg pipeline.py:154-170)
//   k_plan       expert-major permutation, page-table read + fault check, GEMM work lists
//   k_gather     fp32 token rows -> bf16 expert-major rows
//   k_gate_up    grouped GEMM  X_e * Wgu_e^T with fused SwiGLU epilogue (tcgen05 + TMA + TMEM)
//   k_down       grouped GEMM  h_e * Wd_e^T, split-K partials (tcgen05 + TMA + TMEM)
//   k_combine    ordered per-token weighted sum (pipeline.py:198-207)
#include <cuda_bf16.h>
#include <cstdio>

#include "launch_count.h"
#include "moe_kernels.cuh"
#include "ptx_sm100.cuh"

namespace xpgb {

// ============================================================================ router

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One warp per (layer, token).  Lane l owns experts j = l+1, l+33, ...; each of
// the kk rounds takes the warp-wide minimum of (score, j) among untaken
// candidates (ties broken by the smaller j, as the reference's tuple sort), and
// the selected ids are finally written in ascending order.
__global__ void k_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k,
                        int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= (long long)layer_count * T) return;
  const int li = (int)(gw / T), t = (int)(gw % T);
  const int layer = layer_first + li;
  const int kk = min(top_k, L);
  const uint64_t base = seed * 0x9E37ull + (uint64_t)(uint32_t)layer * 0xC2B2ull + (uint64_t)(uint32_t)t * 0x85EBull;
  const int ncand = (L - lane + 31) / 32;  // candidates owned by this lane
  uint32_t taken = 0;
  int mine = 0x7fffffff;
  for (int r = 0; r < kk; ++r) {
    uint64_t bs = ~0ull;
    int bj = 0x7fffffff;
    for (int c = 0; c < ncand; ++c) {
      if (taken & (1u << c)) continue;
      const int j = lane + 1 + 32 * c;
      const uint64_t s = splitmix64(base + (uint64_t)j);
      if (s < bs || (s == bs && j < bj)) { bs = s; bj = j; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const uint64_t os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (os < bs || (os == bs && oj < bj)) { bs = os; bj = oj; }
    }
    if (((bj - 1) & 31) == lane) taken |= 1u << ((bj - 1) >> 5);
    if (lane == r) mine = bj;
  }
  int rank = 0;
  for (int i = 0; i < kk; ++i) {
    const int other = __shfl_sync(0xffffffffu, mine, i);
    rank += (other < mine);
  }
  if (lane < kk) out[((long long)li * T + t) * kk + rank] = mine;
}

void launch_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int32_t* out,
                  cudaStream_t s) {
  const long long warps = (long long)layer_count * T;
  if (warps == 0) return;
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  k_route<<<(unsigned)blocks, threads, 0, s>>>(seed, layer_first, layer_count, T, L, top_k, out);
  note_launch();
}

// ============================================================================ plan

// Block-wide exclusive scan of one int per thread (blockDim.x == 1024).
__device__ int block_exclusive_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = warp_tot[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, off);
      if (lane >= off) s += y;
    }
    warp_tot[lane] = s;  // inclusive
    if (lane == 31) *total = s;
  }
  __syncthreads();
  const int excl = x - v + (w > 0 ? warp_tot[w - 1] : 0);
  __syncthreads();
  return excl;
}

struct PlanShared {
  int cnt[kMaxExperts];
  int off[kMaxExperts];
  int cur[kMaxExperts];
  int warp_tot[32];
  int total;
  int fault;
};

// Resolve slots, emit GEMM units.  Shared by the routed and the pre-grouped (EP) plans.
__device__ void plan_tail(PlanShared& sh, const LayerWork& w, const int32_t* pt_gu, const int32_t* pt_dn,
                          int layer, int e_first, int e_count, int F, int H, int bn1, int bn2, int splits) {
  const int tid = threadIdx.x;
  const int e = tid;
  const int n = (e < e_count) ? sh.cnt[e] : 0;
  if (e < e_count) {
    w.offsets[e] = sh.off[e];
    if (e == e_count - 1) w.offsets[e_count] = sh.off[e] + n;
    int sg = -1, sd = -1;
    if (n > 0) {
      // read_page semantics (paging.py:228-237): only RESIDENT pages may be read.
      const int32_t eg = pt_gu[(long long)(layer - 1) * e_count + e];
      const int32_t ed = pt_dn[(long long)(layer - 1) * e_count + e];
      if (pt_state(eg) != 2) {
        atomicCAS((unsigned long long*)w.fault, 0ull,
                  (unsigned long long)fault_pack(layer, e_first + e + 1, 1, pt_state(eg)));
        sh.fault = 1;
      } else {
        sg = pt_block0(eg);
      }
      if (pt_state(ed) != 2) {
        atomicCAS((unsigned long long*)w.fault, 0ull,
                  (unsigned long long)fault_pack(layer, e_first + e + 1, 2, pt_state(ed)));
        sh.fault = 1;
      } else {
        sd = pt_block0(ed);
      }
    }
    w.slot_gu[e] = sg;
    w.slot_dn[e] = sd;
  }
  __syncthreads();
  const int mt1 = (F + kBM - 1) / kBM, mt2 = (H + kBM - 1) / kBM;
  const int nt1 = (n + bn1 - 1) / bn1, nt2 = (n + bn2 - 1) / bn2;
  const int u1 = sh.fault ? 0 : nt1 * mt1;
  const int u2 = sh.fault ? 0 : nt2 * mt2 * splits;
  const int b1 = block_exclusive_scan(u1, sh.warp_tot, &sh.total);
  const int tot1 = sh.total;
  __syncthreads();
  const int b2 = block_exclusive_scan(u2, sh.warp_tot, &sh.total);
  const int tot2 = sh.total;
  if (u1 > 0) {
    int idx = b1;
    for (int m = 0; m < mt1; ++m)
      for (int t = 0; t < nt1; ++t) {
        const int rows = min(bn1, n - t * bn1);
        w.units1[idx++] = GemmUnit{e, m * kBM, sh.off[e] + t * bn1, rows};
      }
  }
  if (u2 > 0) {
    int idx = b2;
    for (int m = 0; m < mt2; ++m)
      for (int s = 0; s < splits; ++s)
        for (int t = 0; t < nt2; ++t) {
          const int rows = min(bn2, n - t * bn2);
          w.units2[idx++] = GemmUnit{e, m * kBM, sh.off[e] + t * bn2, rows | (s << 16)};
        }
  }
  if (tid == 0) {
    w.counters[0] = tot1;
    w.counters[1] = tot2;
  }
}

__global__ void __launch_bounds__(1024, 1)
    k_plan(LayerWork w, const int32_t* __restrict__ pt_gu, const int32_t* __restrict__ pt_dn, int layer, int T,
           int kk, int e_first, int e_count, int F, int H, int bn1, int bn2, int splits) {
  __shared__ PlanShared sh;
  const int tid = threadIdx.x;
  const int pairs = T * kk;
  if (tid == 0) sh.fault = (*(volatile long long*)w.fault != 0);
  for (int e = tid; e < e_count; e += blockDim.x) sh.cnt[e] = 0;
  __syncthreads();
  if (sh.fault) {
    if (tid == 0) { w.counters[0] = 0; w.counters[1] = 0; w.counters[2] = 0; }
    return;
  }
  for (int p = tid; p < pairs; p += blockDim.x) {
    const int e = w.topk[p] - 1 - e_first;
    if (e >= 0 && e < e_count) atomicAdd(&sh.cnt[e], 1);
  }
  __syncthreads();
  const int v = (tid < e_count) ? sh.cnt[tid] : 0;
  const int ex = block_exclusive_scan(v, sh.warp_tot, &sh.total);
  if (tid < e_count) { sh.off[tid] = ex; sh.cur[tid] = ex; }
  if (tid == 0) w.counters[2] = sh.total;
  __syncthreads();
  // Row order inside an expert is irrelevant to the result: every output
  // column of the GEMM depends only on its own activation row.
  for (int p = tid; p < pairs; p += blockDim.x) {
    const int e = w.topk[p] - 1 - e_first;
    w.pos[p] = (e >= 0 && e < e_count) ? atomicAdd(&sh.cur[e], 1) : -1;
  }
  __syncthreads();
  plan_tail(sh, w, pt_gu, pt_dn, layer, e_first, e_count, F, H, bn1, bn2, splits);
}

__global__ void __launch_bounds__(1024, 1)
    k_plan_rows(LayerWork w, const int32_t* __restrict__ offsets_in, const int32_t* __restrict__ pt_gu,
                const int32_t* __restrict__ pt_dn, int layer, int e_first, int e_count, int F, int H, int bn1,
                int bn2, int splits) {
  __shared__ PlanShared sh;
  const int tid = threadIdx.x;
  if (tid == 0) sh.fault = (*(volatile long long*)w.fault != 0);
  if (tid < e_count) {
    sh.off[tid] = offsets_in[tid];
    sh.cnt[tid] = offsets_in[tid + 1] - offsets_in[tid];
  }
  __syncthreads();
  if (sh.fault) {
    if (tid == 0) { w.counters[0] = 0; w.counters[1] = 0; }
    return;
  }
  plan_tail(sh, w, pt_gu, pt_dn, layer, e_first, e_count, F, H, bn1, bn2, splits);
}

void launch_plan(const LayerWork& w, const int32_t* pt_gu, const int32_t* pt_dn, int layer, int T, int kk,
                 int e_first, int e_count, int F, int H, int bn1, int bn2, int splits, cudaStream_t s) {
  k_plan<<<1, 1024, 0, s>>>(w, pt_gu, pt_dn, layer, T, kk, e_first, e_count, F, H, bn1, bn2, splits);
  note_launch();
}
void launch_plan_rows(const LayerWork& w, const int32_t* offsets_in, const int32_t* pt_gu, const int32_t* pt_dn,
                      int layer, int e_first, int e_count, int F, int H, int bn1, int bn2, int splits,
                      cudaStream_t s) {
  k_plan_rows<<<1, 1024, 0, s>>>(w, offsets_in, pt_gu, pt_dn, layer, e_first, e_count, F, H, bn1, bn2, splits);
  note_launch();
}

// ============================================================================ gather / combine

// One block per token: convert the fp32 row to bf16 once, store it at each of
// its kk expert-major positions (8-byte vector stores).
__global__ void k_gather(const float* __restrict__ x, const int32_t* __restrict__ pos,
                         const long long* __restrict__ fault, __nv_bfloat16* __restrict__ xp, int kk, int H) {
  if (*fault) return;
  const int t = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)t * H);
  int p[kMaxTopK];
  for (int s = 0; s < kk; ++s) p[s] = pos[t * kk + s];
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
    const float4 v = xr[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&a);
    packed.y = *reinterpret_cast<uint32_t*>(&b);
    for (int s = 0; s < kk; ++s)
      if (p[s] >= 0) *reinterpret_cast<uint2*>(xp + (size_t)p[s] * H + 4 * i) = packed;
  }
}

void launch_gather(const LayerWork& w, const float* x, int T, int kk, int H, cudaStream_t s) {
  if (T == 0) return;
  const int threads = min(256, max(32, H / 4));
  k_gather<<<T, threads, 0, s>>>(x, w.pos, w.fault, w.xp, kk, H);
  note_launch();
}

// y_t = sum over routed experts in ascending order of (sum_split part) * inv_k,
// with explicit round-to-nearest adds/multiplies (no FMA contraction) so the
// accumulation mirrors `y += expert_output(...) * inv_k` (pipeline.py:206).
__global__ void k_combine(const float* __restrict__ part, const int32_t* __restrict__ pos,
                          const long long* __restrict__ fault, float* __restrict__ y, int kk, int H, int splits,
                          long long split_stride, float inv_k) {
  if (*fault) return;
  const int t = blockIdx.x;
  int p[kMaxTopK];
  for (int s = 0; s < kk; ++s) p[s] = pos[t * kk + s];
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < kk; ++s) {
      if (p[s] < 0) continue;
      const float4* src = reinterpret_cast<const float4*>(part + (size_t)p[s] * H) + i;
      float4 v = src[0];
      for (int k = 1; k < splits; ++k) {
        const float4 q = src[k * split_stride / 4];
        v.x = __fadd_rn(v.x, q.x); v.y = __fadd_rn(v.y, q.y); v.z = __fadd_rn(v.z, q.z); v.w = __fadd_rn(v.w, q.w);
      }
      acc.x = __fadd_rn(acc.x, __fmul_rn(v.x, inv_k));
      acc.y = __fadd_rn(acc.y, __fmul_rn(v.y, inv_k));
      acc.z = __fadd_rn(acc.z, __fmul_rn(v.z, inv_k));
      acc.w = __fadd_rn(acc.w, __fmul_rn(v.w, inv_k));
    }
    reinterpret_cast<float4*>(y + (size_t)t * H)[i] = acc;
  }
}

void launch_combine(const LayerWork& w, float* y, int T, int kk, int H, int splits, int cap_rows, float inv_k,
                    cudaStream_t s) {
  if (T == 0) return;
  const int threads = min(256, max(32, H / 4));
  k_combine<<<T, threads, 0, s>>>(w.part, w.pos, w.fault, y, kk, H, splits, (long long)cap_rows * H, inv_k);
  note_launch();
}

// Sum split-K partials of pre-grouped rows (EP path): out[r] = sum_split part[split][r].
__global__ void k_reduce_rows(const float* __restrict__ part, const long long* __restrict__ fault,
                              float* __restrict__ out, long long n4, int splits, long long split_stride4) {
  if (*fault) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4* src = reinterpret_cast<const float4*>(part) + i;
    float4 v = src[0];
    for (int k = 1; k < splits; ++k) {
      const float4 q = src[k * split_stride4];
      v.x = __fadd_rn(v.x, q.x); v.y = __fadd_rn(v.y, q.y); v.z = __fadd_rn(v.z, q.z); v.w = __fadd_rn(v.w, q.w);
    }
    reinterpret_cast<float4*>(out)[i] = v;
  }
}

void launch_reduce_rows(const LayerWork& w, float* out, int n_rows, int H, int splits, int cap_rows,
                        cudaStream_t s) {
  const long long n4 = (long long)n_rows * H / 4;
  if (n4 == 0) return;
  const long long nb = (n4 + 255) / 256;
  const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
  k_reduce_rows<<<blocks, 256, 0, s>>>(w.part, w.fault, out, n4, splits, (long long)cap_rows * H / 4);
  note_launch();
}

// ============================================================================ tcgen05 grouped GEMMs
//
// Warp roles (192 threads, one CTA per SM, persistent over the unit list):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (lane 0 issues tcgen05.mma)
//   warps 2..5  epilogue: TMEM -> registers -> global (warp w reads lanes 32*(w%4)..)
// Swap-AB: the weight tile (128 rows x 64 K) is the UMMA A operand, the
// expert's activation rows (n <= BN) are B, so decode-size n costs N=16..BN
// columns instead of padding M.  Weights are addressed through the page
// table: row = block * rows_per_block + m0 inside one tensor map over the pool.

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ float silu_f(float g) { return g * (1.0f / (1.0f + __expf(-g))); }

template <int BN, int STAGES>
struct GateUpCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE = 2 * A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_gate_up(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, LayerWork w,
              int F, int H) {
  using C = GateUpCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  if (*w.fault != 0) return;
  const int n_units = w.counters[0];
  if ((int)blockIdx.x >= n_units) return;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (H + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const GemmUnit un = w.units1[u];
        const int n_rows = un.n_and_split & 0xFFFF;
        const int nb = (n_rows + kBoxRowsB - 1) / kBoxRowsB;
        const int gate_row = w.slot_gu[un.expert] * 2 * F + un.m0;
        const uint32_t bytes = 2 * C::A_BYTES + nb * kBoxRowsB * kBK * 2;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d(sa, &map_w, &full[stage], kb * kBK, gate_row, pol_w);
          tma_load_2d(sa + C::A_BYTES, &map_w, &full[stage], kb * kBK, gate_row + F, pol_w);
          for (int i = 0; i < nb; ++i)
            tma_load_2d(sa + 2 * C::A_BYTES + i * kBoxRowsB * kBK * 2, &map_x, &full[stage], kb * kBK,
                        un.row_begin + i * kBoxRowsB, pol_x);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const GemmUnit un = w.units1[u];
      const int n_rows = un.n_and_split & 0xFFFF;
      const uint32_t idesc = idesc_bf16_f32(kBM, (n_rows + 15) & ~15);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_par ^ 1);
      tc_fence_after();
      const uint32_t d_gate = tmem + acc * 256;
      const uint32_t d_up = d_gate + 128;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + stage * C::STAGE);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t bdesc = sdesc_k_sw128(base + 2 * C::A_BYTES + 32 * k);
            const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
            umma_bf16(d_gate, sdesc_k_sw128(base + 32 * k), bdesc, idesc, accum);
            umma_bf16(d_up, sdesc_k_sw128(base + C::A_BYTES + 32 * k), bdesc, idesc, accum);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const GemmUnit un = w.units1[u];
      const int n_rows = un.n_and_split & 0xFFFF;
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_par);
      tc_fence_after();
      const int r = un.m0 + q * 32 + lane;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * 256;
      __nv_bfloat16* hcol = w.hbuf + (size_t)un.row_begin * F + r;
      for (int c0 = 0; c0 < n_rows; c0 += 16) {
        float g[16], v[16];
        tmem_ld16(tbase + c0, g);
        tmem_ld16(tbase + 128 + c0, v);
        if (r < F) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < n_rows) hcol[(size_t)(c0 + i) * F] = __float2bfloat16_rn(silu_f(g[i]) * v[i]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int BN, int STAGES>
struct DownCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_down(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_h, LayerWork w,
           int F, int H, int splits, long long split_stride) {
  using C = DownCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  if (*w.fault != 0) return;
  const int n_units = w.counters[1];
  if ((int)blockIdx.x >= n_units) return;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_h);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (F + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const GemmUnit un = w.units2[u];
        const int n_rows = un.n_and_split & 0xFFFF;
        const int split = un.n_and_split >> 16;
        const int kb0 = split * KB / splits, kb1 = (split + 1) * KB / splits;
        const int nb = (n_rows + kBoxRowsB - 1) / kBoxRowsB;
        const int wrow = w.slot_dn[un.expert] * H + un.m0;
        const uint32_t bytes = C::A_BYTES + nb * kBoxRowsB * kBK * 2;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d(sa, &map_w, &full[stage], kb * kBK, wrow, pol_w);
          for (int i = 0; i < nb; ++i)
            tma_load_2d(sa + C::A_BYTES + i * kBoxRowsB * kBK * 2, &map_h, &full[stage], kb * kBK,
                        un.row_begin + i * kBoxRowsB, pol_x);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const GemmUnit un = w.units2[u];
      const int n_rows = un.n_and_split & 0xFFFF;
      const int split = un.n_and_split >> 16;
      const int kb0 = split * KB / splits, kb1 = (split + 1) * KB / splits;
      const uint32_t idesc = idesc_bf16_f32(kBM, (n_rows + 15) & ~15);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_par ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * 128;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + stage * C::STAGE);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(d, sdesc_k_sw128(base + 32 * k), sdesc_k_sw128(base + C::A_BYTES + 32 * k), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const GemmUnit un = w.units2[u];
      const int n_rows = un.n_and_split & 0xFFFF;
      const int split = un.n_and_split >> 16;
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_par);
      tc_fence_after();
      const int r = un.m0 + q * 32 + lane;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * 128;
      float* out = w.part + split * split_stride + (size_t)un.row_begin * H + r;
      for (int c0 = 0; c0 < n_rows; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
        if (r < H) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < n_rows) out[(size_t)(c0 + i) * H] = v[i];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

// ---- instantiations / launchers

#define XPGB_GU_CFG(BN, ST) \
  case BN:                  \
    kern = k_gate_up<BN, ST>; smem = GateUpCfg<BN, ST>::SMEM; break;
#define XPGB_DN_CFG(BN, ST) \
  case BN:                  \
    kern = k_down<BN, ST>; smem = DownCfg<BN, ST>::SMEM; break;

int gemm_smem_bytes(int which, int bn) {
  if (which == 0) {
    switch (bn) {
      case 32: return GateUpCfg<32, 6>::SMEM;
      case 64: return GateUpCfg<64, 5>::SMEM;
      default: return GateUpCfg<128, 4>::SMEM;
    }
  }
  switch (bn) {
    case 32: return DownCfg<32, 10>::SMEM;
    case 64: return DownCfg<64, 8>::SMEM;
    default: return DownCfg<128, 6>::SMEM;
  }
}

void set_gemm_attrs() {
  cudaFuncSetAttribute(k_gate_up<32, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, GateUpCfg<32, 6>::SMEM);
  cudaFuncSetAttribute(k_gate_up<64, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, GateUpCfg<64, 5>::SMEM);
  cudaFuncSetAttribute(k_gate_up<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, GateUpCfg<128, 4>::SMEM);
  cudaFuncSetAttribute(k_down<32, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, DownCfg<32, 10>::SMEM);
  cudaFuncSetAttribute(k_down<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, DownCfg<64, 8>::SMEM);
  cudaFuncSetAttribute(k_down<128, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, DownCfg<128, 6>::SMEM);
}

void launch_gate_up(const CUtensorMap& map_w, const CUtensorMap& map_x, const LayerWork& w, int F, int H, int bn,
                    int grid, cudaStream_t s) {
  void (*kern)(const CUtensorMap, const CUtensorMap, LayerWork, int, int) = nullptr;
  int smem = 0;
  switch (bn) {
    XPGB_GU_CFG(32, 6)
    XPGB_GU_CFG(64, 5)
    default:
      kern = k_gate_up<128, 4>; smem = GateUpCfg<128, 4>::SMEM; break;
  }
  kern<<<grid, 192, smem, s>>>(map_w, map_x, w, F, H);
  note_launch();
}

void launch_down(const CUtensorMap& map_w, const CUtensorMap& map_h, const LayerWork& w, int F, int H, int bn,
                 int splits, int cap_rows, int grid, cudaStream_t s) {
  void (*kern)(const CUtensorMap, const CUtensorMap, LayerWork, int, int, int, long long) = nullptr;
  int smem = 0;
  switch (bn) {
    XPGB_DN_CFG(32, 10)
    XPGB_DN_CFG(64, 8)
    default:
      kern = k_down<128, 6>; smem = DownCfg<128, 6>::SMEM; break;
  }
  kern<<<grid, 192, smem, s>>>(map_w, map_h, w, F, H, splits, (long long)cap_rows * H);
  note_launch();
}

}  // namespace xpgb
