// MoE layer kernels for sm_100a:
//   k_route        hash router top-k (bit-exact with xpg pipeline.py:154-170)
//   k_route_plan   router + per-expert counts + expert-major positions, one CTA per layer
//   k_gather       fp32 token rows -> bf16 expert-major rows (first layer of a run)
//   k_moe_gemm     grouped GEMM, tcgen05 + TMA + TMEM, persistent; two instantiations:
//                    gate/up:  X_e * Wgu_e^T with the SwiGLU epilogue -> bf16 h rows
//                    down:     h_e * Wd_e^T, split-K partials          -> fp32 rows
//   k_combine      ordered per-token weighted sum (pipeline.py:198-207) + next-layer gather
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

// Warp-cooperative top-k of one (layer, token).  Lane l owns experts
// j = l+1, l+33, ... (NC slots, the scores hashed once into registers); each of
// the kk rounds takes the warp-wide minimum of (score, j) over untaken
// candidates (ties -> smaller j, the reference's tuple order).  Returns, in
// lanes 0..kk-1, the selected id and its ascending rank.
template <int NC>
__device__ __forceinline__ void route_token(uint64_t seed, int layer, int t, int L, int kk, int lane, int* id,
                                            int* rank) {
  const uint64_t base =
      seed * 0x9E37ull + (uint64_t)(uint32_t)layer * 0xC2B2ull + (uint64_t)(uint32_t)t * 0x85EBull;
  uint64_t sc[NC];
  uint32_t live = 0;  // candidate slots still in play
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = lane + 1 + 32 * c;
    sc[c] = splitmix64(base + (uint64_t)j);
    if (j <= L) live |= 1u << c;
  }
  int mine = 0x7fffffff;
  for (int r = 0; r < kk; ++r) {
    uint64_t bs = ~0ull;
    int bj = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = lane + 1 + 32 * c;
      if ((live >> c) & 1u)
        if (sc[c] < bs || (sc[c] == bs && j < bj)) { bs = sc[c]; bj = j; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const uint64_t os = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (os < bs || (os == bs && oj < bj)) { bs = os; bj = oj; }
    }
    if (((bj - 1) & 31) == lane) live &= ~(1u << ((bj - 1) >> 5));
    if (lane == r) mine = bj;
  }
  int rk = 0;
  for (int i = 0; i < kk; ++i) rk += (__shfl_sync(0xffffffffu, mine, i) < mine);
  *id = mine;
  *rank = rk;
}

// Candidate slots per lane for L experts, rounded to an instantiated width.
static inline int route_nc(int L) {
  const int n = (L + 31) / 32;
  return n <= 1 ? 1 : n <= 2 ? 2 : n <= 4 ? 4 : n <= 8 ? 8 : n <= 16 ? 16 : 32;
}

#define XPGB_ROUTE_DISPATCH(NCV, KERNEL, GRID, BLOCK, STREAM, ...)                 \
  switch (NCV) {                                                                   \
    case 1: KERNEL<1><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
    case 2: KERNEL<2><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
    case 4: KERNEL<4><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
    case 8: KERNEL<8><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;              \
    case 16: KERNEL<16><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;            \
    default: KERNEL<32><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__); break;            \
  }

template <int NC>
__global__ void k_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k,
                        int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (gw >= (long long)layer_count * T) return;
  const int li = (int)(gw / T), t = (int)(gw % T);
  const int kk = min(top_k, L);
  int id, rank;
  route_token<NC>(seed, layer_first + li, t, L, kk, lane, &id, &rank);
  if (lane < kk) out[((long long)li * T + t) * kk + rank] = id;
}

void launch_route(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int32_t* out,
                  cudaStream_t s) {
  const long long warps = (long long)layer_count * T;
  if (warps == 0) return;
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  XPGB_ROUTE_DISPATCH(route_nc(L), k_route, (unsigned)blocks, threads, s, seed, layer_first, layer_count, T, L,
                      top_k, out);
  note_launch();
}

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
    warp_tot[lane] = s;
    if (lane == 31) *total = s;
  }
  __syncthreads();
  const int excl = x - v + (w > 0 ? warp_tot[w - 1] : 0);
  __syncthreads();
  return excl;
}

// Local GEMM group of a plan id: routed ids 1..L map onto this shard's experts
// [0, E) (or -1 off-shard); shared ids L+1..L+S onto groups E..E+S-1.
__device__ __forceinline__ int local_group(int id, int L, int e_first, int E) {
  if (id < 1) return -1;
  if (id > L) return E + (id - L - 1);
  const int el = id - 1 - e_first;
  return (el >= 0 && el < E) ? el : -1;
}

// One CTA (1024 threads) per layer: route every token, count rows per local
// expert, exclusive-scan the counts into row offsets, place each (token, slot)
// pair.  Row order inside an expert is irrelevant to the result: every GEMM
// output column depends only on its own activation row.
template <int NC>
__global__ void __launch_bounds__(1024, 1)
    k_route_plan(uint64_t seed, int layer_first, int T, int L, int top_k, int e_first, int E, int S, int sh0,
                 int sh1, int32_t* __restrict__ topk, int32_t* __restrict__ pos, int32_t* __restrict__ offsets,
                 const long long* __restrict__ fault) {
  __shared__ int cnt[kMaxExperts];
  __shared__ int warp_tot[32];
  __shared__ int total;
  if (fault && *fault) return;
  const int li = blockIdx.x, layer = layer_first + li;
  const int kk = min(top_k, L), kt = kk + S, G = E + S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int32_t* tk = topk + (long long)li * T * kt;
  int32_t* ps = pos + (long long)li * T * kt;
  int32_t* of = offsets + (long long)li * (G + 1);
  for (int e = threadIdx.x; e < G; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  for (int t = warp; t < T; t += nwarps) {
    int id, rank;
    route_token<NC>(seed, layer, t, L, kk, lane, &id, &rank);
    if (lane < kk) {
      tk[(long long)t * kt + rank] = id;
      const int el = local_group(id, L, e_first, E);
      if (el >= 0) atomicAdd(&cnt[el], 1);
    } else if (lane < kt) {
      // shared expert: every token of [sh0, sh1) after its routed slots (0 = not here)
      tk[(long long)t * kt + lane] = (t >= sh0 && t < sh1) ? L + 1 + (lane - kk) : 0;
    }
  }
  for (int e = threadIdx.x; e < S; e += blockDim.x) cnt[E + e] = max(0, min(T, sh1) - sh0);
  __syncthreads();
  int carry = 0;
  for (int e0 = 0; e0 < G; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const int v = e < G ? cnt[e] : 0;
    const int ex = block_exclusive_scan(v, warp_tot, &total);
    if (e < G) {
      of[e] = carry + ex;
      cnt[e] = carry + ex;  // becomes the placement cursor
    }
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) of[G] = carry;
  __syncthreads();
  for (int p = threadIdx.x; p < T * kt; p += blockDim.x) {
    const int el = local_group(tk[p], L, e_first, E);
    ps[p] = el >= 0 ? atomicAdd(&cnt[el], 1) : -1;
  }
}

// ---- multi-CTA plan (large T): route+count, then scan+place, for every layer at once.
// cnt / cur: [layers][E] zeroed scratch.  Row order inside an expert comes from
// atomics, which the result does not depend on (see k_route_plan).
constexpr int kPlanTokensPerCta = 16;    // k_route_count: 8 warps x 2 tokens (spread over the SMs)
constexpr int kPlanPairsPerCta = 4096;   // k_plan_place: (token, slot) pairs per CTA

template <int NC>
__global__ void __launch_bounds__(256)
    k_route_count(uint64_t seed, int layer_first, int T, int L, int top_k, int e_first, int E, int S, int sh0,
                  int sh1, int32_t* __restrict__ topk, int32_t* __restrict__ cnt, const long long* __restrict__ fault) {
  __shared__ int lc[kMaxExperts];
  if (fault && *fault) return;
  const int li = blockIdx.y, layer = layer_first + li;
  const int kk = min(top_k, L), kt = kk + S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < E; e += blockDim.x) lc[e] = 0;
  __syncthreads();
  int32_t* tk = topk + (long long)li * T * kt;
  const int t0 = blockIdx.x * kPlanTokensPerCta, t1 = min(T, t0 + kPlanTokensPerCta);
  for (int t = t0 + warp; t < t1; t += nwarps) {
    int id, rank;
    route_token<NC>(seed, layer, t, L, kk, lane, &id, &rank);
    if (lane < kk) {
      tk[(long long)t * kt + rank] = id;
      const int el = local_group(id, L, e_first, E);
      if (el >= 0) atomicAdd(&lc[el], 1);
    } else if (lane < kt) {
      tk[(long long)t * kt + lane] = (t >= sh0 && t < sh1) ? L + 1 + (lane - kk) : 0;
    }
  }
  __syncthreads();
  int* gc = cnt + (long long)li * (E + S);
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (lc[e]) atomicAdd(&gc[e], lc[e]);
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < S; e += blockDim.x) atomicAdd(&gc[E + e], max(0, min(T, sh1) - sh0));
}

__global__ void __launch_bounds__(1024, 1)
    k_plan_place(int T, int kt, int L, int e_first, int Er, int E, const int32_t* __restrict__ topk, int32_t* __restrict__ pos,
                 int32_t* __restrict__ offsets, const int32_t* __restrict__ cnt, int32_t* __restrict__ cur,
                 const long long* __restrict__ fault) {
  __shared__ int off[kMaxExperts];
  __shared__ int lc[kMaxExperts];
  __shared__ int warp_tot[32];
  __shared__ int total;
  if (fault && *fault) return;
  const int li = blockIdx.y;
  const int32_t* gc = cnt + (long long)li * E;
  int carry = 0;
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const int v = e < E ? gc[e] : 0;
    const int ex = block_exclusive_scan(v, warp_tot, &total);
    if (e < E) {
      off[e] = carry + ex;
      lc[e] = 0;
    }
    carry += total;
    __syncthreads();
  }
  int32_t* of = offsets + (long long)li * (E + 1);
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) of[e] = off[e];
    if (threadIdx.x == 0) of[E] = carry;
  }
  __syncthreads();
  const int32_t* tk = topk + (long long)li * T * kt;
  int32_t* ps = pos + (long long)li * T * kt;
  const int p0 = blockIdx.x * kPlanPairsPerCta, p1 = min(T * kt, p0 + kPlanPairsPerCta);
  constexpr int PER = kPlanPairsPerCta / 1024;
  int el[PER], rk[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int p = p0 + i * 1024 + threadIdx.x;
    el[i] = -1;
    if (p < p1) {
      const int x = local_group(tk[p], L, e_first, Er);
      if (x >= 0) {
        el[i] = x;
        rk[i] = atomicAdd(&lc[x], 1);
      }
    }
  }
  __syncthreads();
  int32_t* gcur = cur + (long long)li * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (lc[e]) lc[e] = off[e] + atomicAdd(&gcur[e], lc[e]);  // this CTA's base row of expert e
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int p = p0 + i * 1024 + threadIdx.x;
    if (p < p1) ps[p] = el[i] >= 0 ? lc[el[i]] + rk[i] : -1;
  }
}

void launch_route_plan(uint64_t seed, int layer_first, int layer_count, int T, int L, int top_k, int e_first, int E,
                       int S, int sh0, int sh1, int32_t* topk, int32_t* pos, int32_t* offsets, int32_t* scratch,
                       const long long* fault, cudaStream_t s) {
  if (layer_count <= 0) return;
  sh0 = max(0, sh0);
  const int kk = min(top_k, L), kt = kk + S, G = E + S;
  const int nc = route_nc(L);
  if ((long long)T * kt <= kPlanSingleCtaPairs || scratch == nullptr) {
    XPGB_ROUTE_DISPATCH(nc, k_route_plan, layer_count, 1024, s, seed, layer_first, T, L, top_k, e_first, E, S, sh0, sh1, topk,
                        pos, offsets, fault);
    note_launch();
    return;
  }
  int32_t* cnt = scratch;
  int32_t* cur = scratch + (size_t)layer_count * G;
  cudaMemsetAsync(scratch, 0, (size_t)2 * layer_count * G * sizeof(int32_t), s);
  const dim3 g1((T + kPlanTokensPerCta - 1) / kPlanTokensPerCta, layer_count);
  XPGB_ROUTE_DISPATCH(nc, k_route_count, g1, 256, s, seed, layer_first, T, L, top_k, e_first, E, S, sh0, sh1, topk, cnt,
                      fault);
  note_launch();
  const dim3 g2((T * kt + kPlanPairsPerCta - 1) / kPlanPairsPerCta, layer_count);
  k_plan_place<<<g2, 1024, 0, s>>>(T, kt, L, e_first, E, G, topk, pos, offsets, cnt, cur, fault);
  note_launch();
}

// ============================================================================ gather / combine

// fp32 x4 -> the hi and lo bf16 planes (moe_kernels.cuh: split_bf16), 8 bytes each.
__device__ __forceinline__ void pack_split4(float4 v, uint2* hi, uint2* lo) {
  __nv_bfloat16 h[4], l[4];
  split_bf16(v.x, &h[0], &l[0]);
  split_bf16(v.y, &h[1], &l[1]);
  split_bf16(v.z, &h[2], &l[2]);
  split_bf16(v.w, &h[3], &l[3]);
  *hi = *reinterpret_cast<const uint2*>(h);
  *lo = *reinterpret_cast<const uint2*>(l);
}

// One block per token: split the fp32 row into its bf16 planes once, store both at each of
// its kk expert-major positions (8-byte vector stores).
__global__ void k_gather(const float* __restrict__ x, const int32_t* __restrict__ pos,
                         const long long* __restrict__ fault, __nv_bfloat16* __restrict__ xp, long long lo_rows,
                         int kk, int H) {
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (*fault) return;
  const int t = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)t * H);
  int p[kMaxTopK];
  for (int s = 0; s < kk; ++s) p[s] = pos[t * kk + s];
  const size_t lo_off = (size_t)lo_rows * H;
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
    uint2 hi, lo;
    pack_split4(xr[i], &hi, &lo);
    for (int s = 0; s < kk; ++s)
      if (p[s] >= 0) {
        __nv_bfloat16* d = xp + (size_t)p[s] * H + 4 * i;
        *reinterpret_cast<uint2*>(d) = hi;
        *reinterpret_cast<uint2*>(d + lo_off) = lo;
      }
  }
}

void launch_gather(const float* x, const int32_t* pos, const long long* fault, __nv_bfloat16* xp, long long lo_rows,
                   int T, int kk, int H, cudaStream_t s) {
  if (T == 0) return;
  const int threads = min(256, max(32, H / 4));
  k_gather<<<T, threads, 0, s>>>(x, pos, fault, xp, lo_rows, kk, H);
  note_launch();
}

// Plan of the shared-expert pass (xpgb_shared_forward): row s*T + t holds token t for
// shared expert s, offsets [0, T, 2T, ..., S*T].
__global__ void k_shared_plan(int32_t* __restrict__ pos, int32_t* __restrict__ off, int T, int S) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T * S; i += gridDim.x * blockDim.x)
    pos[i] = (i % S) * T + i / S;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= S; e += blockDim.x) off[e] = e * T;
}

void launch_shared_plan(int32_t* pos, int32_t* off, int T, int S, cudaStream_t s) {
  const int n = T * S;
  const int g = (n + 255) / 256;
  k_shared_plan<<<g < 1 ? 1 : (g > 148 ? 148 : g), 256, 0, s>>>(pos, off, T, S);
  note_launch();
}

// y_t = sum over routed experts in ascending order of (sum_split part) * inv_k,
// with explicit round-to-nearest adds/multiplies (no FMA contraction) so the
// accumulation mirrors `y += expert_output(...) * inv_k` (pipeline.py:206).
// With next_pos, bf16(y_t) also lands in the next layer's expert-major rows.
__global__ void k_combine(const float* __restrict__ part, const int32_t* __restrict__ pos,
                          const long long* __restrict__ fault, float* __restrict__ y, int kk, int kr, int H,
                          int splits, long long split_stride, float inv_k, const int32_t* __restrict__ next_pos,
                          __nv_bfloat16* __restrict__ xp, long long lo_rows, int accumulate) {
  if (threadIdx.x == 0) griddep_launch_dependents();  // the next layer's GEMM may stage its prologue
  if (*fault) return;
  const int t = blockIdx.x;
  int p[kMaxTopK], q[kMaxTopK];
  for (int s = 0; s < kk; ++s) {
    p[s] = pos[t * kk + s];
    q[s] = next_pos ? next_pos[t * kk + s] : -1;
  }
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
    float4 acc = accumulate ? reinterpret_cast<const float4*>(y + (size_t)t * H)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < kk; ++s) {
      if (p[s] < 0) continue;
      const float4* src = reinterpret_cast<const float4*>(part + (size_t)p[s] * H) + i;
      float4 v = src[0];
      for (int k = 1; k < splits; ++k) {
        const float4 w = src[k * split_stride / 4];
        v.x = __fadd_rn(v.x, w.x); v.y = __fadd_rn(v.y, w.y); v.z = __fadd_rn(v.z, w.z); v.w = __fadd_rn(v.w, w.w);
      }
      const float sc = s < kr ? inv_k : 1.0f;  // routed slots x 1/top_k, shared experts x 1
      acc.x = __fadd_rn(acc.x, __fmul_rn(v.x, sc));
      acc.y = __fadd_rn(acc.y, __fmul_rn(v.y, sc));
      acc.z = __fadd_rn(acc.z, __fmul_rn(v.z, sc));
      acc.w = __fadd_rn(acc.w, __fmul_rn(v.w, sc));
    }
    reinterpret_cast<float4*>(y + (size_t)t * H)[i] = acc;
    if (next_pos) {
      uint2 hi, lo;
      pack_split4(acc, &hi, &lo);
      for (int s = 0; s < kk; ++s)
        if (q[s] >= 0) {
          __nv_bfloat16* d = xp + (size_t)q[s] * H + 4 * i;
          *reinterpret_cast<uint2*>(d) = hi;
          *reinterpret_cast<uint2*>(d + (size_t)lo_rows * H) = lo;
        }
    }
  }
}

void launch_combine(const float* part, const int32_t* pos, const long long* fault, float* y, int T, int kk, int kr,
                    int H, int splits, long long split_stride, float inv_k, const int32_t* next_pos,
                    __nv_bfloat16* xp, long long lo_rows, cudaStream_t s, bool accumulate) {
  if (T == 0) return;
  const int threads = min(256, max(32, H / 4));
  k_combine<<<T, threads, 0, s>>>(part, pos, fault, y, kk, kr, H, splits, split_stride, inv_k, next_pos, xp,
                                  lo_rows, accumulate ? 1 : 0);
  note_launch();
}

// Sum split-K partials of pre-grouped rows (EP path): out[r] = sum_split part[split][r].
__global__ void k_reduce_rows(const float* __restrict__ part, const long long* __restrict__ fault,
                              float* __restrict__ out, long long n4, int splits, long long split_stride4) {
  if (*fault) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4* src = reinterpret_cast<const float4*>(part) + i;
    float4 v = src[0];
    for (int k = 1; k < splits; ++k) {
      const float4 w = src[k * split_stride4];
      v.x = __fadd_rn(v.x, w.x); v.y = __fadd_rn(v.y, w.y); v.z = __fadd_rn(v.z, w.z); v.w = __fadd_rn(v.w, w.w);
    }
    reinterpret_cast<float4*>(out)[i] = v;
  }
}

void launch_reduce_rows(const float* part, const long long* fault, float* out, int n_rows, int H, int splits,
                        long long split_stride, cudaStream_t s) {
  const long long n4 = (long long)n_rows * H / 4;
  if (n4 == 0) return;
  const long long nb = (n4 + 255) / 256;
  const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
  k_reduce_rows<<<blocks, 256, 0, s>>>(part, fault, out, n4, splits, split_stride / 4);
  note_launch();
}

// ============================================================================ tcgen05 grouped GEMM
//
// Warp roles (192 threads, one CTA per SM, persistent over the work units):
//   warp 0      TMA producer (lane 0)
//   warp 1      TMEM allocator + MMA issuer (lane 0 issues tcgen05.mma)
//   warps 2..5  epilogue: TMEM -> registers -> global (warp w reads lanes 32*(w%4)..)
// Swap-AB: the weight tile (128 rows x 64 K) is the UMMA A operand and the
// expert's activation rows (n <= BN) are B, so a decode-size expert costs an
// N = 16..BN MMA instead of a padded M.  Weights are addressed through the page
// table: row = block * rows_per_block + m0 inside one tensor map over the pool.
// The work-unit list is derived in every CTA's prologue from the expert row
// offsets (no global unit array), and the same prologue performs read_page's
// residency check (paging.py:228-237) on every routed expert's page.

// Offset arithmetic on the shared pointer itself: a round trip through uintptr_t loses the
// address space, and every table read through the result becomes a generic LD instead of LDS.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(p)) & 1023u)) & 1023u);
}

__device__ __forceinline__ float silu_f(float g) { return g * (1.0f / (1.0f + __expf(-g))); }

template <bool GU, int BN, int STAGES>
struct GemmCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  // A tiles per stage: gate + up, or (down, BN <= 128) two consecutive 128-row tiles of W_down
  // so each activation tile staged feeds 256 weight rows (halves the L2->SM activation bytes)
  static constexpr int NA = (GU || BN <= 128) ? 2 : 1;
  static constexpr int UNIT_ROWS = GU ? kBM : NA * kBM;  // weight rows per unit (per projection)
  static constexpr int B_BYTES = BN * kBK * 2;  // one activation plane
  static constexpr int STAGE = NA * A_BYTES + 2 * B_BYTES;  // weights + the hi and lo activation planes
  // TMEM columns per accumulator stage: gate+up = 2 x 128; down = BN (128 or 256 for prefill)
  static constexpr int ACC_COLS = (GU || BN <= 128) ? 256 : BN;
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
  static constexpr int TAB_BYTES = (3 * kMaxExperts + 8) * 4;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256 + TAB_BYTES;
  static_assert(SMEM <= 227 * 1024, "GEMM stages exceed the 227 KB of shared memory per CTA");
};

struct Unit {
  int e, m0, row_begin, n_rows, split;
};

__device__ __forceinline__ Unit decode_unit(int u, const int* s_up, const int* s_off, int E, int bn, int splits,
                                            bool gate_up, int unit_rows) {
  int lo = 0, hi = E;  // largest e with s_up[e] <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_up[mid] <= u) lo = mid; else hi = mid;
  }
  Unit r;
  r.e = lo;
  const int local = u - s_up[lo];
  const int n = s_off[lo + 1] - s_off[lo];
  const int nt_count = (n + bn - 1) / bn;
  int m, nt;
  if (gate_up) {
    m = local / nt_count;
    nt = local % nt_count;
    r.split = 0;
  } else {
    m = local / (splits * nt_count);
    const int rem = local % (splits * nt_count);
    r.split = rem / nt_count;
    nt = rem % nt_count;
  }
  r.m0 = m * unit_rows;
  r.row_begin = s_off[lo] + nt * bn;
  r.n_rows = min(bn, n - nt * bn);
  return r;
}

template <bool GU, int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_moe_gemm(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_ws, GemmParams p) {
  using C = GemmCfg<GU, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_off = reinterpret_cast<int*>(smem + STAGES * C::STAGE + 256);
  int* s_up = s_off + kMaxExperts + 1;
  int* s_slot = s_up + kMaxExperts + 1;
  int* s_flag = s_slot + kMaxExperts;

  const int E = p.E;
  const int MT = ((GU ? p.F : p.H) + C::UNIT_ROWS - 1) / C::UNIT_ROWS;
  const int S = GU ? 1 : p.splits;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;

  // ---- prologue: unit prefix + page-table residency check
  if (threadIdx.x == 0) *s_flag = (*(volatile long long*)p.fault != 0);
  for (int e = threadIdx.x; e <= E; e += blockDim.x) s_off[e] = p.offsets[e];
  __syncthreads();
  if (*s_flag) return;
  if (warp == 0) {
    int carry = 0;
    bool bad = false;
    if (lane == 0) s_up[0] = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      int u = 0;
      if (e < E) {
        const int n = s_off[e + 1] - s_off[e];
        // groups read in place run in k_moe_gemm_dec
        if (n > 0 && !(p.dec && e < p.E_routed && p.dec[e].sm && ((p.dec_fmt_mask >> p.dec[e].fmt) & 1u))) {
          u = ((n + BN - 1) / BN) * MT * S;
          if (e < p.E_routed) {
            const int32_t ent = p.pt[e];
            if (pt_state(ent) != 2) {
              atomicCAS((unsigned long long*)p.fault, 0ull,
                        (unsigned long long)fault_pack(p.layer, p.e_first + e + 1, GU ? 1 : 2, pt_state(ent)));
              bad = true;
            }
            s_slot[e] = pt_block0(ent);
          } else {
            s_slot[e] = p.shared_block0 + (e - p.E_routed);  // always-resident shared expert
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
  if (*s_flag || (int)blockIdx.x >= n_units) return;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_b);
    if (p.E > p.E_routed) tma_prefetch_desc(&map_ws);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int K = GU ? p.H : p.F;
  const int KB = (K + kBK - 1) / kBK;
  const int rows_per_block = GU ? 2 * p.F : p.H;
  // Programmatic dependent launch (launch_gate_up / launch_down with pdl): everything above --
  // unit prefix, residency check, barriers, TMEM -- and an L2 prefetch of this CTA's first unit
  // of weights (resident before the previous kernel started: loads are ordered by events) overlap
  // the previous kernel's tail; activations are read and outputs written only after the wait.
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (warp == 0 && lane == 0) {
    const Unit un = decode_unit(blockIdx.x, s_up, s_off, E, BN, S, GU, C::UNIT_ROWS);
    int kb0 = 0, kb1 = KB;
    if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
    const int wrow = s_slot[un.e] * rows_per_block + un.m0;
    const CUtensorMap* mw = un.e < p.E_routed ? &map_w : &map_ws;
    for (int kb = kb0; kb < kb1; ++kb) {
      tma_prefetch_l2_2d(mw, kb * kBK, wrow);
      if (C::NA == 2) tma_prefetch_l2_2d(mw, kb * kBK, wrow + (GU ? p.F : kBM));
    }
  }
  // a down launch paired with counting gate/up launch waits per group on the counters instead
  // (before its h loads); its outputs are written only after its group's gate/up units counted,
  // which happens after that gate/up grid's own wait, so nothing it writes is still being read
  if (GU || !p.unit_done) griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit un = decode_unit(u, s_up, s_off, E, BN, S, GU, C::UNIT_ROWS);
        int kb0 = 0, kb1 = KB;
        if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
        const int nb = (un.n_rows + kBoxRowsB - 1) / kBoxRowsB;
        const int wrow = s_slot[un.e] * rows_per_block + un.m0;
        const CUtensorMap* mw = un.e < p.E_routed ? &map_w : &map_ws;
        const uint32_t bytes = C::NA * C::A_BYTES + (p.act_lo ? 2 : 1) * nb * kBoxRowsB * kBK * 2;
        if (!GU && p.unit_done) {
          const int n = s_off[un.e + 1] - s_off[un.e];
          const int need = ((n + p.unit_bn - 1) / p.unit_bn) * ((p.F + kBM - 1) / kBM);
          for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.unit_done + un.e) : "memory");
            if (v >= need || *(volatile long long*)p.fault != 0) break;
            __nanosleep(200);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE;
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d(sa, mw, &full[stage], kb * kBK, wrow, pol_w);
          if (C::NA == 2) tma_load_2d(sa + C::A_BYTES, mw, &full[stage], kb * kBK, wrow + (GU ? p.F : kBM), pol_w);
          uint8_t* sb = sa + C::NA * C::A_BYTES;
          for (int i = 0; i < nb; ++i) {
            tma_load_2d(sb + i * kBoxRowsB * kBK * 2, &map_b, &full[stage], kb * kBK, un.row_begin + i * kBoxRowsB,
                        pol_b);
            if (p.act_lo)
              tma_load_2d(sb + C::B_BYTES + i * kBoxRowsB * kBK * 2, &map_b, &full[stage], kb * kBK,
                          (int)(un.row_begin + p.act_lo_rows) + i * kBoxRowsB, pol_b);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const Unit un = decode_unit(u, s_up, s_off, E, BN, S, GU, C::UNIT_ROWS);
      int kb0 = 0, kb1 = KB;
        if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
      const uint32_t idesc = idesc_bf16_f32(kBM, (un.n_rows + 15) & ~15);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_par ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + acc * C::ACC_COLS;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + stage * C::STAGE);
          const uint32_t bbase = base + C::NA * C::A_BYTES;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t bdesc = sdesc_k_sw128(bbase + 32 * k);
            const uint64_t bdesc_lo = sdesc_k_sw128(bbase + C::B_BYTES + 32 * k);
            const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
            const uint64_t adesc = sdesc_k_sw128(base + 32 * k);
            umma_bf16(d0, adesc, bdesc, idesc, accum);
            if (p.act_lo) umma_bf16(d0, adesc, bdesc_lo, idesc, 1u);
            if (C::NA == 2) {
              const uint64_t adesc_u = sdesc_k_sw128(base + C::A_BYTES + 32 * k);
              umma_bf16(d0 + 128, adesc_u, bdesc, idesc, accum);
              if (p.act_lo) umma_bf16(d0 + 128, adesc_u, bdesc_lo, idesc, 1u);
            }
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
      const Unit un = decode_unit(u, s_up, s_off, E, BN, S, GU, C::UNIT_ROWS);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_par);
      tc_fence_after();
      const int r = un.m0 + q * 32 + lane;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS;
      if (GU) {
        __nv_bfloat16* hcol = p.hbuf + (size_t)un.row_begin * p.F + r;
        const size_t lo_off = (size_t)p.h_lo_rows * p.F;
        for (int c0 = 0; c0 < un.n_rows; c0 += 16) {
          float g[16], v[16];
          tmem_ld16(tbase + c0, g);
          tmem_ld16(tbase + 128 + c0, v);
          if (r < p.F) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < un.n_rows) {
                __nv_bfloat16 hi, lo;
                split_bf16(silu_f(g[i]) * v[i], &hi, &lo);
                hcol[(size_t)(c0 + i) * p.F] = hi;
                hcol[(size_t)(c0 + i) * p.F + lo_off] = lo;
              }
          }
        }
      } else {
#pragma unroll
        for (int half = 0; half < C::NA; ++half) {  // the unit's 128-row tiles of W_down
          const int rh = r + half * kBM;
          float* out = p.part + un.split * p.split_stride + (size_t)un.row_begin * p.H + rh;
          for (int c0 = 0; c0 < un.n_rows; c0 += 16) {
            float v[16];
            tmem_ld16(tbase + half * 128 + c0, v);
            if (rh < p.H) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (c0 + i < un.n_rows) out[(size_t)(c0 + i) * p.H] = v[i];
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (GU && p.unit_done) {
        // the unit's h rows are stored: count it for the down launch (all 128 epilogue threads'
        // stores, then one fenced release increment)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && lane == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          atomicAdd(p.unit_done + un.e, 1);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ---- instantiations / launchers

using GemmKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, GemmParams);

template <bool GU, int BN, int ST>
static void set_attr() {
  cudaFuncSetAttribute(k_moe_gemm<GU, BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<GU, BN, ST>::SMEM);
}

// Stage counts: the weight bytes in flight per SM set the achieved HBM bandwidth of
// these memory-bound launches, so each token-tile width BN gets as many stages as fit
// in 227 KB (stage = weight tile(s) + BN x 128 B of activations).
// (stage = weight tile(s) + BN x 128 B of each activation plane)
#define XPGB_GU_TILES(X) X(32, 5) X(48, 4) X(64, 4) X(80, 4) X(96, 3) X(128, 3)
#define XPGB_DN_TILES(X) X(32, 5) X(48, 4) X(64, 4) X(80, 4) X(96, 3) X(128, 3) X(256, 2)
// Lean tiles (<= ~175 KB): one stage fewer, so decoder CTAs (10 KB each) fit on the same
// SM.  The paged runner with a compressed tier uses them: a window's GEMM then runs beside
// the decode of the next window instead of waiting for its CTAs to drain (Mixtral, 80%
// budget: 11.3 K -> 13.2 K tok/s; the GEMM alone loses ~1%).
#define XPGB_GU_LEAN(X) X(32, 4) X(48, 3) X(64, 3) X(80, 3) X(96, 2) X(128, 2)
#define XPGB_DN_LEAN(X) X(32, 4) X(48, 3) X(64, 3) X(80, 3) X(96, 2) X(128, 2) X(256, 2)

void set_gemm_attrs() {
#define XPGB_SET_GU(BN, ST) set_attr<true, BN, ST>();
#define XPGB_SET_DN(BN, ST) set_attr<false, BN, ST>();
  XPGB_GU_TILES(XPGB_SET_GU)
  XPGB_DN_TILES(XPGB_SET_DN)
  XPGB_GU_LEAN(XPGB_SET_GU)
  XPGB_DN_LEAN(XPGB_SET_DN)
#undef XPGB_SET_GU
#undef XPGB_SET_DN
}

// Grouped-GEMM launch with programmatic stream serialization (PDL): the CTAs may start
// during the tail of the previous kernel in the stream and wait (griddep_wait) before touching
// its outputs.  XPGB_PDL=0 launches them plainly (A/B).
static void launch_gemm_pdl(GemmKernel kern, int grid, int smem, cudaStream_t s, const CUtensorMap& a,
                            const CUtensorMap& b, const CUtensorMap& c, const GemmParams& p) {
  static const bool pdl = !(getenv("XPGB_PDL") && atoi(getenv("XPGB_PDL")) == 0);
  if (!pdl) {
    kern<<<grid, 192, smem, s>>>(a, b, c, p);
    note_launch();
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a, b, c, p);
  note_launch();
}

void launch_gate_up(const CUtensorMap& map_w, const CUtensorMap& map_x, const CUtensorMap& map_ws,
                    const GemmParams& p, int bn, int grid, cudaStream_t s, bool lean) {
  GemmKernel kern = nullptr;
  int smem = 0;
#define XPGB_PICK_GU(BN, ST) \
  if (bn == BN) { kern = k_moe_gemm<true, BN, ST>; smem = GemmCfg<true, BN, ST>::SMEM; }
  if (lean) {
    XPGB_GU_LEAN(XPGB_PICK_GU)
  } else {
    XPGB_GU_TILES(XPGB_PICK_GU)
  }
#undef XPGB_PICK_GU
  if (!kern) { kern = k_moe_gemm<true, 128, 3>; smem = GemmCfg<true, 128, 3>::SMEM; }
  launch_gemm_pdl(kern, grid, smem, s, map_w, map_x, map_ws, p);
}

void launch_down(const CUtensorMap& map_w, const CUtensorMap& map_h, const CUtensorMap& map_ws,
                 const GemmParams& p, int bn, int grid, cudaStream_t s, bool lean) {
  GemmKernel kern = nullptr;
  int smem = 0;
#define XPGB_PICK_DN(BN, ST) \
  if (bn == BN) { kern = k_moe_gemm<false, BN, ST>; smem = GemmCfg<false, BN, ST>::SMEM; }
  if (lean) {
    XPGB_DN_LEAN(XPGB_PICK_DN)
  } else {
    XPGB_DN_TILES(XPGB_PICK_DN)
  }
#undef XPGB_PICK_DN
  if (!kern) { kern = k_moe_gemm<false, 128, 3>; smem = GemmCfg<false, 128, 3>::SMEM; }
  launch_gemm_pdl(kern, grid, smem, s, map_w, map_h, map_ws, p);
}

}  // namespace xpgb
