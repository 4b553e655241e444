// Expert-parallel dispatch/combine over peer memory (SURVEY §8(e) fusion target).
//
// Every rank computes the global routing table locally (the router is a pure function of
// (seed, token, layer)), so every rank knows, for each (token, slot) pair, the row it
// occupies in its owner's expert-major input and in its sender's return buffer.  The
// exchange is therefore a scatter: one kernel writes each row straight into the peer's
// window (CUDA IPC mapping over NVLink; a local store for rows that stay home), then its
// last CTA releases the step's epoch into every peer's flag slot.  The receiver's stream
// waits on its flags with an acquire spin.  No count exchange, no staging buffer, no
// permutation pass after arrival: the dispatch lands rows in the layout the grouped GEMM
// reads, and the combine lands them in the order the ordered combine reads.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ep_p2p.cuh"
#include "launch_count.h"
#include "moe_kernels.cuh"

namespace xpgb {

__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Raise every peer's fault word (this rank's rows are invalid), before the epoch release.
__device__ __forceinline__ void ep_publish(const EpPeers& peers, int32_t epoch, bool faulted) {
  if (faulted)
    for (int p = 0; p < peers.world; ++p) atomicExch(peers.flags[p] + kEpFaultWord, peers.rank + 1);
  __threadfence_system();
  for (int p = 0; p < peers.world; ++p) st_release_sys(peers.flags[p] + peers.rank, epoch);
}

// One warp per row; float4 loads, the bf16 hi/lo planes (8 B each) or float4 stores into the
// peer's window.
template <bool TO_BF16>
__global__ void __launch_bounds__(256) k_ep_scatter(const float* __restrict__ src, const int32_t* __restrict__ src_rows,
                                                    const int32_t* __restrict__ dst_rank,
                                                    const int32_t* __restrict__ dst_row, int n,
                                                    const int32_t* __restrict__ n_dev, int H, long long lo_rows,
                                                    const __grid_constant__ EpPeers peers, int32_t epoch,
                                                    const long long* fault, unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const bool faulted = fault && *fault != 0;
  if (n_dev) n = min(n, *n_dev);
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); !faulted && row < n; row += gridDim.x * warps) {
    const int sr = src_rows ? src_rows[row] : row;
    const float4* s = reinterpret_cast<const float4*>(src + (size_t)sr * H);
    const size_t drow = (size_t)dst_row[row];
    uint8_t* base = reinterpret_cast<uint8_t*>(peers.rows[dst_rank[row]]);
    if (TO_BF16) {
      uint2* d = reinterpret_cast<uint2*>(base + drow * H * 2);
      uint2* dl = reinterpret_cast<uint2*>(base + (drow + lo_rows) * H * 2);
      for (int c = lane; c < H / 4; c += 32) {
        const float4 v = s[c];
        __nv_bfloat16 h[4], l[4];
        split_bf16(v.x, &h[0], &l[0]);
        split_bf16(v.y, &h[1], &l[1]);
        split_bf16(v.z, &h[2], &l[2]);
        split_bf16(v.w, &h[3], &l[3]);
        d[c] = *reinterpret_cast<const uint2*>(h);
        dl[c] = *reinterpret_cast<const uint2*>(l);
      }
    } else {
      float4* d = reinterpret_cast<float4*>(base + drow * H * 4);
      for (int c = lane; c < H / 4; c += 32) d[c] = s[c];
    }
  }
  // every CTA makes its stores visible system-wide before it counts itself done; the last
  // CTA then publishes the epoch to every rank (release: the rows happen-before the flag)
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {
      *counter = 0u;
      ep_publish(peers, epoch, faulted);
    }
  }
}

// Combine fused with the split-K reduction: row i of the owner's expert outputs is the sum
// of its split-K partials (part + k * split_stride4 float4s), stored straight into rank
// dst_rank[i]'s return buffer at row dst_row[i]; the last CTA publishes the epoch.  A
// faulted run (a page read before it was resident) writes nothing, raises every peer's fault
// word and still publishes, so no peer waits and no peer combines stale rows silently.
__global__ void __launch_bounds__(256) k_ep_reduce_scatter(const float* __restrict__ part, const long long* fault,
                                                           int splits, long long split_stride4,
                                                           const int32_t* __restrict__ dst_rank,
                                                           const int32_t* __restrict__ dst_row, int n,
                                                           const int32_t* __restrict__ n_dev, int H,
                                                           const __grid_constant__ EpPeers peers, int32_t epoch,
                                                           unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const bool ok = *fault == 0;
  if (n_dev) n = min(n, *n_dev);
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); ok && row < n; row += gridDim.x * warps) {
    const float4* s = reinterpret_cast<const float4*>(part) + (size_t)row * (H / 4);
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(peers.rows[dst_rank[row]]) +
                                          (size_t)dst_row[row] * H * 4);
    for (int c = lane; c < H / 4; c += 32) {
      float4 v = s[c];
      for (int k = 1; k < splits; ++k) {
        const float4 w = s[c + k * split_stride4];
        v.x = __fadd_rn(v.x, w.x); v.y = __fadd_rn(v.y, w.y); v.z = __fadd_rn(v.z, w.z); v.w = __fadd_rn(v.w, w.w);
      }
      d[c] = v;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {
      *counter = 0u;
      ep_publish(peers, epoch, !ok);
    }
  }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// The stream waits until every rank has published `epoch` into this rank's flag slots.  The
// wait is bounded (20 s): a peer that never arrives sets this rank's fault word instead of
// trapping (a trap would destroy the context), and a peer that published a fault marker
// passes it on -- either way this rank's later kernels skip and its RunReport shows it.
__global__ void k_ep_wait(const int32_t* flags, int world, int32_t epoch, long long* fault) {
  const int lane = threadIdx.x;
  // a rank that already faulted skips its waits: its kernels skip and its scatters write no
  // rows, so it needs nothing from its peers (and does not stall 20 s per wait)
  if (fault && *reinterpret_cast<volatile long long*>(fault)) return;
  if (lane < world) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(flags + lane) < epoch) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
        if (fault) atomicCAS(reinterpret_cast<unsigned long long*>(fault), 0ull, (unsigned long long)ep_fault(lane, 2));
        break;
      }
    }
  }
  __syncwarp();
  if (lane == 0 && fault) {
    const int32_t peer = ld_acquire_sys(flags + kEpFaultWord);
    if (peer) atomicCAS(reinterpret_cast<unsigned long long*>(fault), 0ull, (unsigned long long)ep_fault(peer - 1, 1));
  }
}

// ---------------------------------------------------------------- device dispatch plan

// First expert of rank r under shard_bounds (contiguous, balanced; expert_parallel.py).
__device__ __forceinline__ int ep_first(int r, int L, int G) {
  const int base = L / G, rem = L % G;
  return r * base + min(r, rem);
}

__device__ __forceinline__ int ep_owner(int e, int L, int G) {
  const int base = L / G, rem = L % G;
  const int big = rem * (base + 1);
  return e < big ? e / (base + 1) : rem + (e - big) / base;
}

long long ep_plan_scratch_words(int world, int tokens, int num_experts) {
  const long long W = ((long long)world * tokens + 31) / 32 + 1;
  return 2 * (long long)num_experts * W + (long long)(world + 1) * num_experts + (long long)world * (num_experts + 1) +
         2 * (long long)num_experts + 64;
}

__global__ void __launch_bounds__(1024, 1)
    k_ep_plan(const int32_t* __restrict__ routes, int T, int G, int me, int kk, int L, int32_t* __restrict__ scratch,
              EpPlanOut o) {
  const int GT = G * T;
  const int W = (GT + 31) / 32 + 1;  // one spare word: rank(e, GT) reads word GT/32
  uint32_t* M = reinterpret_cast<uint32_t*>(scratch);       // [L][W] token bitmaps per expert
  int32_t* P = scratch + (long long)L * W;                    // [L][W] exclusive popcount prefix
  int32_t* Tb = P + (long long)L * W;                         // [G+1][L] tokens < s*T routed to e
  int32_t* sb = Tb + (long long)(G + 1) * L;                  // [G][L+1] send base of (sender, expert)
  int32_t* ob = sb + (long long)G * (L + 1);                  // [L] expert-major base at the owner
  int32_t* cnt = ob + L;                                      // [L]
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  for (long long i = tid; i < (long long)L * W; i += nth) M[i] = 0u;
  __syncthreads();
  for (int p = tid; p < GT * kk; p += nth) {
    const int g = p / kk, e = routes[p] - 1;
    atomicOr(&M[(long long)e * W + (g >> 5)], 1u << (g & 31));
  }
  __syncthreads();
  // prefix of every expert's bitmap, one warp per expert
  for (int e = warp; e < L; e += nw) {
    int carry = 0;
    for (int w0 = 0; w0 < W; w0 += 32) {
      const int w = w0 + lane;
      const int v = w < W ? __popc(M[(long long)e * W + w]) : 0;
      int x = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (w < W) P[(long long)e * W + w] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) cnt[e] = carry;
  }
  __syncthreads();
  auto rank_of = [&](int e, int g) {  // routed tokens of expert e with global index < g
    const long long i = (long long)e * W + (g >> 5);
    return P[i] + __popc(M[i] & ((1u << (g & 31)) - 1u));
  };
  for (int i = tid; i < (G + 1) * L; i += nth) {
    const int s = i / L, e = i % L;
    Tb[i] = rank_of(e, s * T);
  }
  __syncthreads();
  // send bases (warp per sender) and owner-local expert-major bases (warp per owner)
  for (int job = warp; job < 2 * G; job += nw) {
    const int r = job % G;
    const bool send = job < G;
    const int e_lo = send ? 0 : ep_first(r, L, G), e_hi = send ? L : ep_first(r + 1, L, G);
    int carry = 0;
    for (int e0 = e_lo; e0 < e_hi; e0 += 32) {
      const int e = e0 + lane;
      const int v = e < e_hi ? (send ? Tb[(r + 1) * L + e] - Tb[r * L + e] : cnt[e]) : 0;
      int x = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (e < e_hi) {
        if (send) sb[r * (L + 1) + e] = carry + x - v;
        else ob[e] = carry + x - v;
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (send && lane == 0) sb[r * (L + 1) + L] = carry;
  }
  __syncthreads();
  const int f_me = ep_first(me, L, G), n_me = ep_first(me + 1, L, G) - f_me;
  for (int e = tid; e <= n_me; e += nth) o.offsets[e] = e < n_me ? ob[f_me + e] : (n_me ? ob[f_me + n_me - 1] + cnt[f_me + n_me - 1] : 0);
  if (tid < G) {  // rows this rank sends to rank tid, and receives from rank tid
    const int f = ep_first(tid, L, G), n = ep_first(tid + 1, L, G) - f;
    o.counts[tid] = sb[me * (L + 1) + f + n] - sb[me * (L + 1) + f];
    o.counts[G + tid] = sb[tid * (L + 1) + f_me + n_me] - sb[tid * (L + 1) + f_me];
  }
  if (tid == 0) o.counts[2 * G] = n_me ? ob[f_me + n_me - 1] + cnt[f_me + n_me - 1] : 0;
  __syncthreads();
  for (int p = tid; p < GT * kk; p += nth) {
    const int g = p / kk, slot = p - g * kk, e = routes[p] - 1;
    const int s = g / T, d = ep_owner(e, L, G);
    const int r_e = rank_of(e, g);
    const int send_pos = sb[s * (L + 1) + e] + r_e - Tb[s * L + e];
    const int em = ob[e] + r_e;
    if (s == me) {
      o.src_rows[send_pos] = g - s * T;
      o.dst_rank[send_pos] = d;
      o.dst_row[send_pos] = em;
      o.ret_index[(g - s * T) * kk + slot] = send_pos;
    }
    if (d == me) {
      o.c_rank[em] = s;
      o.c_row[em] = send_pos;
      int recv_base = 0;  // rows from senders before s
      for (int q = 0; q < s; ++q) recv_base += sb[q * (L + 1) + f_me + n_me] - sb[q * (L + 1) + f_me];
      const int arr = recv_base + send_pos - sb[s * (L + 1) + f_me];
      o.to_arrival[em] = arr;
      o.from_arrival[arr] = em;
    }
  }
}

void launch_ep_plan(const int32_t* routes, int tokens, int world, int rank, int kk, int num_experts, int32_t* scratch,
                    const EpPlanOut& out, cudaStream_t s) {
  k_ep_plan<<<1, 1024, 0, s>>>(routes, tokens, world, rank, kk, num_experts, scratch, out);
  note_launch();
}

void launch_ep_scatter(const float* src, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                       int n, const int32_t* n_dev, int H, bool to_bf16, long long lo_rows, const EpPeers& peers,
                       int32_t epoch, const long long* fault, unsigned int* counter, int num_sms, cudaStream_t s) {
  // at least one CTA even with no rows: the epoch must still be published
  const int warps = 8;
  int grid = (n + warps - 1) / warps;
  grid = grid < 1 ? 1 : (grid > num_sms * 4 ? num_sms * 4 : grid);
  if (to_bf16)
    k_ep_scatter<true><<<grid, warps * 32, 0, s>>>(src, src_rows, dst_rank, dst_row, n, n_dev, H, lo_rows, peers,
                                                   epoch, fault, counter);
  else
    k_ep_scatter<false><<<grid, warps * 32, 0, s>>>(src, src_rows, dst_rank, dst_row, n, n_dev, H, lo_rows, peers,
                                                    epoch, fault, counter);
  note_launch();
}

void launch_ep_reduce_scatter(const float* part, const long long* fault, int splits, long long split_stride,
                              const int32_t* dst_rank, const int32_t* dst_row, int n, const int32_t* n_dev, int H,
                              const EpPeers& peers, int32_t epoch, unsigned int* counter, int num_sms,
                              cudaStream_t s) {
  const int warps = 8;
  int grid = (n + warps - 1) / warps;
  grid = grid < 1 ? 1 : (grid > num_sms * 4 ? num_sms * 4 : grid);
  k_ep_reduce_scatter<<<grid, warps * 32, 0, s>>>(part, fault, splits, split_stride / 4, dst_rank, dst_row, n, n_dev,
                                                  H, peers, epoch, counter);
  note_launch();
}

void launch_ep_wait(const int32_t* flags, int world, int32_t epoch, long long* fault, cudaStream_t s) {
  k_ep_wait<<<1, 32, 0, s>>>(flags, world, epoch, fault);
  note_launch();
}

}  // namespace xpgb
