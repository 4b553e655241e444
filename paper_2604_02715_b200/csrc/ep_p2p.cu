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

namespace xpgb {

__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One warp per row; float4 loads, bf16x4 (8 B) or float4 stores into the peer's window.
template <bool TO_BF16>
__global__ void __launch_bounds__(256) k_ep_scatter(const float* __restrict__ src, const int32_t* __restrict__ src_rows,
                                                    const int32_t* __restrict__ dst_rank,
                                                    const int32_t* __restrict__ dst_row, int n, int H,
                                                    const __grid_constant__ EpPeers peers, int32_t epoch,
                                                    unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < n; row += gridDim.x * warps) {
    const int sr = src_rows ? src_rows[row] : row;
    const float4* s = reinterpret_cast<const float4*>(src + (size_t)sr * H);
    const size_t drow = (size_t)dst_row[row];
    uint8_t* base = reinterpret_cast<uint8_t*>(peers.rows[dst_rank[row]]);
    if (TO_BF16) {
      uint2* d = reinterpret_cast<uint2*>(base + drow * H * 2);
      for (int c = lane; c < H / 4; c += 32) {
        const float4 v = s[c];
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        d[c] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
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
      __threadfence_system();
      for (int p = 0; p < peers.world; ++p) st_release_sys(peers.flags[p] + peers.rank, epoch);
    }
  }
}

// Combine fused with the split-K reduction: row i of the owner's expert outputs is the sum
// of its split-K partials (part + k * split_stride4 float4s), stored straight into rank
// dst_rank[i]'s return buffer at row dst_row[i]; the last CTA publishes the epoch.  A
// faulted run (a page read before it was resident) writes nothing but still publishes, so
// no peer waits forever.
__global__ void __launch_bounds__(256) k_ep_reduce_scatter(const float* __restrict__ part, const long long* fault,
                                                           int splits, long long split_stride4,
                                                           const int32_t* __restrict__ dst_rank,
                                                           const int32_t* __restrict__ dst_row, int n, int H,
                                                           const __grid_constant__ EpPeers peers, int32_t epoch,
                                                           unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const bool ok = *fault == 0;
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
      __threadfence_system();
      for (int p = 0; p < peers.world; ++p) st_release_sys(peers.flags[p] + peers.rank, epoch);
    }
  }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// The stream waits until every rank has published `epoch` into this rank's flag slots.  A
// peer that never arrives (a crashed rank) traps after 20 s instead of hanging the device.
__global__ void k_ep_wait(const int32_t* flags, int world, int32_t epoch) {
  const int lane = threadIdx.x;
  if (lane < world) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(flags + lane) < epoch) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) __trap();
    }
  }
  __syncwarp();
}

void launch_ep_scatter(const float* src, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                       int n, int H, bool to_bf16, const EpPeers& peers, int32_t epoch, unsigned int* counter,
                       int num_sms, cudaStream_t s) {
  // at least one CTA even with no rows: the epoch must still be published
  const int warps = 8;
  int grid = (n + warps - 1) / warps;
  grid = grid < 1 ? 1 : (grid > num_sms * 4 ? num_sms * 4 : grid);
  if (to_bf16)
    k_ep_scatter<true><<<grid, warps * 32, 0, s>>>(src, src_rows, dst_rank, dst_row, n, H, peers, epoch, counter);
  else
    k_ep_scatter<false><<<grid, warps * 32, 0, s>>>(src, src_rows, dst_rank, dst_row, n, H, peers, epoch, counter);
  note_launch();
}

void launch_ep_reduce_scatter(const float* part, const long long* fault, int splits, long long split_stride,
                              const int32_t* dst_rank, const int32_t* dst_row, int n, int H, const EpPeers& peers,
                              int32_t epoch, unsigned int* counter, int num_sms, cudaStream_t s) {
  const int warps = 8;
  int grid = (n + warps - 1) / warps;
  grid = grid < 1 ? 1 : (grid > num_sms * 4 ? num_sms * 4 : grid);
  k_ep_reduce_scatter<<<grid, warps * 32, 0, s>>>(part, fault, splits, split_stride / 4, dst_rank, dst_row, n, H, peers,
                                                  epoch, counter);
  note_launch();
}

void launch_ep_wait(const int32_t* flags, int world, int32_t epoch, cudaStream_t s) {
  k_ep_wait<<<1, 32, 0, s>>>(flags, world, epoch);
  note_launch();
}

}  // namespace xpgb
