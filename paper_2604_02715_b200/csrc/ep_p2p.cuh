#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xpgb {

constexpr int kMaxEpWorld = 16;

// Base pointers of every rank's receive region (this rank's own region included) and of
// every rank's flag array (int32[kMaxEpWorld], slot r written by rank r).
struct EpPeers {
  void* rows[kMaxEpWorld];
  int32_t* flags[kMaxEpWorld];
  int world;
  int rank;
};

// Scatter n rows (src row src_rows[i], or i when src_rows is null) to rank dst_rank[i],
// row dst_row[i] of its region, as bf16 (to_bf16) or f32; the last CTA then releases
// `epoch` into flag slot `rank` of every rank.  counter: a device word private to this
// call site, zero between launches.
void launch_ep_scatter(const float* src, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                       int n, int H, bool to_bf16, const EpPeers& peers, int32_t epoch, unsigned int* counter,
                       int num_sms, cudaStream_t s);
// Combine fused with the split-K reduction: row i = sum of its `splits` partial planes of
// part (split_stride floats apart), scattered like launch_ep_scatter (f32).
void launch_ep_reduce_scatter(const float* part, const long long* fault, int splits, long long split_stride,
                              const int32_t* dst_rank, const int32_t* dst_row, int n, int H, const EpPeers& peers,
                              int32_t epoch, unsigned int* counter, int num_sms, cudaStream_t s);
// Stream-ordered acquire wait until flags[0..world) >= epoch.
void launch_ep_wait(const int32_t* flags, int world, int32_t epoch, cudaStream_t s);

}  // namespace xpgb
