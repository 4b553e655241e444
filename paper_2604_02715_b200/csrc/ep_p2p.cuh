#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xpgb {

constexpr int kMaxEpWorld = 16;
// Layout of a rank's flag region (the first 512 bytes of its window): int32 epoch flags
// [kMaxEpWorld] at 0 (slot r written by rank r), an int32 peer-fault word at kEpFaultWord,
// the scatter's CTA counter at byte 256.
constexpr int kEpFaultWord = 32;  // int32 index
// Fault word of a peer event (moe_kernels.cuh fault_pack layout, kind 3): the peer rank and
// what happened (1 = the peer's step faulted, so its rows are invalid; 2 = no epoch from it
// within the wait bound).
__host__ __device__ inline long long ep_fault(int peer, int what) {
  return 1LL | (3LL << 1) | ((long long)what << 3) | ((long long)(peer + 1) << 8);
}

// Base pointers of every rank's receive region (this rank's own region included) and of
// every rank's flag array (int32[kMaxEpWorld], slot r written by rank r).
struct EpPeers {
  void* rows[kMaxEpWorld];
  int32_t* flags[kMaxEpWorld];
  int world;
  int rank;
};

// Scatter n rows (src row src_rows[i], or i when src_rows is null) to rank dst_rank[i],
// row dst_row[i] of its region, as the two bf16 planes (to_bf16: hi at dst_row, lo lo_rows
// rows later) or f32; the last CTA then releases `epoch` into flag slot `rank` of every rank.
// fault (nullable): this rank's fault word; when set, the rows are not written and every
// peer's fault word is raised before the release.  n_dev (nullable): the row count, read on
// the device (n is then an upper bound).  counter: a device word private to this call site,
// zero between launches.
void launch_ep_scatter(const float* src, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                       int n, const int32_t* n_dev, int H, bool to_bf16, long long lo_rows, const EpPeers& peers,
                       int32_t epoch, const long long* fault, unsigned int* counter, int num_sms, cudaStream_t s);
// Combine fused with the split-K reduction: row i = sum of its `splits` partial planes of
// part (split_stride floats apart), scattered like launch_ep_scatter (f32).
void launch_ep_reduce_scatter(const float* part, const long long* fault, int splits, long long split_stride,
                              const int32_t* dst_rank, const int32_t* dst_row, int n, const int32_t* n_dev, int H,
                              const EpPeers& peers, int32_t epoch, unsigned int* counter, int num_sms,
                              cudaStream_t s);
// Per-step dispatch plan of one rank, on the device (one CTA; no host round trip).  From the
// global routing table routes [world*T][kk] (1-based ids, ascending per row -- the router
// kernel's output) it derives every row position both exchanges need, in the canonical
// orders of expert_parallel.build_plan:
//   send order of a sender s : (owner rank, expert, local token)   -> send_pos
//   expert-major order, owner: (expert, global token)              -> em_pos
//   arrival order at an owner: (sender, expert, local token)       (NCCL all_to_all)
// Outputs (device int32): src_rows/dst_rank/dst_row [T*kk] (this rank's pairs in send
// order), ret_index [T][kk] (send position of each of its (token, slot) pairs), c_rank/c_row
// [n_own] (sender rank and send position of each expert-major row it owns), to_arrival /
// from_arrival [n_own] (expert-major <-> arrival permutation), offsets [count+1], counts
// [2*world+1] (rows sent to each rank, received from each rank, n_own).  scratch: at least
// ep_plan_scratch_words(...) int32.
struct EpPlanOut {
  int32_t *src_rows, *dst_rank, *dst_row, *ret_index, *c_rank, *c_row, *to_arrival, *from_arrival, *offsets, *counts;
};
long long ep_plan_scratch_words(int world, int tokens, int num_experts);
void launch_ep_plan(const int32_t* routes, int tokens, int world, int rank, int kk, int num_experts, int32_t* scratch,
                    const EpPlanOut& out, cudaStream_t s);
// Stream-ordered acquire wait until flags[0..world) >= epoch, bounded (20 s): a missing
// epoch, or a peer's raised fault word, sets this rank's fault word (ep_fault) instead of
// trapping, so the rank's later kernels skip and its report carries the fault.
void launch_ep_wait(const int32_t* flags, int world, int32_t epoch, long long* fault, cudaStream_t s);

}  // namespace xpgb
