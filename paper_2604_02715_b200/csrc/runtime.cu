// Runtime behind the C ABI (include/xpgb.h): context, pinned host pool,
// device tier, PagedTensor (host bookkeeping + device slot table), page-in
// engine on two copy streams with RAW/WAR event ordering, ordering log,
// and the MoE forward pipeline.
//
// Reference mapping (xpg 0.1.0):
//   PageTable            paging.py:97-271      -> PageTableHost + d_pt (device slot table)
//   StorageHierarchy     storage.py:214-243    -> host pool (pinned) + device tier, fetch()
//   StreamedRunner       pipeline.py:299-483   -> run(): copy streams = loaders, compute stream
//   OrderingLog          pipeline.py:94-116    -> device log written by stream-ordered kernels
//   layer_forward        pipeline.py:192-208   -> enqueue_forward(): route/plan/gather/GEMMs/combine
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <set>
#include <thread>
#include <string>
#include <vector>

#include "../../include/xpgb.h"
#include "codec.cuh"
#include "fx4.cuh"
#include "ep_p2p.cuh"
#include "launch_count.h"
#include "moe_kernels.cuh"
#include "ptx_sm100.cuh"

namespace xpgb {

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static thread_local std::string g_err;

struct Err {
  int code;
  std::string msg;
};

static std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

#define XFAIL(code, ...) throw Err{code, fmt(__VA_ARGS__)}
#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw Err{XPGB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define CKLAUNCH() CK(cudaGetLastError())

template <class Fn>
static int guard(Fn&& fn) {
  try {
    fn();
    return XPGB_OK;
  } catch (const Err& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return XPGB_ERR;
  }
}

// --------------------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) XFAIL(XPGB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
// Row-major bf16 [rows][cols] -> box {64 cols, box_rows}, 128-B swizzle.
static CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) XFAIL(XPGB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r,
                               (unsigned long long)rows, (unsigned long long)cols);
  return m;
}

// Row-major bytes [rows][cols] -> box {box_cols, 128 rows} (FX4 planes of the device tier).
static CUtensorMap make_map_u8(const void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                               CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols};
  cuuint32_t box[2] = {box_cols, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) XFAIL(XPGB_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed (%d) rows=%llu cols=%llu", (int)r,
                               (unsigned long long)rows, (unsigned long long)cols);
  return m;
}

// --------------------------------------------------------------------------- small kernels

struct PtOp {
  int32_t* unmap_row;
  int32_t unmap_n;
  int32_t set_n;
  int32_t* set_row;
  xpgb_record* log;
  int32_t* log_count;
  int32_t log_cap;
  int32_t n_rec;
  int32_t rec[3][7];  // event, it, layer, kind, target_it, target_layer, group word
  int32_t vals[448];
};
static_assert(sizeof(PtOp) < 4000, "kernel parameter block too large");

__device__ void write_record(xpgb_record* log, int32_t* count, int cap, const int32_t* r) {
  const int t = atomicAdd(count, 1);
  if (t < cap) {
    xpgb_record rec;
    rec.t = t;
    rec.event = r[0];
    rec.iteration = r[1];
    rec.layer = r[2];
    rec.kind = r[3];
    rec.target_iteration = r[4];
    rec.target_layer = r[5];
    rec.group = r[6];
    rec.wall_ns = (int64_t)globaltimer_ns();
    log[t] = rec;
    __threadfence();
  }
}

// Stream-ordered page-table update + ordering-log append (copy streams and compute stream).
__global__ void k_pt_op(PtOp op) {
  if (threadIdx.x == 0 && op.log && op.n_rec > 0) write_record(op.log, op.log_count, op.log_cap, op.rec[0]);
  __syncthreads();
  for (int i = threadIdx.x; i < op.unmap_n; i += blockDim.x) op.unmap_row[i] = -1;
  for (int i = threadIdx.x; i < op.set_n; i += blockDim.x) op.set_row[i] = op.vals[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && op.log)
    for (int i = 1; i < op.n_rec; ++i) write_record(op.log, op.log_count, op.log_cap, op.rec[i]);
}

__global__ void k_sleep(uint64_t ns) {
  const uint64_t t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(20000);
}

// --------------------------------------------------------------------------- context

static const char* state_name(int s) {
  switch (s) {
    case XPGB_PAGE_LOADING: return "loading";
    case XPGB_PAGE_RESIDENT: return "resident";
    case XPGB_PAGE_EVICTING: return "evicting";
    default: return "unmapped";
  }
}

struct Session;

constexpr int kEvRing = 8;        // load / compute events per step, indexed g % kEvRing
constexpr int kMaxRingDepth = 6;  // windows in flight (< kEvRing)

struct Ctx {
  Session* sess = nullptr;
  int N, L, H, F;
  int device;
  int pool;
  int e_first = 0, E = 0;  // expert shard
  int S = 0;               // shared (always-on, always-resident) experts per layer
  int sh0 = 0, sh1 = 0x7fffffff;  // step rows that pass through the shared experts
  uint8_t* shared_w = nullptr;  // [N*S] gate/up blocks, then [N*S] down blocks
  CUtensorMap map_gu_sh{}, map_dn_sh{};
  uint64_t s1, s2;         // sigma per kind
  int num_sms = 148;

  // device pool (arena): kind-1 blocks then kind-2 blocks (paging.py:115-122)
  int blocks = 0;
  uint8_t* arena = nullptr;
  CUtensorMap map_gu{}, map_dn{};

  // host pool (shard-local container order)
  uint8_t* host = nullptr;
  uint64_t host_bytes = 0;
  bool host_owned = false, host_registered = false;

  // device tier
  std::vector<uint8_t> backend;  // [N*E][2] 0 host, 1 device
  uint8_t* dev_tier = nullptr;
  std::vector<int64_t> dev_off;  // [N*E][2] offset of the tensor in dev_tier or -1

  // page table (host bookkeeping)
  std::vector<int8_t> st[2];
  std::vector<int32_t> blk[2];  // 1-based block or 0
  std::vector<int32_t> owner[2];  // block -> page index or -1
  std::set<int32_t> free_ids[2];
  uint64_t bound = 0, peak = 0;
  long long step = 0;
  bool trace_on = false;
  std::string trace;
  int32_t* d_pt = nullptr;  // [2][N*E] device slot table
  std::vector<uint8_t> pinned;  // [N*E] permanently resident experts (residency tier x > 0)
  int ring_blocks = 0;          // blocks per kind that cycle through the schedule
  int ring_limit = 0;           // cap on ring blocks per kind (sub-layer ring); 0 = 2 x streamed experts
  int ring_depth = 2;           // windows in flight on a sub-layer ring (window g recycles g - depth)
  int ep_splits = 1, ep_rows = 0;  // last experts_forward_range: split-K planes and rows in part
  long long ep_split_stride = 0;

  // streams / events
  cudaStream_t s_copy[2] = {nullptr, nullptr};
  cudaStream_t s_comp = nullptr;
  cudaEvent_t ev_load[2][kEvRing], ev_comp[kEvRing], ev_begin, ev_end;

  // workspace
  int cap_T = 0, cap_kk = 0, cap_rows = 0, cap_splits = 8;
  long long part_rows = 0;  // rows of `part`: split-K planes are packed at the launch's row count
  // routing plans: buffer 0/1 alternate per iteration of a run, buffer 2 serves layer_forward
  int32_t* plan_topk[3] = {nullptr, nullptr, nullptr};  // [N][T][kk]
  int32_t* plan_pos[3] = {nullptr, nullptr, nullptr};   // [N][T][kk]
  int32_t* plan_off[3] = {nullptr, nullptr, nullptr};   // [N][E+1]
  int32_t* plan_scr[3] = {nullptr, nullptr, nullptr};   // [2][N][E] multi-CTA plan counters
  __nv_bfloat16* xp = nullptr;    // [2][cap_rows][H]: hi plane, lo plane (moe_kernels.cuh: split_bf16)
  __nv_bfloat16* hbuf = nullptr;  // [2][cap_rows][F]
  float* part = nullptr;          // [part_rows][H]: splits x (rows of a launch) x H
  int32_t* ep_off = nullptr;      // [E+1] scratch for experts_forward
  int last_splits = 1;
  CUtensorMap map_xp{}, map_h{};
  CUtensorMap map_xp_pair{}, map_h_pair{};  // 128-row boxes: the CTA-pair prefill GEMM's A operand
  CUtensorMap map_ep_x{}, map_ep_x_pair{};   // caller rows of experts_forward_range (built per buffer)
  const void* ep_rows_ptr = nullptr;
  long long ep_lo_rows = 0;
  int pair_mode = -1;                        // CTA-pair GEMM: -1 auto (prefill-sized groups), 0 off, 1 always
  bool pair_split = true;                    // CTA-pair GEMM takes both activation planes (XPGB_FAST_PREFILL=1: hi only)
  long long* d_fault = nullptr;

  // log
  xpgb_record* d_log = nullptr;
  int32_t* d_log_count = nullptr;
  int log_cap = 0;
  std::vector<xpgb_record> last_log;

  // exponent codec (compressed tiers)
  bool codec = false, host_codec = false;
  const uint8_t* cpool = nullptr;  // packed records, container order of this shard (pinned host)
  uint64_t cpool_bytes = 0;
  std::vector<uint64_t> rec_off, rec_bits;  // [N*E*2]
  CodecTable ctab{};
  int cchunk = 1024;
  // staging ring per kind: n_stage buffers of stage_cap bytes.  Host-tier copies wait only
  // for their buffer's previous decode (never for the ring's WAR), so the link runs up to
  // n_stage - 1 pieces ahead of the decoder, across windows and layers.
  uint8_t* stage[2][kMaxStageBufs] = {};  // [kind][buffer]
  int n_stage = 4;  // a whole 156 MB Mixtral gate/up record + one piece in flight (80% budget: +9%)
  uint32_t stage_next[2] = {0, 0};
  uint32_t* d_index = nullptr;           // chunk indexes of host-tier records, device-resident
  std::vector<uint64_t> d_index_off;     // [N*E*2] offset (entries) into d_index
  uint64_t stage_cap[2] = {0, 0};
  cudaStream_t s_dec[2] = {nullptr, nullptr};
  cudaStream_t s_cp[2] = {nullptr, nullptr};   // staged host-tier copies (even buffers)
  cudaStream_t s_alt[2] = {nullptr, nullptr};  // staged host-tier copies (odd buffers): hides turnaround
  cudaStream_t s_devdec[2] = {nullptr, nullptr};  // device-tier decodes: never queue behind the link
  cudaEvent_t ev_copied[2][kMaxStageBufs], ev_decoded[2][kMaxStageBufs], ev_mapped[2], ev_raw[2], ev_devdec[2];
  bool codec_events = false;
  // decode-into-GEMM (moe_gemm_dec.cu): device-tier experts are read in place by the GEMM
  // instead of being expanded into their ring block.  fused_mode: 0 off (default; external
  // compute such as the EP runner reads ring blocks), 1 on for the builtin compute;
  // fused_now: on for the current run/session (decode-sized groups, supported shape).
  int fused_mode = 0;  // 2: FX4 tensors in place, Huffman device-tier tensors expanded into the ring
  bool fused_now = false;
  // race hardening (xpgb_set_hazard_checks): poison every block a window maps with 0xFF
  // bytes (bf16 NaN) before its load, and optionally skip one step's WAR wait, so a WAR
  // hazard shows up as NaNs in the results as well as a violation in the ordering log
  bool poison = false;
  int war_sab_it = 0, war_sab_layer = 0;
  DecRec* d_decrec = nullptr;  // [N][2][E]: record of each device-tier tensor (sm == nullptr: not device tier)
  CUtensorMap* d_fxmaps = nullptr;  // [N*E*2][2]: FX4 sign/mantissa and nibble planes as TMA maps
  // device-tier record format per tensor [N*E*2]: 0 exponent-Huffman (the host pool's records,
  // staged as they are), 1 FX4 (fx4.cuh: encoded on the GPU from the raw pool at staging)
  std::vector<uint8_t> tfmt;
  std::vector<int> fx_base;         // [N*E*2] FX4 base exponent of each device-tier tensor
  std::vector<uint64_t> fx_bytes;   // [N*E*2] FX4 record bytes

  // profiling
  bool prof = false;
  cudaEvent_t pev[7];
  cudaEvent_t* cur_ev = nullptr;          // 7 events bracketing the next enqueue_forward
  std::vector<cudaEvent_t> run_ev;        // per-step event sets for opts.profile
  // opts.profile: every exponent-decoder launch of the run bracketed by events on its own
  // stream, with its algorithmic bytes (records read + bf16 written) -- xpgb_decode_stats
  std::vector<cudaEvent_t> dec_ev;
  std::vector<uint64_t> dec_bytes;
  // decode-into-GEMM launches of a profiled run: events around each launch (compute stream),
  // the record bytes of the experts it read in place
  std::vector<cudaEvent_t> fz_ev;
  std::vector<uint64_t> fz_bytes;
  size_t fz_n = 0;
  // sampled profiling (opts.profile >= 2): events bracket 1 in prof_every decoder / fused launches
  int prof_every = 1, prof_mode = 0;
  int* d_unit_done = nullptr;  // per-group gate/up unit counters of the fused gate/up -> down overlap
  int act_planes = 2;          // activation planes the 1-CTA GEMMs multiply (xpgb_set_activation_planes)
  size_t dec_seen = 0, fz_seen = 0;
  bool dec_skip = false, fz_skip = false;
  double fz_total_ns = 0;
  uint64_t fz_total_bytes = 0, fz_launches = 0;
  size_t dec_n = 0;
  double dec_total_ns = 0;
  uint64_t dec_total_bytes = 0, dec_launches = 0;
  xpgb_kernel_times last_times{};  // last xpgb_profile_layer
};

static int page_index(Ctx* c, int layer, int expert, int kind) {
  if (layer < 1 || layer > c->N) XFAIL(XPGB_ERR_OUT_OF_RANGE, "layer %d outside [1, %d]", layer, c->N);
  if (expert < 1 || expert > c->L) XFAIL(XPGB_ERR_OUT_OF_RANGE, "expert %d outside [1, %d]", expert, c->L);
  if (kind != 1 && kind != 2) XFAIL(XPGB_ERR_OUT_OF_RANGE, "unknown tensor kind %d", kind);
  const int el = expert - 1 - c->e_first;
  if (el < 0 || el >= c->E)
    XFAIL(XPGB_ERR_OUT_OF_RANGE, "expert %d outside this shard [%d, %d]", expert, c->e_first + 1,
          c->e_first + c->E);
  return (layer - 1) * c->E + el;
}

// Plan slots per token: routed min(top_k, L) + shared S.
static int slots_of(Ctx* c, int top_k) { return std::min(top_k, c->L) + c->S; }
static int groups_of(Ctx* c) { return c->E + c->S; }

static std::string tid_str(int layer, int expert, int kind) { return fmt("L%dE%dK%d", layer, expert, kind); }

static uint64_t sigma_of(Ctx* c, int kind) { return kind == 1 ? c->s1 : c->s2; }

static uint8_t* block_ptr(Ctx* c, int kind, int block1) {
  return kind == 1 ? c->arena + (uint64_t)(block1 - 1) * c->s1
                   : c->arena + (uint64_t)c->blocks * c->s1 + (uint64_t)(block1 - 1) * c->s2;
}

static void emit(Ctx* c, const char* ev, int layer, int expert, int kind, int block, const char* extra) {
  if (!c->trace_on) return;
  c->trace += fmt("event=%s layer=%d expert=%d kind=%d block=%d t=%lld", ev, layer, expert, kind, block, c->step);
  if (extra && *extra) {
    c->trace += " ";
    c->trace += extra;
  }
  c->trace += "\n";
}

static void free_pools(Ctx* c) {
  if (c->arena) cudaFree(c->arena);
  if (c->d_pt) cudaFree(c->d_pt);
  if (c->dev_tier) cudaFree(c->dev_tier);
  if (c->d_decrec) cudaFree(c->d_decrec);
  c->d_decrec = nullptr;
  if (c->d_fxmaps) cudaFree(c->d_fxmaps);
  c->d_fxmaps = nullptr;
  if (c->d_unit_done) cudaFree(c->d_unit_done);
  c->d_unit_done = nullptr;
  c->arena = nullptr;
  c->d_pt = nullptr;
  c->dev_tier = nullptr;
}

static void init_pools(Ctx* c, int ring_blocks = -1, int pinned_blocks = 0) {
  free_pools(c);
  c->ring_blocks = ring_blocks >= 0 ? ring_blocks : ((c->pool == XPGB_POOL_RING) ? 2 * c->E : c->N * c->E);
  c->blocks = c->ring_blocks + pinned_blocks;
  const uint64_t bytes = (uint64_t)c->blocks * (c->s1 + c->s2);
  CK(cudaMalloc(&c->arena, bytes));
  CK(cudaMemset(c->arena, 0, bytes));
  const size_t pages = (size_t)c->N * c->E;
  CK(cudaMalloc(&c->d_pt, 2 * pages * sizeof(int32_t)));
  CK(cudaMemset(c->d_pt, 0xFF, 2 * pages * sizeof(int32_t)));
  for (int k = 0; k < 2; ++k) {
    c->st[k].assign(pages, XPGB_PAGE_UNMAPPED);
    c->blk[k].assign(pages, 0);
    c->owner[k].assign(c->blocks + 1, -1);
    c->free_ids[k].clear();
    for (int b = 1; b <= c->blocks; ++b) c->free_ids[k].insert(b);
  }
  c->bound = c->peak = 0;
  c->step = 0;
  c->backend.assign(pages * 2, 0);
  c->dev_off.assign(pages * 2, -1);
  c->pinned.assign(pages, 0);
  c->map_gu = make_map(c->arena, (uint64_t)c->blocks * 2 * c->F, c->H, kBM);
  c->map_dn = make_map(c->arena + (uint64_t)c->blocks * c->s1, (uint64_t)c->blocks * c->H, c->F, kBM);
}

static void ensure_log(Ctx* c, int cap) {
  if (cap <= c->log_cap) {
    CK(cudaMemset(c->d_log_count, 0, sizeof(int32_t)));
    return;
  }
  if (c->d_log) cudaFree(c->d_log);
  CK(cudaMalloc(&c->d_log, (size_t)cap * sizeof(xpgb_record)));
  c->log_cap = cap;
  CK(cudaMemset(c->d_log_count, 0, sizeof(int32_t)));
}

static void free_work(Ctx* c) {
  auto fr = [](void* p) { if (p) cudaFree(p); };
  for (int b = 0; b < 3; ++b) {
    fr(c->plan_topk[b]); fr(c->plan_pos[b]); fr(c->plan_off[b]); fr(c->plan_scr[b]);
    c->plan_topk[b] = c->plan_pos[b] = c->plan_off[b] = c->plan_scr[b] = nullptr;
  }
  fr(c->xp); fr(c->hbuf); fr(c->part); fr(c->ep_off);
  c->xp = c->hbuf = nullptr;
  c->part = nullptr;
  c->ep_off = nullptr;
  c->cap_T = c->cap_kk = c->cap_rows = 0;
}

static void ensure_work(Ctx* c, int T, int kk) {
  if (kk > kMaxTopK)
    XFAIL(XPGB_ERR_OUT_OF_RANGE, "top_k + shared experts = %d slots above the kernel limit %d", kk, kMaxTopK);
  if (T <= c->cap_T && kk <= c->cap_kk && c->xp) return;
  const int nT = std::max(T, std::max(c->cap_T, 16));
  const int nkk = std::max(kk, c->cap_kk);
  CK(cudaDeviceSynchronize());
  free_work(c);
  const long long rows = (long long)nT * nkk;
  const int E = groups_of(c), N = c->N;
  for (int b = 0; b < 3; ++b) {
    CK(cudaMalloc(&c->plan_topk[b], (size_t)N * rows * 4));
    CK(cudaMalloc(&c->plan_pos[b], (size_t)N * rows * 4));
    CK(cudaMalloc(&c->plan_off[b], (size_t)N * (E + 1) * 4));
    CK(cudaMalloc(&c->plan_scr[b], (size_t)2 * N * E * 4));
  }
  CK(cudaMalloc(&c->xp, (size_t)2 * rows * c->H * 2));  // hi rows, then lo rows
  CK(cudaMemset(c->xp, 0, (size_t)2 * rows * c->H * 2));
  CK(cudaMalloc(&c->hbuf, (size_t)2 * rows * c->F * 2));
  CK(cudaMemset(c->hbuf, 0, (size_t)2 * rows * c->F * 2));
  // split-K only pays for few rows (decode); prefill launches run unsplit, so the partial
  // buffer holds all rows once, or up to 8 planes of small launches
  c->part_rows = std::max<long long>(rows, (long long)c->cap_splits * std::min<long long>(rows, 4096));
  CK(cudaMalloc(&c->part, (size_t)c->part_rows * c->H * 4));
  CK(cudaMalloc(&c->ep_off, (size_t)(E + 1) * 4));
  c->cap_T = nT;
  c->cap_kk = nkk;
  c->cap_rows = (int)rows;
  c->map_xp = make_map(c->xp, 2 * rows, c->H, kBoxRowsB);
  c->map_h = make_map(c->hbuf, 2 * rows, c->F, kBoxRowsB);
  c->map_xp_pair = make_map(c->xp, 2 * rows, c->H, kBM);
  c->map_h_pair = make_map(c->hbuf, 2 * rows, c->F, kBM);
}

// Token-tile width of the 1-CTA kernels: the smallest instantiated BN covering the
// expected rows of an expert group (mean + 2 sd of the binomial count), so the weight
// tiles of a memory-bound launch get the most pipeline stages (moe_kernels.cu).
static int pick_bn_rows(double avg_rows) {
  static const int forced = [] {  // XPGB_BN: tile experiments (profiling only)
    const char* e = getenv("XPGB_BN");
    return e ? atoi(e) : 0;
  }();
  if (forced) return forced;
  const double want = avg_rows + 2.0 * std::sqrt(std::max(avg_rows, 0.0));
  for (int bn : {32, 48, 64, 80, 96}) if (want <= bn) return bn;
  return 128;
}

static double avg_group_rows(Ctx* c, int T, int kk) {
  const double local = (double)T * kk * c->E / c->L + (double)std::max(0, std::min(T, c->sh1) - c->sh0) * c->S;
  return local / std::max(1, c->E + c->S);
}

static int pick_bn(Ctx* c, int T, int kk) { return pick_bn_rows(avg_group_rows(c, T, kk)); }

// Decode-into-GEMM tile: every extra token tile of an expert decodes its weights again, so
// cover mean + 3 sd of the rows per expert (capped at the 128-column accumulators).
static int pick_bn_dec(Ctx* c, int T, int kk) {
  static const int force = getenv("XPGB_BN_DEC") ? atoi(getenv("XPGB_BN_DEC")) : 0;  // A/B
  if (force == 32 || force == 48 || force == 64 || force == 80 || force == 96 || force == 128) return force;
  const double avg = avg_group_rows(c, T, kk);
  const double want = avg + 3.0 * std::sqrt(std::max(avg, 0.0));
  for (int bn : {32, 48, 64, 80, 96}) if (want <= bn) return bn;
  return 128;
}

// Lean GEMM tiles while a compressed tier decodes on the SMs of a paged run (moe_kernels.cu:
// XPGB_GU_LEAN); XPGB_COSCHED=0/1 forces either.
static bool lean_gemm(const Ctx* c) {
  static const int force = [] {
    const char* e = getenv("XPGB_COSCHED");
    return e ? atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  return c->codec && c->pool == XPGB_POOL_RING && c->ring_blocks > 0;  // something is decoded each step
}

// Down projection at prefill sizes: N = 256 token rows per tile halves the weight-tile
// re-reads and the smem traffic per MMA flop (one 256-column accumulator, double-buffered).
static int pick_bn_down(Ctx* c, int T, int kk) {
  return avg_group_rows(c, T, kk) >= 384 ? 256 : pick_bn(c, T, kk);
}

// Split-K factor for the down projection: balance (units x splits) over the SMs.
static int pick_splits(Ctx* c, int T, int kk, int bn) {
  const int KB = (c->F + kBK - 1) / kBK;
  const long long max_s = std::min<long long>(c->cap_splits, c->part_rows / std::max<long long>(1, (long long)T * kk));
  const long long active = std::min<long long>(c->E, (long long)T * kk);
  if (active <= 0) return 1;
  const long long rows_per = std::max<long long>(1, ((long long)T * kk + active - 1) / active);
  const int unit_rows = bn <= 128 ? 2 * kBM : kBM;  // k_moe_gemm<down>: two 128-row tiles per unit at bn <= 128
  const long long tiles = active * ((c->H + unit_rows - 1) / unit_rows) * ((rows_per + bn - 1) / bn);
  int best = 1;
  double best_eff = -1;
  for (int s = 1; s <= max_s; ++s) {
    if (KB / s < 4) break;
    const double work = (double)tiles * s / c->num_sms;
    const double eff = work / std::ceil(work) * std::min(1.0, work);  // wave quantisation x fill
    if (eff > best_eff + 0.02) { best_eff = eff; best = s; }
  }
  return best;
}

static void prof_rec(Ctx* c, int i, cudaStream_t s) {
  if (c->cur_ev) CK(cudaEventRecord(c->cur_ev[i], s));
  else if (c->prof) CK(cudaEventRecord(c->pev[i], s));
}

// Expert groups of >= 128 rows on average run on CTA pairs (256 x 256 tiles, unsplit);
// measured crossover on B200 (profiles/r1_pair_crossover.jsonl): at 64 rows per expert the
// 1-CTA swap-AB kernel is ahead, from 128 rows the pair kernel wins (up to 2.4x at 8K rows)
static bool use_pair(Ctx* c, int T, int kk) {
  return pair_gemm_supported(c->H, c->F) &&
         (c->pair_mode == 1 || (c->pair_mode < 0 && avg_group_rows(c, T, kk) >= 128.0));
}

// Decode-into-GEMM for this run: builtin compute asked for it, a compressed device tier
// exists, the shape is supported and the groups are decode-sized (1-CTA kernels).
static bool fused_for(Ctx* c, int T, int top_k) {
  return c->fused_mode != 0 && c->codec && c->d_decrec && c->pool == XPGB_POOL_RING &&
         gemm_dec_supported(c->H, c->F, c->cchunk) && !use_pair(c, T, std::min(top_k, c->L));
}

static int fmt_of(const Ctx* c, size_t ti) { return c->tfmt.empty() ? 0 : c->tfmt[ti]; }

// Device-tier formats read in place by this run's decode-into-GEMM launches (bit f: format f).
static uint32_t fused_fmt_mask(const Ctx* c) {
  if (!c->fused_now) return 0;
  return c->fused_mode == 2 ? 2u : 3u;
}

// Is tensor (layer, local expert e, kind) read in place by the decode-into-GEMM kernel?
static bool fused_tensor(const Ctx* c, int layer, int e, int kind) {
  if (!c->fused_now || e >= c->E) return false;
  const size_t ti = ((size_t)(layer - 1) * c->E + e) * 2 + (kind - 1);
  return c->backend[ti] == 1 && c->pinned[(size_t)(layer - 1) * c->E + e] == 0 &&
         ((fused_fmt_mask(c) >> fmt_of(c, ti)) & 1u);
}

// Profiled runs (c->cur_ev set by session_compute): events around each decode-into-GEMM launch.
static void fz_mark(Ctx* c, cudaStream_t s, uint64_t bytes, bool begin) {
  if (!c->prof_mode) return;
  if (begin) {
    c->fz_skip = (c->fz_seen++ % (size_t)c->prof_every) != 0;
    if (c->fz_skip) return;
    while (c->fz_ev.size() < 2 * (c->fz_n + 1)) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->fz_ev.push_back(e);
    }
    if (c->fz_bytes.size() < c->fz_n + 1) c->fz_bytes.resize(c->fz_n + 1);
    c->fz_bytes[c->fz_n] = bytes;
    CK(cudaEventRecord(c->fz_ev[2 * c->fz_n], s));
  } else {
    if (c->fz_skip) return;
    CK(cudaEventRecord(c->fz_ev[2 * c->fz_n + 1], s));
    ++c->fz_n;
  }
}

// Record bytes the decode-into-GEMM launch of window [e0, e1), kind, reads in place.
static uint64_t fused_bytes(Ctx* c, int layer, int e0, int e1, int kind, int fmt) {
  uint64_t b = 0;
  for (int e = e0; e < std::min(e1, c->E); ++e) {
    if (!fused_tensor(c, layer, e, kind)) continue;
    const size_t ti = ((size_t)(layer - 1) * c->E + e) * 2 + (kind - 1);
    if (fmt_of(c, ti) != fmt) continue;
    const uint64_t n = ((kind == 2) ? c->s2 : c->s1) / 2;
    b += fmt_of(c, ti) == 1 ? c->fx_bytes[ti] : xpgb_codec_record_bytes(n, c->rec_bits[ti], c->cchunk);
  }
  return b;
}

static GemmParams gemm_params(Ctx* c, int layer, int kind, const int32_t* offsets, int splits,
                              bool with_shared = true) {
  GemmParams p;
  p.offsets = offsets;
  p.pt = c->d_pt + (size_t)(kind - 1) * c->N * c->E + (size_t)(layer - 1) * c->E;
  p.fault = c->d_fault;
  p.act_lo_rows = c->cap_rows;
  p.h_lo_rows = c->cap_rows;
  p.hbuf = c->hbuf;
  p.part = c->part;
  p.split_stride = 0;  // set per launch: (rows of the launch) x H
  p.layer = layer;
  p.e_first = c->e_first;
  p.E = with_shared ? groups_of(c) : c->E;
  p.E_routed = c->E;
  p.shared_block0 = (layer - 1) * c->S;
  p.F = c->F;
  p.H = c->H;
  p.splits = splits;
  p.dec = nullptr;
  p.dec_fmt_mask = 0;
  p.unit_done = nullptr;
  p.unit_bn = 0;
  p.act_lo = c->act_planes >= 2 ? 1 : 0;
  return p;
}

// Plan (route + positions) layers [1, N] of one iteration into buffer b.
static void enqueue_plan(Ctx* c, int b, int layer_first, int layer_count, int T, int top_k, uint64_t seed,
                         cudaStream_t s) {
  const int kt = slots_of(c, top_k);
  const size_t lo = (size_t)(layer_first - 1);
  launch_route_plan(seed, layer_first, layer_count, T, c->L, top_k, c->e_first, c->E, c->S, c->sh0, c->sh1,
                    c->plan_topk[b] + lo * T * kt, c->plan_pos[b] + lo * T * kt,
                    c->plan_off[b] + lo * (groups_of(c) + 1), c->plan_scr[b], c->d_fault, s);
  CKLAUNCH();
}

// layer_forward (pipeline.py:192-208) on `s` from plan buffer b; y may alias x.
// Window [e0, e1) of local expert groups: the GEMMs of those experts only (rows are
// absolute, so windows of one layer write disjoint rows); `last` runs the combine.
// gather: x -> expert-major bf16 rows first (else the previous combine already did it);
// next_pos: fuse the next layer's gather into this layer's combine.
static void enqueue_window(Ctx* c, int layer, const float* x, float* y, int T, int top_k, int b, bool gather,
                           int e0, int e1, bool last, const int32_t* next_pos, cudaStream_t s) {
  const int kk = std::min(top_k, c->L), kt = slots_of(c, top_k);
  if (T == 0) return;
  const int32_t* pos = c->plan_pos[b] + (size_t)(layer - 1) * T * kt;
  const int32_t* off = c->plan_off[b] + (size_t)(layer - 1) * (groups_of(c) + 1);
  const int bn = pick_bn(c, T, kk);
  const int bn_dn = pick_bn_down(c, T, kk);
  const bool pair = use_pair(c, T, kk);
  const int splits = pair ? 1 : pick_splits(c, T, kt, bn_dn);
  prof_rec(c, 1, s);
  if (gather) {
    launch_gather(x, pos, c->d_fault, c->xp, c->cap_rows, T, kt, c->H, s);
    CKLAUNCH();
  }
  prof_rec(c, 2, s);
  prof_rec(c, 3, s);
  GemmParams pg = gemm_params(c, layer, 1, off, 1), pd = gemm_params(c, layer, 2, off, splits);
  const long long split_stride = (long long)T * kt * c->H;
  pd.split_stride = split_stride;
  for (GemmParams* p : {&pg, &pd}) {  // restrict to the window: groups [e0, e1)
    p->offsets += e0;
    p->pt += std::min(e0, c->E);
    p->e_first += e0;
    p->E = e1 - e0;
    p->E_routed = std::max(0, std::min(e1, c->E) - e0);
  }
  // decode-into-GEMM: the window's device-tier groups run in k_moe_gemm_dec, the rest
  // (ring blocks, pinned and shared experts) in k_moe_gemm, which skips the fused groups
  // (one decode-into-GEMM launch per record format present in the window)
  bool fused[2][2] = {{false, false}, {false, false}}, rest[2] = {e1 > c->E, e1 > c->E};  // [kind][fmt]
  if (!pair && c->fused_now) {
    for (int kind = 1; kind <= 2; ++kind)
      for (int e = e0; e < std::min(e1, c->E); ++e) {
        const size_t ti = ((size_t)(layer - 1) * c->E + e) * 2 + (kind - 1);
        if (fused_tensor(c, layer, e, kind)) fused[kind - 1][fmt_of(c, ti)] = true;
        else rest[kind - 1] = true;
      }
    const DecRec* base = c->d_decrec + (size_t)(layer - 1) * 2 * c->E + e0;
    pg.dec = base;
    pd.dec = base + c->E;
    pg.dec_fmt_mask = pd.dec_fmt_mask = fused_fmt_mask(c);
  } else {
    rest[0] = rest[1] = true;
  }
  // gate/up -> down overlap (FX4 windows read wholly in place): the fused down launch starts in
  // the fused gate/up launch's tail and waits per group on the gate/up units' counters
  static const bool overlap_env = !(getenv("XPGB_FUSED_OVERLAP") && atoi(getenv("XPGB_FUSED_OVERLAP")) == 0);
  const bool overlap = overlap_env && !pair && fused[0][1] && !fused[0][0] && !rest[0] && fused[1][1] && !fused[1][0];
  if (overlap) {
    if (!c->d_unit_done) CK(cudaMalloc(&c->d_unit_done, sizeof(int) * (kMaxExperts + 1)));
    CK(cudaMemsetAsync(c->d_unit_done, 0, sizeof(int) * (e1 - e0), s));
    pg.unit_done = pd.unit_done = c->d_unit_done;
  }
  // the same overlap for the regular grouped GEMMs when they carry the whole window
  const bool overlap_reg = overlap_env && !pair && !overlap && rest[0] && rest[1] && !fused[0][0] && !fused[0][1] &&
                           !fused[1][0] && !fused[1][1];
  if (overlap_reg) {
    if (!c->d_unit_done) CK(cudaMalloc(&c->d_unit_done, sizeof(int) * (kMaxExperts + 1)));
    CK(cudaMemsetAsync(c->d_unit_done, 0, sizeof(int) * (e1 - e0), s));
    pg.unit_done = pd.unit_done = c->d_unit_done;
    pg.unit_bn = pd.unit_bn = bn;
  }
  auto fused_launch = [&](bool gate_up, GemmParams& gp, const CUtensorMap& map, int kind) {
    for (int f = 0; f < 2; ++f) {
      if (!fused[kind - 1][f]) continue;
      fz_mark(c, s, fused_bytes(c, layer, e0, e1, kind, f), true);
      launch_gemm_dec(gate_up, map, gp, c->ctab, c->cchunk, pick_bn_dec(c, T, kk), c->num_sms, s, f == 1);
      fz_mark(c, s, 0, false);
    }
  };
  if (pair)
    launch_gemm_pair(true, c->map_xp_pair, c->map_gu, c->S ? c->map_gu_sh : c->map_gu, pg, c->num_sms, s,
                     c->pair_split);
  else {
    fused_launch(true, pg, c->map_xp, 1);
    if (rest[0])
      launch_gate_up(c->map_gu, c->map_xp, c->S ? c->map_gu_sh : c->map_gu, pg, bn, c->num_sms, s, lean_gemm(c));
  }
  CKLAUNCH();
  prof_rec(c, 4, s);
  if (pair)
    launch_gemm_pair(false, c->map_h_pair, c->map_dn, c->S ? c->map_dn_sh : c->map_dn, pd, c->num_sms, s,
                     c->pair_split);
  else {
    fused_launch(false, pd, c->map_h, 2);
    if (rest[1]) {
      if (!overlap_reg) pd.unit_done = nullptr;  // the regular down runs after the fused one (stream order)
      launch_down(c->map_dn, c->map_h, c->S ? c->map_dn_sh : c->map_dn, pd, bn_dn, c->num_sms, s, lean_gemm(c));
    }
  }
  CKLAUNCH();
  prof_rec(c, 5, s);
  if (last) {
    launch_combine(c->part, pos, c->d_fault, y, T, kt, kk, c->H, splits, split_stride,
                   (float)(1.0 / top_k), next_pos, c->xp, c->cap_rows, s);
    CKLAUNCH();
  }
  prof_rec(c, 6, s);
  c->last_splits = splits;
}

static void enqueue_forward(Ctx* c, int layer, const float* x, float* y, int T, int top_k, int b, bool gather,
                            const int32_t* next_pos, cudaStream_t s) {
  enqueue_window(c, layer, x, y, T, top_k, b, gather, 0, groups_of(c), true, next_pos, s);
}

// Standalone layer_forward: plan this layer into buffer 2, then the chain.
static void enqueue_layer(Ctx* c, int layer, const float* x, float* y, int T, int top_k, uint64_t seed,
                          cudaStream_t s) {
  ensure_work(c, T, slots_of(c, top_k));
  if (T == 0) return;
  prof_rec(c, 0, s);
  enqueue_plan(c, 2, layer, 1, T, top_k, seed, s);
  enqueue_forward(c, layer, x, y, T, top_k, 2, true, nullptr, s);
}

// --------------------------------------------------------------------------- page table ops

// A device-tier expert read in place by the decode-into-GEMM kernel is mapped without an arena
// block: its slot-table entry goes LOADING -> RESIDENT in stream order like any page (the GEMM
// prologue's residency check and the ordering log are unchanged), but it holds no ring memory,
// so a window may carry any number of them beside its ring-backed experts.
constexpr int kVirtualBlock = 0x3FFFFFFF;

static int pt_map_virtual(Ctx* c, int layer, int expert, int kind) {
  const int pi = page_index(c, layer, expert, kind);
  const int k = kind - 1;
  if (c->st[k][pi] != XPGB_PAGE_UNMAPPED || c->blk[k][pi] != 0)
    XFAIL(XPGB_ERR_DOUBLE_MAP, "%s is already mapped (%s)", tid_str(layer, expert, kind).c_str(),
          state_name(c->st[k][pi]));
  c->blk[k][pi] = kVirtualBlock;
  c->st[k][pi] = XPGB_PAGE_LOADING;
  c->step += 1;
  emit(c, "map", layer, expert, kind, 0, "in place (device tier, decode-into-GEMM)");
  return kVirtualBlock;
}

// device slot-table block field of a host block id (virtual maps point at block 0: unused)
static int32_t dev_block0(int b) { return b == kVirtualBlock ? 0 : b - 1; }

static int pt_map(Ctx* c, int layer, int expert, int kind) {
  const int pi = page_index(c, layer, expert, kind);
  const int k = kind - 1;
  if (c->st[k][pi] != XPGB_PAGE_UNMAPPED || c->blk[k][pi] != 0)
    XFAIL(XPGB_ERR_DOUBLE_MAP, "%s is already mapped (%s)", tid_str(layer, expert, kind).c_str(),
          state_name(c->st[k][pi]));
  if (c->free_ids[k].empty())
    XFAIL(XPGB_ERR_POOL_EXHAUSTED, "no free kind-%d block for %s; protocol bug", kind,
          tid_str(layer, expert, kind).c_str());
  const int b = *c->free_ids[k].begin();  // lowest id first (paging.py:160-161)
  c->free_ids[k].erase(c->free_ids[k].begin());
  c->blk[k][pi] = b;
  c->owner[k][b] = pi;
  c->st[k][pi] = XPGB_PAGE_LOADING;
  c->bound += sigma_of(c, kind);
  c->peak = std::max(c->peak, c->bound);
  c->step += 1;
  emit(c, "map", layer, expert, kind, b, "");
  return b;
}

static void pt_mark_resident(Ctx* c, int layer, int expert, int kind) {
  const int pi = page_index(c, layer, expert, kind);
  const int k = kind - 1;
  if (c->st[k][pi] != XPGB_PAGE_LOADING)
    XFAIL(XPGB_ERR_NOT_MAPPED, "%s is %s, expected loading", tid_str(layer, expert, kind).c_str(),
          state_name(c->st[k][pi]));
  c->st[k][pi] = XPGB_PAGE_RESIDENT;
  c->step += 1;
  emit(c, "state", layer, expert, kind, c->blk[k][pi], "state=resident");
}

static void pt_unmap(Ctx* c, int layer, int expert, int kind) {
  const int pi = page_index(c, layer, expert, kind);
  const int k = kind - 1;
  const int b = c->blk[k][pi];
  if (b == 0 || (c->st[k][pi] != XPGB_PAGE_RESIDENT && c->st[k][pi] != XPGB_PAGE_EVICTING))
    XFAIL(XPGB_ERR_NOT_MAPPED, "%s is %s; nothing to unmap", tid_str(layer, expert, kind).c_str(),
          state_name(c->st[k][pi]));
  c->st[k][pi] = XPGB_PAGE_EVICTING;
  c->step += 1;
  emit(c, "state", layer, expert, kind, b, "state=evicting");
  c->blk[k][pi] = 0;
  c->st[k][pi] = XPGB_PAGE_UNMAPPED;
  if (b != kVirtualBlock) {
    c->owner[k][b] = -1;
    c->free_ids[k].insert(b);
    c->bound -= sigma_of(c, kind);
  }
  c->step += 1;
  emit(c, "unmap", layer, expert, kind, b, "");
}

// Device table := host table (bulk upload; used after drains and pinning).
static void pt_upload(Ctx* c) {
  const size_t pages = (size_t)c->N * c->E;
  std::vector<int32_t> tab(2 * pages);
  for (int k = 0; k < 2; ++k)
    for (size_t pi = 0; pi < pages; ++pi)
      tab[k * pages + pi] = c->st[k][pi] == XPGB_PAGE_UNMAPPED ? -1 : pt_entry(c->blk[k][pi] - 1, c->st[k][pi]);
  CK(cudaMemcpy(c->d_pt, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
}

static void pt_sync_entry(Ctx* c, int layer, int expert, int kind) {
  const int pi = page_index(c, layer, expert, kind);
  const int k = kind - 1;
  const int32_t v = c->st[k][pi] == XPGB_PAGE_UNMAPPED ? -1 : pt_entry(c->blk[k][pi] - 1, c->st[k][pi]);
  CK(cudaMemcpy(c->d_pt + (size_t)k * c->N * c->E + pi, &v, 4, cudaMemcpyHostToDevice));
}

// StorageHierarchy.fetch (storage.py:228-243): exact bytes into dst on stream.
static uint64_t fetch(Ctx* c, int layer, int expert, int kind, void* dst, uint64_t dst_bytes, cudaStream_t s,
                      bool* from_host) {
  const int pi = page_index(c, layer, expert, kind);
  const uint64_t sz = sigma_of(c, kind);
  if (dst_bytes != sz)
    XFAIL(XPGB_ERR_BACKEND_MISS, "%s: fetched %llu bytes into a %llu-byte block",
          tid_str(layer, expert, kind).c_str(), (unsigned long long)sz, (unsigned long long)dst_bytes);
  const uint64_t within = (kind == 2) ? c->s1 : 0;
  const size_t ti = (size_t)pi * 2 + (kind - 1);
  if (c->backend[ti] == 1) {
    if (c->dev_off[ti] < 0) XFAIL(XPGB_ERR_BACKEND_MISS, "%s is not staged on the device tier",
                                  tid_str(layer, expert, kind).c_str());
    CK(cudaMemcpyAsync(dst, c->dev_tier + c->dev_off[ti], sz, cudaMemcpyDeviceToDevice, s));
    if (from_host) *from_host = false;
  } else {
    if (!c->host) XFAIL(XPGB_ERR_BACKEND_MISS, "%s: no host pool attached", tid_str(layer, expert, kind).c_str());
    const uint64_t off = (uint64_t)pi * (c->s1 + c->s2) + within;
    CK(cudaMemcpyAsync(dst, c->host + off, sz, cudaMemcpyHostToDevice, s));
    if (from_host) *from_host = true;
  }
  return sz;
}

// --------------------------------------------------------------------------- run (StreamedRunner)

struct RunState {
  Ctx* c;
  const xpgb_run_opts* o;
  float* acts;
  long long h2d = 0, d2d = 0;
  bool log;
  long long decoded = 0;
};

static void set_rec(PtOp& op, int idx, int ev, int it, int layer, int kind, int tit, int tl, int group = 0) {
  op.rec[idx][6] = group;
  op.rec[idx][0] = ev;
  op.rec[idx][1] = it;
  op.rec[idx][2] = layer;
  op.rec[idx][3] = kind;
  op.rec[idx][4] = tit;
  op.rec[idx][5] = tl;
  op.n_rec = idx + 1;
}

static PtOp blank_op(Ctx* c, bool log) {
  PtOp op;
  memset(&op, 0, sizeof(op));
  if (log) {
    op.log = c->d_log;
    op.log_count = c->d_log_count;
    op.log_cap = c->log_cap;
  }
  return op;
}

static void launch_op(const PtOp& op, cudaStream_t s) {
  k_pt_op<<<1, 128, 0, s>>>(op);
  note_launch();
  CKLAUNCH();
}

static void log_only(Ctx* c, bool log, cudaStream_t s, int ev, int it, int layer, int group = 0) {
  if (!log) return;
  PtOp op = blank_op(c, true);
  set_rec(op, 0, ev, it, layer, -1, -1, -1, group);
  launch_op(op, s);
}

// One step of the schedule: a layer, or -- with a sub-layer ring -- one window of it.
// The window [e0, e1) of local expert groups holds exactly the step's streamed experts
// (plus any pinned ones between them); the layer's last window also covers its shared
// experts [E, E+S).  Reference geometry: one window [0, E+S) per layer.
struct Step {
  int it, layer, w, e0, e1;
  bool first, last;
};

// Alg. 1 MaterializeLayer (pipeline.py:335-360) for one kind, enqueued on copy stream `kind`:
// recycle the blocks of step g-2 (the reference's target_layer, paging.py:29-38, once the
// steps are layers) after its compute event, map + load this step's streamed experts.
// opts.profile: bracket one decoder launch with events on its stream
static void dec_mark(RunState& rs, cudaStream_t s, uint64_t bytes, bool begin) {
  Ctx* c = rs.c;
  if (!rs.o->profile) return;
  if (begin) {
    c->dec_skip = (c->dec_seen++ % (size_t)c->prof_every) != 0;
    if (c->dec_skip) return;
    while (c->dec_ev.size() < 2 * (c->dec_n + 1)) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->dec_ev.push_back(e);
    }
    if (c->dec_bytes.size() < c->dec_n + 1) c->dec_bytes.resize(c->dec_n + 1);
    c->dec_bytes[c->dec_n] = bytes;
    CK(cudaEventRecord(c->dec_ev[2 * c->dec_n], s));
  } else {
    if (c->dec_skip) return;
    CK(cudaEventRecord(c->dec_ev[2 * c->dec_n + 1], s));
    ++c->dec_n;
  }
}

// windows in flight: the sub-layer ring's depth, else the reference's two layers
static int depth_of(const Ctx* c) { return c->ring_limit > 0 ? c->ring_depth : 2; }

static void materialize(RunState& rs, int g, const Step& st, const Step* tg, int kind) {
  Ctx* c = rs.c;
  const int N = c->N, E = c->E, k = kind - 1;
  const int it = st.it, layer = st.layer;
  const int wlo = st.e0, whi = std::min(st.e1, E);
  cudaStream_t s = c->s_copy[k];
  const bool seq = rs.o->sequential != 0;
  PtOp op = blank_op(c, rs.log);
  int nrec = 0;
  const bool any_pinned = std::find(c->pinned.begin(), c->pinned.end(), 1) != c->pinned.end();
  auto is_pinned = [&](int l, int e) { return c->pinned[(size_t)(l - 1) * E + e] != 0; };
  const int chunk = (int)(sizeof(op.vals) / sizeof(int32_t));
  if (tg) {
    const int tgt = tg->layer, tlo = tg->e0, thi = std::min(tg->e1, E);
    const bool skip_war = c->war_sab_it == it && c->war_sab_layer == layer;  // hazard test only
    if (!skip_war) CK(cudaStreamWaitEvent(s, c->ev_comp[(g - depth_of(c)) % kEvRing], 0));  // WAR
    for (int e = tlo; e < thi; ++e)
      if (!is_pinned(tgt, e)) pt_unmap(c, tgt, c->e_first + e + 1, kind);
    if (rs.log) set_rec(op, nrec++, XPGB_EV_RECYCLE, it, layer, kind, tg->it, tgt, st.w | (tg->w << 16));
    int32_t* trow = c->d_pt + (size_t)k * N * E + (size_t)(tgt - 1) * E;
    if (!any_pinned) {
      op.unmap_row = trow + tlo;
      op.unmap_n = thi - tlo;
    } else {
      // keep the pinned entries of the recycled window: rewrite its range explicitly
      for (int e0 = tlo; e0 < thi; e0 += chunk) {
        PtOp ou = (e0 == tlo) ? op : blank_op(c, false);
        if (e0 > tlo) ou.n_rec = 0;
        ou.set_row = trow + e0;
        ou.set_n = std::min(chunk, thi - e0);
        for (int i = 0; i < ou.set_n; ++i) {
          const size_t pi = (size_t)(tgt - 1) * E + e0 + i;
          ou.vals[i] = c->st[k][pi] == XPGB_PAGE_UNMAPPED ? -1 : pt_entry(dev_block0(c->blk[k][pi]), c->st[k][pi]);
        }
        launch_op(ou, s);
      }
      op = blank_op(c, rs.log);
      nrec = 0;
    }
  }
  const float* delays = rs.o->fetch_delay_s;
  auto delay_of = [&](int e) -> float {
    return delays ? delays[((size_t)(layer - 1) * c->L + (c->e_first + e)) * 2 + k] : 0.f;
  };
  // a window whose streamed experts are all read in place (or pinned) has nothing to load: one
  // slot-table launch takes it straight to RESIDENT (its LOAD_START and LOAD_DONE records in
  // order inside it) instead of a LOADING launch and a RESIDENT launch on the decode stream
  bool no_load = whi > wlo && whi - wlo <= chunk;
  for (int e = wlo; e < whi && no_load; ++e)
    no_load = is_pinned(layer, e) || (fused_tensor(c, layer, e, kind) && delay_of(e) <= 0.f);
  // map every streamed expert of the window (lowest free block first) -> LOADING entries
  std::vector<int> blocks(E, 0);
  for (int e = wlo; e < whi; ++e)
    blocks[e] = is_pinned(layer, e)              ? c->blk[k][(size_t)(layer - 1) * E + e]
                : fused_tensor(c, layer, e, kind) ? pt_map_virtual(c, layer, c->e_first + e + 1, kind)
                                                  : pt_map(c, layer, c->e_first + e + 1, kind);
  if (rs.log) set_rec(op, nrec++, XPGB_EV_LOAD_START, it, layer, kind, -1, -1, st.w);
  int32_t* row = c->d_pt + (size_t)k * N * E + (size_t)(layer - 1) * E;
  for (int e0 = wlo; e0 < whi; e0 += chunk) {
    PtOp o2 = (e0 == wlo) ? op : blank_op(c, false);
    if (e0 > wlo) { o2.unmap_n = 0; o2.n_rec = 0; }
    o2.set_row = row + e0;
    o2.set_n = std::min(chunk, whi - e0);
    for (int i = 0; i < o2.set_n; ++i)
      o2.vals[i] = pt_entry(dev_block0(blocks[e0 + i]),
                            (no_load || is_pinned(layer, e0 + i)) ? XPGB_PAGE_RESIDENT : XPGB_PAGE_LOADING);
    if (no_load && rs.log) set_rec(o2, nrec++, XPGB_EV_LOAD_DONE, it, layer, kind, -1, -1, st.w);
    launch_op(o2, s);
  }
  if (no_load) {
    for (int e = wlo; e < whi; ++e)
      if (!is_pinned(layer, e)) pt_mark_resident(c, layer, c->e_first + e + 1, kind);
    CK(cudaEventRecord(c->ev_load[k][g % kEvRing], s));
    if (seq) CK(cudaStreamSynchronize(s));
    return;
  }
  if (whi <= wlo && (op.n_rec > 0 || op.unmap_n > 0)) launch_op(op, s);  // window without routed experts
  static const bool env_poison = getenv("XPGB_POISON") && atoi(getenv("XPGB_POISON")) != 0;
  if (c->poison || env_poison)
    for (int e = wlo; e < whi; ++e)
      if (!is_pinned(layer, e) && blocks[e] != kVirtualBlock)
        CK(cudaMemsetAsync(block_ptr(c, kind, blocks[e]), 0xFF, sigma_of(c, kind), s));
  auto sleep_on = [&](cudaStream_t st, float d) {
    k_sleep<<<1, 1, 0, st>>>((uint64_t)(d * 1e9));
    note_launch();
    CKLAUNCH();
  };
  cudaStream_t done_stream = s;
  if (!c->codec) {
    for (int e = wlo; e < whi; ++e) {
      if (is_pinned(layer, e)) continue;
      if (delay_of(e) > 0) sleep_on(s, delay_of(e));
      bool from_host = true;
      const uint64_t n = fetch(c, layer, c->e_first + e + 1, kind, block_ptr(c, kind, blocks[e]), sigma_of(c, kind), s,
                               &from_host);
      (from_host ? rs.h2d : rs.d2d) += n;
    }
  } else {
    // compressed tiers: records reach a decode stream (copied over PCIe into a staging
    // buffer for the host tier, read in place for the device tier) and are expanded
    // straight into the ring block; staging is double-buffered so the link never waits.
    // host-tier records decode on d behind their copies; device-tier records decode on dv,
    // which only waits for the window's mapping, so they run while the link is busy
    cudaStream_t d = c->s_dec[k], dv = c->s_devdec[k];
    CK(cudaEventRecord(c->ev_mapped[k], s));
    CK(cudaStreamWaitEvent(d, c->ev_mapped[k], 0));
    bool dev_on_dv = false;
    bool raw_on_s = false;
    const uint64_t n = sigma_of(c, kind) / 2;
    const uint64_t sm16 = (n + 15) & ~15ull;
    auto tix = [&](int e) { return ((size_t)(layer - 1) * E + e) * 2 + k; };
    auto rec_bytes = [&](int e) { return xpgb_codec_record_bytes(n, c->rec_bits[tix(e)], c->cchunk); };
    // decoder's algorithmic bytes for one whole tensor: sign/mantissa + bitstream + chunk index read, bf16 written
    auto algo_bytes = [&](size_t t) { return n + c->rec_bits[t] + (n + c->cchunk - 1) / c->cchunk * 4 + 2 * n; };
    // a staged run may take expert e' after e when its record follows e's in the pool
    auto joins_run = [&](int e, int e2, int tier) {
      return e2 < whi && !is_pinned(layer, e2) && c->backend[tix(e2)] == tier && delay_of(e2) <= 0.f &&
             !(tier == 1 && fmt_of(c, tix(e2)) != 0) && !fused_tensor(c, layer, e2, kind) &&
             (tier == 1 || c->rec_off[tix(e2)] == c->rec_off[tix(e)] + rec_bytes(e));
    };
    DecodeTensor dt[kMaxDecodeTensors];
    for (int e = wlo; e < whi;) {
      if (is_pinned(layer, e)) { ++e; continue; }
      if (fused_tensor(c, layer, e, kind)) {  // read in place by the GEMM: nothing to expand
        if (delay_of(e) > 0) sleep_on(d, delay_of(e));  // an injected fetch delay still holds the load
        ++e;
        continue;
      }
      const size_t ti = tix(e);
      uint8_t* dst = block_ptr(c, kind, blocks[e]);
      const float dl = delay_of(e);
      if (c->backend[ti] == 1 && fmt_of(c, ti) == 1) {
        // FX4 device tier, expanded into the ring (groups the fused GEMM does not take)
        if (!dev_on_dv) CK(cudaStreamWaitEvent(dv, c->ev_mapped[k], 0));
        dev_on_dv = true;
        if (dl > 0) sleep_on(dv, dl);
        dec_mark(rs, dv, c->fx_bytes[ti] + 2 * n, true);
        launch_fx4_decode(c->dev_tier + c->dev_off[ti], n, c->fx_base[ti], reinterpret_cast<uint16_t*>(dst), dv);
        CKLAUNCH();
        dec_mark(rs, dv, 0, false);
        rs.decoded += 2 * n;
        ++e;
      } else if (c->backend[ti] == 1) {
        // device tier: consecutive device-tier experts of the layer decode in one launch
        if (!dev_on_dv) CK(cudaStreamWaitEvent(dv, c->ev_mapped[k], 0));
        dev_on_dv = true;
        if (dl > 0) sleep_on(dv, dl);
        int cnt = 0;
        for (int e2 = e;; ++e2) {
          const size_t t2 = tix(e2);
          const uint8_t* rec = c->dev_tier + c->dev_off[t2];
          const uint64_t bits16 = (c->rec_bits[t2] + 8 + 15) & ~15ull;
          dt[cnt++] = DecodeTensor{rec, reinterpret_cast<const uint32_t*>(rec + sm16),
                                   reinterpret_cast<const uint32_t*>(rec + sm16 + bits16),
                                   reinterpret_cast<uint16_t*>(block_ptr(c, kind, blocks[e2])), 0u};
          if (cnt == kMaxDecodeTensors || !joins_run(e2, e2 + 1, 1)) break;
        }
        uint64_t ab = 0;
        for (int i = 0; i < cnt; ++i) ab += algo_bytes(tix(e + i));
        dec_mark(rs, dv, ab, true);
        launch_exp_decode_multi(dt, cnt, n, c->cchunk, c->ctab, dv);
        CKLAUNCH();
        dec_mark(rs, dv, 0, false);
        rs.decoded += 2 * n * cnt;
        e += cnt;
      } else if (c->host_codec && rec_bytes(e) <= c->stage_cap[k]) {
        // host tier, small records: a run of whole consecutive records in ONE copy and
        // ONE decode launch (per-copy turnaround would otherwise dominate small experts)
        uint64_t run = rec_bytes(e);
        int cnt = 1;
        while (cnt < kMaxDecodeTensors && joins_run(e + cnt - 1, e + cnt, 0) && run + rec_bytes(e + cnt) <= c->stage_cap[k]) {
          run += rec_bytes(e + cnt);
          ++cnt;
        }
        const uint64_t base = c->rec_off[ti];
        const int lastx = e + cnt - 1;
        // the last record's trailing chunk index stays home (it is device-resident)
        const uint64_t bytes = c->rec_off[tix(lastx)] - base + sm16 + ((c->rec_bits[tix(lastx)] + 8 + 15) & ~15ull);
        const int buf = (int)(c->stage_next[k]++ % (uint32_t)c->n_stage);
        uint8_t* st = c->stage[k][buf];
        cudaStream_t cs = (buf & 1) ? c->s_alt[k] : c->s_cp[k];
        CK(cudaStreamWaitEvent(cs, c->ev_decoded[k][buf], 0));
        if (dl > 0) sleep_on(cs, dl);  // the injected fetch delay holds this record's copy
        CK(cudaMemcpyAsync(st, c->cpool + base, bytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(c->ev_copied[k][buf], cs));
        rs.h2d += bytes;
        CK(cudaStreamWaitEvent(d, c->ev_copied[k][buf], 0));
        for (int i = 0; i < cnt; ++i) {
          const size_t t2 = tix(e + i);
          uint8_t* rec = st + (c->rec_off[t2] - base);
          dt[i] = DecodeTensor{rec, reinterpret_cast<const uint32_t*>(rec + sm16), c->d_index + c->d_index_off[t2],
                               reinterpret_cast<uint16_t*>(block_ptr(c, kind, blocks[e + i])), 0u};
        }
        uint64_t ab = 0;
        for (int i = 0; i < cnt; ++i) ab += algo_bytes(tix(e + i));
        dec_mark(rs, d, ab, true);
        launch_exp_decode_multi(dt, cnt, n, c->cchunk, c->ctab, d);
        CKLAUNCH();
        dec_mark(rs, d, 0, false);
        CK(cudaEventRecord(c->ev_decoded[k][buf], d));
        rs.decoded += 2 * n * cnt;
        e += cnt;
      } else if (c->host_codec) {
        // stream the record in pieces of whole chunks (<= kStagePieceBytes) so the staging
        // buffers stay small: sm slice | stream slice (+8 B lookahead) | index slice
        const uint64_t nb = c->rec_bits[ti];
        const uint64_t ch = (uint64_t)c->cchunk;
        const uint64_t nc = (n + ch - 1) / ch;
        const uint64_t bits16 = (nb + 8 + 15) & ~15ull;
        const uint8_t* rec = c->cpool + c->rec_off[ti];
        const uint32_t* idx = reinterpret_cast<const uint32_t*>(rec + sm16 + bits16);
        auto piece_bytes = [&](uint64_t a, uint64_t b) -> uint64_t {  // staged size of chunks [a, b)
          const uint64_t va = a * ch, vb = std::min(n, b * ch);
          const uint64_t ba = ((uint64_t)idx[a] >> 5) * 4, bb = (b < nc) ? (((uint64_t)idx[b] + 7) / 8) : nb;
          return ((vb - va + 15) & ~15ull) + ((bb - ba + 8 + 15) & ~15ull);
        };
        for (uint64_t c0 = 0, c1 = 0; c0 < nc; c0 = c1) {
          // largest c1 whose piece fits the staging buffer (sizes grow with c1)
          uint64_t lo = c0 + 1, hi = nc;
          while (lo < hi) {
            const uint64_t mid = (lo + hi + 1) / 2;
            if (piece_bytes(c0, mid) <= c->stage_cap[k]) lo = mid; else hi = mid - 1;
          }
          c1 = lo;
          const uint64_t v0 = c0 * ch, v1 = std::min(n, c1 * ch);
          const uint64_t b0 = ((uint64_t)idx[c0] >> 5) * 4;
          const uint64_t b1 = (c1 < nc) ? (((uint64_t)idx[c1] + 7) / 8) : nb;
          const uint64_t ns = v1 - v0, nbits = b1 - b0 + 8;
          const uint64_t o_bits = (ns + 15) & ~15ull;
          if (o_bits + nbits > c->stage_cap[k]) XFAIL(XPGB_ERR, "codec piece exceeds staging buffer");
          const int buf = (int)(c->stage_next[k]++ % (uint32_t)c->n_stage);
          uint8_t* st = c->stage[k][buf];
          // odd and even buffers fill from their own copy streams, so one stream's
          // wait/turnaround bubble hides behind the other's transfer
          cudaStream_t cs = (buf & 1) ? c->s_alt[k] : c->s_cp[k];
          CK(cudaStreamWaitEvent(cs, c->ev_decoded[k][buf], 0));
          if (dl > 0 && c0 == 0) sleep_on(cs, dl);
          CK(cudaMemcpyAsync(st, rec + v0, ns, cudaMemcpyHostToDevice, cs));
          CK(cudaMemcpyAsync(st + o_bits, rec + sm16 + b0, nbits, cudaMemcpyHostToDevice, cs));
          CK(cudaEventRecord(c->ev_copied[k][buf], cs));
          rs.h2d += ns + nbits;
          CK(cudaStreamWaitEvent(d, c->ev_copied[k][buf], 0));
          dec_mark(rs, d, ns + (b1 - b0) + (c1 - c0) * 4 + 2 * ns, true);
          launch_exp_decode(st, reinterpret_cast<const uint32_t*>(st + o_bits), c->d_index + c->d_index_off[ti] + c0,
                            ns, c->cchunk, c->ctab, reinterpret_cast<uint16_t*>(dst) + v0, d, (uint32_t)(b0 * 8));
          CKLAUNCH();
          dec_mark(rs, d, 0, false);
          CK(cudaEventRecord(c->ev_decoded[k][buf], d));
        }
        rs.decoded += 2 * n;
        ++e;
      } else {
        if (dl > 0) sleep_on(s, dl);
        bool from_host = true;
        rs.h2d += fetch(c, layer, c->e_first + e + 1, kind, dst, sigma_of(c, kind), s, &from_host);
        raw_on_s = true;
        ++e;
      }
    }
    if (raw_on_s) {
      CK(cudaEventRecord(c->ev_raw[k], s));
      CK(cudaStreamWaitEvent(d, c->ev_raw[k], 0));
    }
    if (dev_on_dv) {
      CK(cudaEventRecord(c->ev_devdec[k], dv));
      CK(cudaStreamWaitEvent(d, c->ev_devdec[k], 0));
    }
    done_stream = d;
  }
  for (int e = wlo; e < whi; ++e)
    if (!is_pinned(layer, e)) pt_mark_resident(c, layer, c->e_first + e + 1, kind);
  for (int e0 = wlo; e0 < std::max(whi, wlo + 1); e0 += chunk) {
    PtOp o3 = blank_op(c, rs.log && e0 + chunk >= whi);
    o3.set_row = row + e0;
    o3.set_n = std::max(0, std::min(chunk, whi - e0));
    for (int i = 0; i < o3.set_n; ++i) o3.vals[i] = pt_entry(dev_block0(blocks[e0 + i]), XPGB_PAGE_RESIDENT);
    if (o3.log) set_rec(o3, 0, XPGB_EV_LOAD_DONE, it, layer, kind, -1, -1, st.w);
    launch_op(o3, done_stream);
  }
  CK(cudaEventRecord(c->ev_load[k][g % kEvRing], done_stream));
  if (seq) {
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(done_stream));
  }
}

// ---- session: the StreamedRunner schedule, one step at a time --------------------

struct Session {
  bool active = false;
  xpgb_run_opts o{};
  std::vector<float> fetch_delay, compute_delay;
  RunState rs{};
  int steps = 0;
  bool paged = false;
  std::vector<Step> sv;  // the flattened schedule: iterations x layers x windows
  int mat_next = 0;      // next step to materialize
  bool builtin_compute = false;  // session_compute ran (its per-launch profile events exist)
};

static Session& session_of(Ctx* c) {
  if (!c->sess) c->sess = new Session();
  return *c->sess;
}

// Windows of one layer for the current ring: each holds ring_blocks/depth streamed experts
// (depth windows in flight: double-buffered halves of the ring by default); one window per
// layer when the ring holds two whole layers (the reference geometry).
static std::vector<std::pair<int, int>> layer_windows(Ctx* c, int layer) {
  const int E = c->E, G = groups_of(c);
  // experts that need a ring block: streamed and not read in place by the decode-into-GEMM kernel
  auto ring_backed = [&](int e) {
    return !c->pinned[(size_t)(layer - 1) * E + e] && !(fused_tensor(c, layer, e, 1) && fused_tensor(c, layer, e, 2));
  };
  int streamed = 0;
  for (int e = 0; e < E; ++e) streamed += ring_backed(e);
  const int gs = std::max(1, c->ring_blocks / depth_of(c));
  std::vector<std::pair<int, int>> w;
  if (c->pool != XPGB_POOL_RING || gs >= streamed) {
    w.push_back({0, G});
    return w;
  }
  int lo = 0, n = 0;
  for (int e = 0; e < E; ++e) {
    n += ring_backed(e);
    if (n == gs) {
      w.push_back({lo, e + 1});
      lo = e + 1;
      n = 0;
    }
  }
  if (lo < E) w.push_back({lo, E});
  w.back().second = G;  // the last window also computes the shared experts
  return w;
}

static void build_schedule(Ctx* c, Session& ss, int iterations) {
  ss.sv.clear();
  std::vector<std::vector<std::pair<int, int>>> per_layer;
  for (int l = 1; l <= c->N; ++l) per_layer.push_back(layer_windows(c, l));
  for (int it = 1; it <= iterations; ++it)
    for (int l = 1; l <= c->N; ++l) {
      const auto& w = per_layer[l - 1];
      for (int i = 0; i < (int)w.size(); ++i)
        ss.sv.push_back(Step{it, l, i, w[i].first, w[i].second, i == 0, i + 1 == (int)w.size()});
    }
  ss.steps = (int)ss.sv.size();
}


// Begin a run: empty ring, fresh log, RUN_BEGIN on the compute stream; copy streams
// start after it.  `acts` (device fp32 [T][H]) is the buffer the built-in compute
// updates in place; external-compute sessions pass nullptr.
static void session_begin(Ctx* c, const xpgb_run_opts* o, float* acts) {
  Session& ss = session_of(c);
  if (ss.active) XFAIL(XPGB_ERR, "a session is already active on this context");
  if (o->iterations < 1) XFAIL(XPGB_ERR, "need at least one iteration");
  if (o->tokens < 0 || o->top_k < 1)
    XFAIL(XPGB_ERR_OUT_OF_RANGE, "bad ForwardSpec (T=%d, top_k=%d)", o->tokens, o->top_k);
  const int N = c->N;
  ss.o = *o;
  c->fused_now = fused_for(c, o->tokens, o->top_k);  // the schedule's windows depend on it
  build_schedule(c, ss, o->iterations);
  ss.mat_next = 0;
  ss.builtin_compute = false;
  c->dec_n = 0;
  c->fz_n = 0;
  c->dec_seen = c->fz_seen = 0;
  c->prof_mode = o->profile;
  c->prof_every = o->profile >= 2 ? o->profile : 1;
  ss.fetch_delay.clear();
  ss.compute_delay.clear();
  if (o->fetch_delay_s) ss.fetch_delay.assign(o->fetch_delay_s, o->fetch_delay_s + (size_t)N * c->L * 2);
  if (o->compute_delay_s)
    ss.compute_delay.assign(o->compute_delay_s, o->compute_delay_s + (size_t)o->iterations * N);
  ss.o.fetch_delay_s = ss.fetch_delay.empty() ? nullptr : ss.fetch_delay.data();
  ss.o.compute_delay_s = ss.compute_delay.empty() ? nullptr : ss.compute_delay.data();
  ensure_work(c, o->tokens, slots_of(c, o->top_k));
  ensure_log(c, ss.steps * 8 + 16);
  if (o->profile) {
    while (c->run_ev.size() < (size_t)ss.steps * 7) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->run_ev.push_back(e);
    }
  }
  CK(cudaMemset(c->d_fault, 0, sizeof(long long)));
  ss.paged = c->pool == XPGB_POOL_RING;
  if (ss.paged) {
    // a run starts from an empty ring, like a fresh PageTable (pipeline.py:325)
    for (int k = 0; k < 2; ++k)
      for (size_t pi = 0; pi < c->st[k].size(); ++pi)
        if (c->st[k][pi] != XPGB_PAGE_UNMAPPED && !c->pinned[pi])
          XFAIL(XPGB_ERR_DOUBLE_MAP, "run() needs an empty page table; page %zu kind %d is mapped", pi, k + 1);
    c->peak = c->bound;  // pinned pages stay bound
  }
  ss.rs = RunState{c, &ss.o, acts, 0, 0, o->log_enable != 0};
  c->fused_now = fused_for(c, o->tokens, o->top_k);
  cudaStream_t s = c->s_comp;
  CK(cudaDeviceSynchronize());  // inputs written by other streams are complete
  log_only(c, ss.rs.log, s, XPGB_EV_RUN_BEGIN, 0, 0);
  CK(cudaEventRecord(c->ev_begin, s));
  CK(cudaStreamWaitEvent(c->s_copy[0], c->ev_begin, 0));
  CK(cudaStreamWaitEvent(c->s_copy[1], c->ev_begin, 0));
  if (o->sequential) CK(cudaStreamSynchronize(s));
  ss.active = true;
}

// Callers follow the reference's order -- mat(0), mat(1), then mat(g+2) right after
// release(g).  With a deeper ring (depth D windows in flight) the call for g+2 enqueues
// every step up to g+D: step j recycles step j-D, released by then.
static void session_materialize(Ctx* c, int g) {
  Session& ss = session_of(c);
  if (!ss.active) XFAIL(XPGB_ERR, "no active session");
  if (!ss.paged || g < 0) return;
  const int D = depth_of(c);
  const int upto = std::min(ss.steps - 1, g + D - 2);
  for (int j = std::max(ss.mat_next, 0); j <= upto; ++j) {
    const Step* tg = j >= D ? &ss.sv[j - D] : nullptr;  // cold start: the first D steps recycle nothing
    for (int kind = 1; kind <= 2; ++kind) materialize(ss.rs, j, ss.sv[j], tg, kind);
    ss.mat_next = j + 1;
  }
}

// RAW: `s` waits for both load events of step g, then compute-start is logged on it.
static void session_acquire(Ctx* c, int g, cudaStream_t s) {
  Session& ss = session_of(c);
  if (!ss.active) XFAIL(XPGB_ERR, "no active session");
  const Step& st = ss.sv[g];
  const xpgb_run_opts* o = &ss.o;
  const bool skip = (o->sabotage_iteration == st.it && o->sabotage_layer == st.layer);
  if (ss.paged && !skip) {
    CK(cudaStreamWaitEvent(s, c->ev_load[0][g % kEvRing], 0));
    CK(cudaStreamWaitEvent(s, c->ev_load[1][g % kEvRing], 0));
  }
  log_only(c, ss.rs.log, s, XPGB_EV_COMPUTE_START, st.it, st.layer, st.w);
  if (o->compute_delay_s && st.first) {
    const float d = o->compute_delay_s[(size_t)(st.it - 1) * c->N + (st.layer - 1)];
    if (d > 0) {
      k_sleep<<<1, 1, 0, s>>>((uint64_t)(d * 1e9));
      note_launch();
      CKLAUNCH();
    }
  }
}

// compute-done on `s` and the WAR event the loaders of step g+2 wait on.
static void session_release(Ctx* c, int g, cudaStream_t s) {
  Session& ss = session_of(c);
  if (!ss.active) XFAIL(XPGB_ERR, "no active session");
  const Step& st = ss.sv[g];
  log_only(c, ss.rs.log, s, XPGB_EV_COMPUTE_DONE, st.it, st.layer, st.w);
  CK(cudaEventRecord(c->ev_comp[g % kEvRing], s));
  if (ss.o.sequential) CK(cudaStreamSynchronize(s));
}

// Built-in compute of step g (single-GPU layer_forward chain) on the compute stream:
// the window's expert GEMMs; the layer's combine after its last window.
static void session_compute(Ctx* c, int g) {
  Session& ss = session_of(c);
  ss.builtin_compute = true;
  const xpgb_run_opts* o = &ss.o;
  const Step& st = ss.sv[g];
  const int it = st.it, layer = st.layer;
  cudaStream_t s = c->s_comp;
  const int kt = slots_of(c, o->top_k);
  const int T = o->tokens;
  c->cur_ev = (o->profile == 1 && T > 0) ? &c->run_ev[(size_t)g * 7] : nullptr;
  prof_rec(c, 0, s);
  if (layer == 1 && st.first && T > 0) {
    // one route+plan launch per decode step covers all N layers; plans alternate between
    // buffers 0/1 so the next step's plan never overwrites rows still in use
    if (it == 1) enqueue_plan(c, 0, 1, c->N, T, o->top_k, o->router_seed, s);
    if (it < o->iterations) enqueue_plan(c, it & 1, 1, c->N, T, o->top_k, o->router_seed, s);
  }
  const int b = (it - 1) & 1;
  const bool last = (g + 1 == ss.steps);
  const bool fresh = o->fresh_inputs != 0;  // each iteration gathers its own new inputs
  const int32_t* next_pos = nullptr;
  if (!last && T > 0) {
    if (layer < c->N) next_pos = c->plan_pos[b] + (size_t)layer * T * kt;
    else if (!fresh) next_pos = c->plan_pos[it & 1];
  }
  const bool gather = g == 0 || (fresh && layer == 1 && st.first);
  enqueue_window(c, layer, ss.rs.acts, ss.rs.acts, T, o->top_k, b, gather, st.e0, st.e1, st.last, next_pos, s);
  c->cur_ev = nullptr;
}

static void session_end(Ctx* c, xpgb_report* rep) {
  Session& ss = session_of(c);
  if (!ss.active) XFAIL(XPGB_ERR, "no active session");
  ss.active = false;
  c->fused_now = false;
  const xpgb_run_opts* o = &ss.o;
  RunState& rs = ss.rs;
  const int N = c->N;
  const int steps = ss.steps;
  const int kk = std::min(o->top_k, c->L), kt = slots_of(c, o->top_k);
  const bool paged = ss.paged;
  cudaStream_t s = c->s_comp;
  CK(cudaEventRecord(c->ev_end, s));
  CK(cudaDeviceSynchronize());

  // collect the log
  int32_t n = 0;
  CK(cudaMemcpy(&n, c->d_log_count, 4, cudaMemcpyDeviceToHost));
  n = std::min(n, c->log_cap);
  c->last_log.resize(n);
  if (n) CK(cudaMemcpy(c->last_log.data(), c->d_log, (size_t)n * sizeof(xpgb_record), cudaMemcpyDeviceToHost));
  std::sort(c->last_log.begin(), c->last_log.end(),
            [](const xpgb_record& a, const xpgb_record& b) { return a.t < b.t; });

  memset(rep, 0, sizeof(*rep));
  // stall = compute stream idle before each compute-start (since the previous
  // compute-done / run begin); war wait = copy stream idle before each recycle.
  int64_t prev_comp = -1, prev_copy[2] = {-1, -1}, load_start[2] = {0, 0};
  int64_t first = 0, last = 0;
  for (size_t i = 0; i < c->last_log.size(); ++i) {
    const xpgb_record& r = c->last_log[i];
    if (i == 0) first = r.wall_ns;
    last = std::max<int64_t>(last, r.wall_ns);
    switch (r.event) {
      case XPGB_EV_RUN_BEGIN:
        prev_comp = r.wall_ns;
        prev_copy[0] = prev_copy[1] = r.wall_ns;
        break;
      case XPGB_EV_COMPUTE_START:
        if (prev_comp >= 0) rep->stall_ns += std::max<int64_t>(0, r.wall_ns - prev_comp);
        break;
      case XPGB_EV_COMPUTE_DONE: prev_comp = r.wall_ns; break;
      case XPGB_EV_RECYCLE:
        if (r.kind >= 1 && prev_copy[r.kind - 1] >= 0)
          rep->war_wait_ns += std::max<int64_t>(0, r.wall_ns - prev_copy[r.kind - 1]);
        break;
      case XPGB_EV_LOAD_START:
        if (r.kind >= 1) load_start[r.kind - 1] = r.wall_ns;
        break;
      case XPGB_EV_LOAD_DONE:
        if (r.kind >= 1) {
          rep->copy_busy_ns[r.kind - 1] += r.wall_ns - load_start[r.kind - 1];
          prev_copy[r.kind - 1] = r.wall_ns;
        }
        break;
    }
  }
  rep->elapsed_ns = last - first;
  rep->arena_peak_bytes = (int64_t)c->peak;
  rep->h2d_bytes = rs.h2d;
  rep->d2d_bytes = rs.d2d;
  rep->decoded_bytes = rs.decoded;
  rep->n_records = (int32_t)c->last_log.size();
  long long fw = 0;
  CK(cudaMemcpy(&fw, c->d_fault, sizeof(fw), cudaMemcpyDeviceToHost));
  rep->page_fault = fw != 0;

  // active groups and local rows per layer (routing is iteration-invariant) -> algorithmic bytes
  if (o->tokens > 0 && rs.acts) {
    const int G = groups_of(c);
    std::vector<int32_t> of((size_t)N * (G + 1));
    CK(cudaMemcpy(of.data(), c->plan_off[0], of.size() * 4, cudaMemcpyDeviceToHost));
    long long active = 0, rows = 0;
    for (int l = 0; l < N; ++l) {
      const int32_t* o2 = of.data() + (size_t)l * (G + 1);
      for (int e = 0; e < G; ++e) active += o2[e + 1] > o2[e];
      rows += o2[G];
    }
    (void)kk;
    (void)kt;
    rep->active_experts = (int32_t)active;
    rep->down_splits = c->last_splits;
    const double a = (double)active / N, r = (double)rows / N;
    rep->gate_up_bytes = (long long)(a * c->s1 + r * c->H * 2 + r * c->F * 2);
    rep->down_bytes = (long long)(a * c->s2 + r * c->F * 2 + r * (double)c->H * 4 * std::max(1, rep->down_splits));
  }
  if (o->profile == 1 && ss.builtin_compute && steps > 0 && o->tokens > 0) {
    double gu = 0, dn = 0, aux = 0;
    for (int g = 0; g < steps; ++g) {
      float ms[6];
      for (int i = 0; i < 6; ++i) CK(cudaEventElapsedTime(&ms[i], c->run_ev[(size_t)g * 7 + i], c->run_ev[(size_t)g * 7 + i + 1]));
      gu += ms[3];
      dn += ms[4];
      aux += ms[0] + ms[1] + ms[2] + ms[5];
    }
    rep->kern_gate_up_ns = gu * 1e6 / steps;
    rep->kern_down_ns = dn * 1e6 / steps;
    rep->kern_aux_ns = aux * 1e6 / steps;
  }
  c->fz_total_ns = 0;
  c->fz_total_bytes = 0;
  c->fz_launches = c->fz_n;
  for (size_t i = 0; i < c->fz_n; ++i) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->fz_ev[2 * i], c->fz_ev[2 * i + 1]));
    c->fz_total_ns += ms * 1e6;
    c->fz_total_bytes += c->fz_bytes[i];
  }
  c->dec_total_ns = 0;
  c->dec_total_bytes = 0;
  c->dec_launches = c->dec_n;
  for (size_t i = 0; i < c->dec_n; ++i) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->dec_ev[2 * i], c->dec_ev[2 * i + 1]));
    c->dec_total_ns += ms * 1e6;
    c->dec_total_bytes += c->dec_bytes[i];
  }
  // sampled runs: the sampled launches' means, scaled to every launch of the run
  if (c->dec_n && c->dec_seen > c->dec_n) {
    const double f = (double)c->dec_seen / (double)c->dec_n;
    c->dec_total_ns *= f;
    c->dec_total_bytes = (decltype(c->dec_total_bytes))(c->dec_total_bytes * f);
    c->dec_launches = c->dec_seen;
  }
  if (c->fz_n && c->fz_seen > c->fz_n) {
    const double f = (double)c->fz_seen / (double)c->fz_n;
    c->fz_total_ns *= f;
    c->fz_total_bytes = (decltype(c->fz_total_bytes))(c->fz_total_bytes * f);
    c->fz_launches = c->fz_seen;
  }
  c->prof_mode = 0;

  if (paged) {
    // drain: the last two layers are still bound; release them like a finished
    // runner would drop its table (the reference keeps them until GC).
    for (int k = 0; k < 2; ++k)
      for (size_t pi = 0; pi < c->st[k].size(); ++pi)
        if (c->st[k][pi] == XPGB_PAGE_RESIDENT && !c->pinned[pi]) {
          const int layer = (int)(pi / c->E) + 1, e = (int)(pi % c->E);
          pt_unmap(c, layer, c->e_first + e + 1, k + 1);
        }
    pt_upload(c);
  }
}


static void session_abort(Ctx* c) {
  Session& ss = session_of(c);
  if (!ss.active) return;
  ss.active = false;
  c->fused_now = false;
  cudaDeviceSynchronize();
  // drop every binding so the next run starts from an empty ring
  for (int k = 0; k < 2; ++k)
    for (size_t pi = 0; pi < c->st[k].size(); ++pi) {
      if (c->pinned[pi]) continue;
      if (c->blk[k][pi]) {
        c->free_ids[k].insert(c->blk[k][pi]);
        c->owner[k][c->blk[k][pi]] = -1;
        c->bound -= sigma_of(c, k + 1);
      }
      c->blk[k][pi] = 0;
      c->st[k][pi] = XPGB_PAGE_UNMAPPED;
    }
  try {
    pt_upload(c);
  } catch (...) {
  }
}

static void run_impl(Ctx* c, const xpgb_run_opts* o, const float* x, float* y, xpgb_report* rep) {
  if (o->tokens > 0 && y != x) {
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyAsync(y, x, (size_t)o->tokens * c->H * 4, cudaMemcpyDeviceToDevice, c->s_comp));
  }
  session_begin(c, o, y);
  Session& ss = session_of(c);
  try {
  // inline order: mat(0), mat(1), then fwd(g) | mat(g+2) (pipeline.py:412-424); the
  // async mode enqueues the same order so every waited event is already recorded.
  session_materialize(c, 0);
  session_materialize(c, 1);
  for (int g = 0; g < ss.steps; ++g) {
    session_acquire(c, g, c->s_comp);
    session_compute(c, g);
    session_release(c, g, c->s_comp);
    session_materialize(c, g + 2);
  }
  } catch (...) {
    session_abort(c);
    throw;
  }
  session_end(c, rep);
}

// The compressed device tier: every device-tier tensor in the record format tfmt[ti] names --
// exponent-Huffman records copied from the host pool as they are (the reference's device tier),
// or FX4 records encoded by the GPU from the raw pool (copied raw into a scratch buffer; histogram
// -> base, escape counts -> size, then the record, straight into its slot).  Two passes over the
// FX4 tensors (sizes, then records), so the allocation is exact.  Setup work: it synchronises.
// Also builds the decode-into-GEMM kernel's record table and, for FX4 tensors, the TMA maps of
// their sign/mantissa and nibble planes.
static void stage_device_tier(Ctx* c) {
  if (c->dev_tier) {
    cudaFree(c->dev_tier);
    c->dev_tier = nullptr;
  }
  if (c->d_decrec) {
    cudaFree(c->d_decrec);
    c->d_decrec = nullptr;
  }
  if (c->d_fxmaps) {
    cudaFree(c->d_fxmaps);
    c->d_fxmaps = nullptr;
  }
  const size_t pages = (size_t)c->N * c->E, nt = pages * 2;
  if (c->tfmt.size() != nt) c->tfmt.assign(nt, 0);
  c->fx_base.assign(nt, 0);
  c->fx_bytes.assign(nt, 0);
  std::fill(c->dev_off.begin(), c->dev_off.end(), -1);
  auto huff_bytes = [&](size_t ti) -> uint64_t {
    const uint64_t raw = (ti & 1) ? c->s2 : c->s1;
    if (!c->codec) return raw;
    return xpgb_codec_record_bytes(raw / 2, c->rec_bits[ti], c->cchunk);
  };
  auto is_fx = [&](size_t ti) { return c->backend[ti] && c->codec && c->tfmt[ti] == 1; };
  auto raw_src = [&](size_t ti) { return c->host + (ti / 2) * (c->s1 + c->s2) + ((ti & 1) ? c->s1 : 0); };
  bool any = false, any_fx = false;
  for (size_t ti = 0; ti < nt; ++ti) {
    any |= c->backend[ti] != 0;
    any_fx |= is_fx(ti);
  }
  if (!any) return;
  if (!c->codec && !c->host) XFAIL(XPGB_ERR_BACKEND_MISS, "device-tier staging needs the host pool");
  if (any_fx && !c->host) XFAIL(XPGB_ERR_BACKEND_MISS, "the FX4 device tier is encoded from the raw host pool");
  const uint64_t maxraw = std::max(c->s1, c->s2);
  uint8_t* raw = nullptr;
  uint32_t* scratch = nullptr;
  cudaStream_t s = c->s_copy[0];
  if (any_fx) {
    CK(cudaMalloc(&raw, maxraw));
    CK(cudaMalloc(&scratch, xpgb_fx4_scratch_bytes(maxraw / 2)));
  }
  uint64_t total = 0;
  for (size_t ti = 0; ti < nt; ++ti) {
    if (!c->backend[ti]) continue;
    if (is_fx(ti)) {
      const uint64_t sz = (ti & 1) ? c->s2 : c->s1;
      CK(cudaMemcpyAsync(raw, raw_src(ti), sz, cudaMemcpyHostToDevice, s));
      int base = 0;
      uint64_t esc = 0;
      fx4_count(reinterpret_cast<const uint16_t*>(raw), sz / 2, scratch, &base, &esc, s);
      CKLAUNCH();
      c->fx_base[ti] = base;
      c->fx_bytes[ti] = fx_layout(sz / 2, esc).total;
      total += (c->fx_bytes[ti] + 255) & ~255ull;
    } else {
      total += (huff_bytes(ti) + 255) & ~255ull;
    }
  }
  CK(cudaMalloc(&c->dev_tier, total + 256));  // slack: stream readers fetch 16-byte blocks ahead
  uint64_t at = 0;
  for (size_t ti = 0; ti < nt; ++ti) {
    if (!c->backend[ti]) continue;
    c->dev_off[ti] = (int64_t)at;
    if (is_fx(ti)) {
      const uint64_t sz = (ti & 1) ? c->s2 : c->s1;
      CK(cudaMemcpyAsync(raw, raw_src(ti), sz, cudaMemcpyHostToDevice, s));
      fx4_encode(reinterpret_cast<const uint16_t*>(raw), sz / 2, c->fx_base[ti], scratch, c->dev_tier + at, s);
      CKLAUNCH();
      at += (c->fx_bytes[ti] + 255) & ~255ull;
    } else {
      const uint64_t sz = huff_bytes(ti);
      const uint8_t* src = c->codec ? c->cpool + c->rec_off[ti] : raw_src(ti);
      CK(cudaMemcpyAsync(c->dev_tier + at, src, sz, cudaMemcpyHostToDevice, s));
      at += (sz + 255) & ~255ull;
    }
  }
  CK(cudaStreamSynchronize(s));
  if (raw) cudaFree(raw);
  if (scratch) cudaFree(scratch);
  if (!c->codec) return;
  // records as the decode-into-GEMM kernel reads them, [layer][kind][expert]; TMA maps of every
  // FX4 tensor's planes (64-B / 32-B swizzles so the decoders' row reads spread banks)
  std::vector<CUtensorMap> maps(nt * 2);
  if (any_fx) {
    for (size_t ti = 0; ti < nt; ++ti) {
      if (!is_fx(ti)) continue;
      const uint64_t rows = (ti & 1) ? (uint64_t)c->H : 2ull * c->F, K = (ti & 1) ? (uint64_t)c->F : (uint64_t)c->H;
      const uint8_t* rec = c->dev_tier + c->dev_off[ti];
      const FxLayout L = fx_layout(rows * K, 0);
      maps[2 * ti] = make_map_u8(rec, rows, K, 64, CU_TENSOR_MAP_SWIZZLE_64B);
      maps[2 * ti + 1] = make_map_u8(rec + L.nib, rows, K / 2, 32, CU_TENSOR_MAP_SWIZZLE_32B);
    }
    CK(cudaMalloc(&c->d_fxmaps, maps.size() * sizeof(CUtensorMap)));
    CK(cudaMemcpy(c->d_fxmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  }
  std::vector<DecRec> recs(nt);
  memset(recs.data(), 0, recs.size() * sizeof(DecRec));
  for (size_t ti = 0; ti < nt; ++ti) {
    if (!c->backend[ti]) continue;
    const uint64_t n = ((ti & 1) ? c->s2 : c->s1) / 2;
    const uint8_t* rec = c->dev_tier + c->dev_off[ti];
    const size_t layer0 = ti / 2 / c->E, e = ti / 2 % c->E, k = ti & 1;
    DecRec& r = recs[(layer0 * 2 + k) * c->E + e];
    if (is_fx(ti)) {
      const FxLayout L = fx_layout(n, 0);
      r = DecRec{rec, reinterpret_cast<const uint32_t*>(rec + L.nib), reinterpret_cast<const uint32_t*>(rec + L.idx),
                 (uint32_t)c->fx_base[ti], 1u, rec + L.esc, c->d_fxmaps + 2 * ti};
    } else {
      const uint64_t sm16 = (n + 15) & ~15ull, bits16 = (c->rec_bits[ti] + 8 + 15) & ~15ull;
      r = DecRec{rec, reinterpret_cast<const uint32_t*>(rec + sm16),
                 reinterpret_cast<const uint32_t*>(rec + sm16 + bits16), 0u, 0u, nullptr, nullptr};
    }
  }
  CK(cudaMalloc(&c->d_decrec, recs.size() * sizeof(DecRec)));
  CK(cudaMemcpy(c->d_decrec, recs.data(), recs.size() * sizeof(DecRec), cudaMemcpyHostToDevice));
}

// Staging ring and device-resident chunk index of the compressed host tier (on), or neither
// (off: a plan that leaves no expert on the host tier gives their HBM back to the budget).
static void alloc_host_staging(Ctx* c, bool host_compressed) {
  const size_t nt = (size_t)c->N * c->E * 2;
  const int chunk = c->cchunk;
  // staging: n_stage buffers per kind, each min(largest record, kStagePieceBytes) + alignment slack
  if (const char* env = getenv("XPGB_STAGE_BUFS")) c->n_stage = std::max(2, std::min(kMaxStageBufs, atoi(env)));
  for (int k = 0; k < 2; ++k) {
    uint64_t cap = 0;
    if (host_compressed) {
      // largest record, or a whole layer's records of this kind when they are small
      uint64_t layer_sum = 0, largest = 0;
      for (size_t ti = k; ti < nt; ti += 2) {
        const uint64_t rb = xpgb_codec_record_bytes(((ti & 1) ? c->s2 : c->s1) / 2, c->rec_bits[ti], chunk);
        if ((ti / 2) % c->E == 0) layer_sum = 0;
        layer_sum += rb;
        largest = std::max(largest, rb);
        cap = std::max(cap, layer_sum);
      }
      // 64 MB pieces: DSv3's 39 MB gate/up records travel whole (98% of the link instead of
      // 93% in 32 MB pieces), Mixtral's 155 MB records in 3 pieces (97.5% vs 96.7%)
      (void)largest;
      uint64_t piece = kStagePieceBytes;
      if (const char* env = getenv("XPGB_STAGE_BYTES")) piece = std::max<uint64_t>(4096, strtoull(env, nullptr, 10));
      cap = std::min(cap, piece) + 64 + (uint64_t)chunk * 8;
    }
    for (int b = 0; b < kMaxStageBufs; ++b) {
      if (c->stage[k][b]) cudaFree(c->stage[k][b]);
      c->stage[k][b] = nullptr;
      if (cap && b < c->n_stage) CK(cudaMalloc(&c->stage[k][b], cap + 256));  // + read-ahead slack
    }
    c->stage_cap[k] = cap;
  }
  if (c->d_index) cudaFree(c->d_index);
  c->d_index = nullptr;
  c->d_index_off.assign(nt, 0);
  if (host_compressed) {
    uint64_t total = 0;
    for (size_t ti = 0; ti < nt; ++ti) {
      c->d_index_off[ti] = total;
      const uint64_t n = ((ti & 1) ? c->s2 : c->s1) / 2;
      total += (n + chunk - 1) / chunk;
    }
    CK(cudaMalloc(&c->d_index, std::max<uint64_t>(total, 1) * 4));
    for (size_t ti = 0; ti < nt; ++ti) {
      const uint64_t n = ((ti & 1) ? c->s2 : c->s1) / 2;
      const uint64_t sm16 = (n + 15) & ~15ull, bits16 = (c->rec_bits[ti] + 8 + 15) & ~15ull;
      CK(cudaMemcpy(c->d_index + c->d_index_off[ti], c->cpool + c->rec_off[ti] + sm16 + bits16,
                    ((n + chunk - 1) / chunk) * 4, cudaMemcpyHostToDevice));
    }
  }
}

static void set_codec(Ctx* c, const void* pool, uint64_t pool_bytes, const uint64_t* rec_offsets,
                      const uint64_t* bits_lens, const uint8_t* lengths, int chunk, bool host_compressed) {
  if (chunk <= 0 || chunk % 8) XFAIL(XPGB_ERR_CONFIG, "codec chunk must be a positive multiple of 8");
  uint32_t codes[kCodecSymbols];
  if (!codec_canonical_codes(lengths, codes)) XFAIL(XPGB_ERR_CONFIG, "invalid code lengths");
  const size_t nt = (size_t)c->N * c->E * 2;
  CK(cudaDeviceSynchronize());
  c->cpool = static_cast<const uint8_t*>(pool);
  c->cpool_bytes = pool_bytes;
  c->rec_off.assign(rec_offsets, rec_offsets + nt);
  c->rec_bits.assign(bits_lens, bits_lens + nt);
  memcpy(c->ctab.len, lengths, kCodecSymbols);
  prepare_decode_tables(c->ctab, nullptr);  // decoder tables built once, before any decode stream uses them
  CKLAUNCH();
  c->cchunk = chunk;
  c->codec = true;
  c->host_codec = host_compressed;
  for (size_t ti = 0; ti < nt; ++ti) {
    const uint64_t rb = xpgb_codec_record_bytes(((ti & 1) ? c->s2 : c->s1) / 2, c->rec_bits[ti], chunk);
    if (c->rec_off[ti] + rb > pool_bytes) XFAIL(XPGB_ERR_CONTAINER_FORMAT, "record %zu outside the packed pool", ti);
  }
  if (!c->codec_events) {
    for (int k = 0; k < 2; ++k) {
      CK(cudaStreamCreateWithFlags(&c->s_dec[k], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->s_alt[k], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->s_cp[k], cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->s_devdec[k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_devdec[k], cudaEventDisableTiming));
      for (int b = 0; b < kMaxStageBufs; ++b) {
        CK(cudaEventCreateWithFlags(&c->ev_copied[k][b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_decoded[k][b], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&c->ev_mapped[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_raw[k], cudaEventDisableTiming));
    }
    c->codec_events = true;
  }
  alloc_host_staging(c, host_compressed);
  stage_device_tier(c);
}

}  // namespace xpgb

using namespace xpgb;

struct xpgb_ctx {
  Ctx c;
};

// =========================================================================== C ABI

extern "C" {

int xpgb_abi_version(void) { return XPGB_ABI_VERSION; }
const char* xpgb_last_error(void) { return g_err.c_str(); }
int64_t xpgb_kernel_launches(void) { return g_launches.load(); }

static void create_impl(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, int32_t expert_first,
                        int32_t expert_count, xpgb_ctx** out);

int xpgb_create(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, xpgb_ctx** out) {
  return guard([&] { create_impl(spec, device, pool, max_tokens, 0, spec ? spec->experts_per_layer : 0, out); });
}

int xpgb_create_shard(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, int32_t expert_first,
                      int32_t expert_count, xpgb_ctx** out) {
  return guard([&] { create_impl(spec, device, pool, max_tokens, expert_first, expert_count, out); });
}

}  // extern "C"

static void create_impl(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, int32_t expert_first,
                        int32_t expert_count, xpgb_ctx** out) {
  {
    if (!spec || !out) XFAIL(XPGB_ERR, "null argument");
    if (spec->num_layers < 2) XFAIL(XPGB_ERR_OUT_OF_RANGE, "num_layers must be >= 2, got %d", spec->num_layers);
    if (spec->experts_per_layer < 1)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "experts_per_layer must be >= 1, got %d", spec->experts_per_layer);
    if (spec->hidden_dim < 1 || spec->intermediate_dim < 1)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "hidden_dim and intermediate_dim must be >= 1");
    if (spec->hidden_dim % 8 || spec->intermediate_dim % 8)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "B200 kernels need hidden_dim and intermediate_dim multiples of 8 (got %d, %d)",
            spec->hidden_dim, spec->intermediate_dim);
    if (spec->experts_per_layer > kMaxExperts)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "experts_per_layer above %d", kMaxExperts);
    if (pool != XPGB_POOL_RING && pool != XPGB_POOL_RESIDENT) XFAIL(XPGB_ERR_CONFIG, "unknown pool kind %d", pool);
    CK(cudaSetDevice(device));
    int major = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) XFAIL(XPGB_ERR_CUDA, "libxpgb is built for sm_100a; device %d has compute capability %d.x",
                           device, major);
    auto* h = new xpgb_ctx();
    Ctx* c = &h->c;
    c->N = spec->num_layers;
    c->L = spec->experts_per_layer;
    c->H = spec->hidden_dim;
    c->F = spec->intermediate_dim;
    c->device = device;
    c->pool = pool;
    if (expert_first < 0 || expert_count < 1 || expert_first + expert_count > c->L) {
      delete h;
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "shard [%d, %d) outside [0, %d)", expert_first, expert_first + expert_count, c->L);
    }
    c->e_first = expert_first;
    c->E = expert_count;  // pools and slot tables are sized for the shard from the start
    c->s1 = 2ull * c->H * 2 * c->F;
    c->s2 = 2ull * c->F * c->H;
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    set_gemm_attrs();
    set_gemm_dec_attrs();
    set_pair_gemm_attrs();
    if (const char* env = getenv("XPGB_PAIR_GEMM")) c->pair_mode = atoi(env) ? 1 : 0;
    if (const char* env = getenv("XPGB_FAST_PREFILL")) c->pair_split = atoi(env) == 0;
    for (int k = 0; k < 2; ++k) CK(cudaStreamCreateWithFlags(&c->s_copy[k], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k)
      for (int i = 0; i < kEvRing; ++i) CK(cudaEventCreateWithFlags(&c->ev_load[k][i], cudaEventDisableTiming));
    for (int i = 0; i < kEvRing; ++i) CK(cudaEventCreateWithFlags(&c->ev_comp[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_begin, cudaEventDisableTiming));
    CK(cudaEventCreate(&c->ev_end));
    for (int i = 0; i < 7; ++i) CK(cudaEventCreate(&c->pev[i]));
    CK(cudaMalloc(&c->d_fault, sizeof(long long)));
    CK(cudaMemset(c->d_fault, 0, sizeof(long long)));
    CK(cudaMalloc(&c->d_log_count, sizeof(int32_t)));
    CK(cudaMemset(c->d_log_count, 0, sizeof(int32_t)));
    init_pools(c);
    ensure_work(c, std::max(1, max_tokens), std::min(c->L, 8));
    *out = h;
  }
}

extern "C" {

int xpgb_destroy(xpgb_ctx* h) {
  return guard([&] {
    if (!h) return;
    Ctx* c = &h->c;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    free_pools(c);
    if (c->shared_w) cudaFree(c->shared_w);
    c->shared_w = nullptr;
    free_work(c);
    void* ptrs[] = {c->d_fault, c->d_log, c->d_log_count};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (c->host && c->host_owned) cudaFreeHost(c->host);
    if (c->host && c->host_registered) cudaHostUnregister(c->host);
    for (int k = 0; k < 2; ++k) {
      cudaStreamDestroy(c->s_copy[k]);
      for (int i = 0; i < kEvRing; ++i) cudaEventDestroy(c->ev_load[k][i]);
    }
    for (int i = 0; i < kEvRing; ++i) cudaEventDestroy(c->ev_comp[i]);
    cudaEventDestroy(c->ev_begin);
    cudaEventDestroy(c->ev_end);
    for (int i = 0; i < 7; ++i) cudaEventDestroy(c->pev[i]);
    for (cudaEvent_t e : c->run_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->dec_ev) cudaEventDestroy(e);
    delete c->sess;
    if (c->codec_events) {
      for (int k = 0; k < 2; ++k) {
        cudaStreamDestroy(c->s_dec[k]);
        cudaStreamDestroy(c->s_alt[k]);
        cudaStreamDestroy(c->s_cp[k]);
        cudaStreamDestroy(c->s_devdec[k]);
        cudaEventDestroy(c->ev_devdec[k]);
        for (int b = 0; b < kMaxStageBufs; ++b) {
          cudaEventDestroy(c->ev_copied[k][b]);
          cudaEventDestroy(c->ev_decoded[k][b]);
          if (c->stage[k][b]) cudaFree(c->stage[k][b]);
        }
        cudaEventDestroy(c->ev_mapped[k]);
        cudaEventDestroy(c->ev_raw[k]);
      }
      if (c->d_index) cudaFree(c->d_index);
    }
    cudaStreamDestroy(c->s_comp);
    delete h;
  });
}

int xpgb_sync(xpgb_ctx* h) {
  return guard([&] { CK(cudaDeviceSynchronize()); (void)h; });
}

int xpgb_pinned_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    *out = nullptr;
    CK(cudaHostAlloc(out, std::max<uint64_t>(bytes, 1), cudaHostAllocPortable));
  });
}
int xpgb_host_register(void* ptr, uint64_t bytes, int32_t read_only) {
  return guard([&] {
    if (!ptr || !bytes) XFAIL(XPGB_ERR, "null host range");
    const uintptr_t page = 4096, a = reinterpret_cast<uintptr_t>(ptr) & ~(page - 1);
    const uintptr_t b = (reinterpret_cast<uintptr_t>(ptr) + bytes + page - 1) & ~(page - 1);
    unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
    cudaError_t e = cudaHostRegister(reinterpret_cast<void*>(a), b - a, flags);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
      return;
    }
    if (e != cudaSuccess) throw Err{XPGB_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e)};
  });
}

int xpgb_host_unregister(void* ptr) {
  return guard([&] {
    const uintptr_t a = reinterpret_cast<uintptr_t>(ptr) & ~uintptr_t(4095);
    cudaError_t e = cudaHostUnregister(reinterpret_cast<void*>(a));
    if (e != cudaSuccess) {
      cudaGetLastError();
      XFAIL(XPGB_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
    }
  });
}

int xpgb_pinned_free(void* ptr) {
  return guard([&] {
    if (ptr) CK(cudaFreeHost(ptr));
  });
}

int xpgb_host_pool_alloc(xpgb_ctx* h, void** host_ptr, uint64_t* bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    const uint64_t need = (uint64_t)c->N * c->E * (c->s1 + c->s2);
    if (c->host && c->host_owned && c->host_bytes == need) {
      *host_ptr = c->host;
      if (bytes) *bytes = need;
      return;
    }
    if (c->host && c->host_owned) cudaFreeHost(c->host);
    if (c->host && c->host_registered) cudaHostUnregister(c->host);
    c->host = nullptr;
    c->host_owned = c->host_registered = false;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&c->host), need, cudaHostAllocPortable));
    c->host_owned = true;
    c->host_bytes = need;
    *host_ptr = c->host;
    if (bytes) *bytes = need;
  });
}

int xpgb_host_pool_register(xpgb_ctx* h, void* host_ptr, uint64_t bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    const uint64_t need = (uint64_t)c->N * c->E * (c->s1 + c->s2);
    if (bytes != need)
      XFAIL(XPGB_ERR_CONTAINER_FORMAT, "payload is %llu bytes, expected %llu", (unsigned long long)bytes,
            (unsigned long long)need);
    if (c->host && c->host_owned) cudaFreeHost(c->host);
    if (c->host && c->host_registered) cudaHostUnregister(c->host);
    c->host = static_cast<uint8_t*>(host_ptr);
    c->host_owned = false;
    c->host_registered = false;
    cudaPointerAttributes attr;
    cudaError_t q = cudaPointerGetAttributes(&attr, host_ptr);
    const bool pinned = (q == cudaSuccess && attr.type == cudaMemoryTypeHost);
    if (q != cudaSuccess) cudaGetLastError();
    if (!pinned) {
      cudaError_t e = cudaHostRegister(host_ptr, bytes, cudaHostRegisterPortable);
      if (e == cudaSuccess) {
        c->host_registered = true;
      } else if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
      } else {
        c->host = nullptr;
        throw Err{XPGB_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e)};
      }
    }
    c->host_bytes = bytes;
  });
}

int xpgb_set_placement(xpgb_ctx* h, const uint8_t* backend_of) {
  return guard([&] {
    Ctx* c = &h->c;
    for (int layer = 0; layer < c->N; ++layer)
      for (int e = 0; e < c->E; ++e)
        for (int k = 0; k < 2; ++k)
          c->backend[((size_t)layer * c->E + e) * 2 + k] =
              backend_of ? (backend_of[((size_t)layer * c->L + c->e_first + e) * 2 + k] ? 1 : 0) : 0;
    stage_device_tier(c);
  });
}

int xpgb_fetch(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, void* dst, uint64_t dst_bytes,
               void* stream) {
  return guard([&] { fetch(&h->c, layer, expert, kind, dst, dst_bytes, (cudaStream_t)stream, nullptr); });
}

int xpgb_pt_map(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, int32_t* block_id) {
  return guard([&] {
    const int b = pt_map(&h->c, layer, expert, kind);
    pt_sync_entry(&h->c, layer, expert, kind);
    if (block_id) *block_id = b;
  });
}
int xpgb_pt_mark_resident(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind) {
  return guard([&] {
    pt_mark_resident(&h->c, layer, expert, kind);
    pt_sync_entry(&h->c, layer, expert, kind);
  });
}
int xpgb_pt_unmap(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind) {
  return guard([&] {
    pt_unmap(&h->c, layer, expert, kind);
    pt_sync_entry(&h->c, layer, expert, kind);
  });
}
int xpgb_pt_state(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, int32_t* state) {
  return guard([&] { *state = h->c.st[kind - 1][page_index(&h->c, layer, expert, kind)]; });
}
int xpgb_pt_block(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, int32_t* block_id) {
  return guard([&] { *block_id = h->c.blk[kind - 1][page_index(&h->c, layer, expert, kind)]; });
}
int xpgb_pt_block_ptr(xpgb_ctx* h, int32_t kind, int32_t block_id, void** dptr, uint64_t* bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    if (kind != 1 && kind != 2) XFAIL(XPGB_ERR_OUT_OF_RANGE, "unknown tensor kind %d", kind);
    if (block_id < 1 || block_id > c->blocks)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "block %d outside [1, %d]", block_id, c->blocks);
    *dptr = block_ptr(c, kind, block_id);
    if (bytes) *bytes = sigma_of(c, kind);
  });
}
int xpgb_pt_loading_view(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, void** dptr, uint64_t* bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    const int pi = page_index(c, layer, expert, kind);
    if (c->st[kind - 1][pi] != XPGB_PAGE_LOADING)
      XFAIL(XPGB_ERR_PAGE_FAULT, "write through %s while %s", tid_str(layer, expert, kind).c_str(),
            state_name(c->st[kind - 1][pi]));
    *dptr = block_ptr(c, kind, c->blk[kind - 1][pi]);
    if (bytes) *bytes = sigma_of(c, kind);
  });
}
int xpgb_pt_read(xpgb_ctx* h, int32_t layer, int32_t expert, int32_t kind, void* host_dst, uint64_t bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    const int pi = page_index(c, layer, expert, kind);
    if (c->st[kind - 1][pi] != XPGB_PAGE_RESIDENT)
      XFAIL(XPGB_ERR_PAGE_FAULT, "read through %s while %s", tid_str(layer, expert, kind).c_str(),
            state_name(c->st[kind - 1][pi]));
    const uint64_t sz = sigma_of(c, kind);
    if (bytes < sz) XFAIL(XPGB_ERR_OUT_OF_RANGE, "destination holds %llu bytes, page has %llu",
                          (unsigned long long)bytes, (unsigned long long)sz);
    CK(cudaMemcpy(host_dst, block_ptr(c, kind, c->blk[kind - 1][pi]), sz, cudaMemcpyDeviceToHost));
  });
}
int xpgb_pt_peak_bytes(xpgb_ctx* h, uint64_t* peak) {
  return guard([&] { *peak = h->c.peak; });
}
int xpgb_pt_pool_bytes(xpgb_ctx* h, uint64_t* bytes) {
  return guard([&] { *bytes = (uint64_t)h->c.blocks * (h->c.s1 + h->c.s2); });
}
int xpgb_pt_check_consistency(xpgb_ctx* h) {
  return guard([&] {
    Ctx* c = &h->c;
    for (int k = 0; k < 2; ++k) {
      size_t bound = 0;
      for (size_t pi = 0; pi < c->blk[k].size(); ++pi) {
        const int b = c->blk[k][pi];
        if (b) {
          ++bound;
          if (c->owner[k][b] != (int)pi) XFAIL(XPGB_ERR, "forward/reverse maps disagree at block %d", b);
          if (c->free_ids[k].count(b)) XFAIL(XPGB_ERR, "block %d both bound and free", b);
        }
      }
      if (bound + c->free_ids[k].size() != (size_t)c->blocks) XFAIL(XPGB_ERR, "block accounting broken");
    }
  });
}
int xpgb_pt_trace_enable(xpgb_ctx* h, int32_t enable) {
  return guard([&] {
    h->c.trace_on = enable != 0;
    h->c.trace.clear();
  });
}
int xpgb_pt_trace_get(xpgb_ctx* h, char* buf, uint64_t cap, uint64_t* needed) {
  return guard([&] {
    const std::string& t = h->c.trace;
    if (needed) *needed = t.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(t.size(), cap - 1);
      memcpy(buf, t.data(), n);
      buf[n] = 0;
    }
  });
}
int xpgb_make_resident(xpgb_ctx* h) {
  return guard([&] {
    Ctx* c = &h->c;
    cudaStream_t s = c->s_copy[0];
    for (int layer = 1; layer <= c->N; ++layer)
      for (int e = 0; e < c->E; ++e)
        for (int kind = 1; kind <= 2; ++kind) {
          const int ex = c->e_first + e + 1;
          const int pi = page_index(c, layer, ex, kind);
          if (c->st[kind - 1][pi] == XPGB_PAGE_RESIDENT) continue;
          const int b = pt_map(c, layer, ex, kind);
          fetch(c, layer, ex, kind, block_ptr(c, kind, b), sigma_of(c, kind), s, nullptr);
          pt_mark_resident(c, layer, ex, kind);
        }
    CK(cudaStreamSynchronize(s));
    // bulk device-table upload
    const size_t pages = (size_t)c->N * c->E;
    std::vector<int32_t> tab(2 * pages);
    for (int k = 0; k < 2; ++k)
      for (size_t pi = 0; pi < pages; ++pi)
        tab[k * pages + pi] = c->st[k][pi] == XPGB_PAGE_UNMAPPED ? -1 : pt_entry(c->blk[k][pi] - 1, c->st[k][pi]);
    CK(cudaMemcpy(c->d_pt, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
  });
}

uint64_t xpgb_codec_record_bytes(uint64_t n, uint64_t bits_len, int32_t chunk) {
  const uint64_t ch = chunk > 0 ? (uint64_t)chunk : 1;
  return ((n + 15) & ~15ull) + ((bits_len + 8 + 15) & ~15ull) + ((((n + ch - 1) / ch) * 4 + 15) & ~15ull);
}

int xpgb_codec_histogram(const void* data, uint64_t bytes, uint64_t* counts256, int32_t threads) {
  return guard([&] {
    if (bytes % 2) XFAIL(XPGB_ERR_ODD_LENGTH, "bf16 payload has odd length %llu", (unsigned long long)bytes);
    codec_histogram(static_cast<const uint8_t*>(data), bytes, counts256, threads);
  });
}

int xpgb_codec_encode(const void* data, uint64_t bytes, const uint8_t* lengths256, void* sm_out, void* bits_out,
                      uint64_t bits_cap, uint64_t* bits_len, uint64_t* bit_count, uint32_t* index_out,
                      int32_t chunk) {
  return guard([&] {
    if (bytes % 2) XFAIL(XPGB_ERR_ODD_LENGTH, "bf16 payload has odd length %llu", (unsigned long long)bytes);
    uint32_t codes[kCodecSymbols];
    if (!codec_canonical_codes(lengths256, codes)) XFAIL(XPGB_ERR_CONFIG, "invalid code lengths");
    size_t bl = 0;
    uint64_t bc = 0;
    int missing = -1;
    const bool ok = codec_encode(static_cast<const uint16_t*>(data), bytes / 2, lengths256, codes,
                                 static_cast<uint8_t*>(sm_out), static_cast<uint8_t*>(bits_out), bits_cap, &bl, &bc,
                                 index_out, chunk, &missing);
    if (missing >= 0) XFAIL(XPGB_ERR_SYMBOL_NOT_IN_TABLE, "exponent bytes [%d] have no codeword; wrong table?", missing);
    if (!ok) XFAIL(XPGB_ERR_OUT_OF_RANGE, "bitstream needs %llu bytes, buffer holds %llu", (unsigned long long)bl,
                   (unsigned long long)bits_cap);
    *bits_len = bl;
    *bit_count = bc;
  });
}

int xpgb_codec_pack(const void* payload, int32_t n_tensors, const uint64_t* value_counts, const uint8_t* lengths256,
                    int32_t chunk, int32_t threads, const int32_t* place_order, void* out, uint64_t out_cap,
                    uint64_t* pool_bytes, uint64_t* rec_offsets, uint64_t* bits_lens, uint64_t* bit_counts) {
  return guard([&] {
    if (chunk <= 0 || chunk % 8) XFAIL(XPGB_ERR_CONFIG, "codec chunk must be a positive multiple of 8");
    uint32_t codes[kCodecSymbols];
    if (!codec_canonical_codes(lengths256, codes)) XFAIL(XPGB_ERR_CONFIG, "invalid code lengths");
    const uint16_t* words = static_cast<const uint16_t*>(payload);
    std::vector<uint64_t> first(n_tensors + 1, 0);
    for (int i = 0; i < n_tensors; ++i) first[i + 1] = first[i] + value_counts[i];
    const int nthr = std::max(1, threads);
    std::vector<int> bad(n_tensors, -1);
    // pass 1: exact stream bits per tensor from per-tensor histograms -> record layout
    {
      std::vector<std::thread> pool_t;
      std::atomic<int> next{0};
      for (int t = 0; t < nthr; ++t)
        pool_t.emplace_back([&] {
          for (int i = next++; i < n_tensors; i = next++) {
            uint64_t cnt[kCodecSymbols] = {0};
            for (uint64_t v = first[i]; v < first[i + 1]; ++v) ++cnt[(words[v] >> 7) & 0xFF];
            uint64_t bits = 0;
            for (int sy = 0; sy < kCodecSymbols; ++sy) {
              if (cnt[sy] && !lengths256[sy]) bad[i] = sy;
              bits += cnt[sy] * lengths256[sy];
            }
            bit_counts[i] = bits;
            bits_lens[i] = (bits + 7) / 8;
          }
        });
      for (auto& th : pool_t) th.join();
    }
    for (int i = 0; i < n_tensors; ++i)
      if (bad[i] >= 0)
        XFAIL(XPGB_ERR_SYMBOL_NOT_IN_TABLE, "exponent bytes [%d] have no codeword; wrong table?", bad[i]);
    if (place_order) {
      std::vector<char> seen(n_tensors, 0);
      for (int j = 0; j < n_tensors; ++j) {
        const int i = place_order[j];
        if (i < 0 || i >= n_tensors || seen[i]) XFAIL(XPGB_ERR_CONFIG, "place_order is not a permutation");
        seen[i] = 1;
      }
    }
    uint64_t total = 0;
    for (int j = 0; j < n_tensors; ++j) {
      const int i = place_order ? place_order[j] : j;
      rec_offsets[i] = total;
      total += xpgb_codec_record_bytes(value_counts[i], bits_lens[i], chunk);
    }
    *pool_bytes = total;
    if (!out) return;  // layout only
    if (out_cap < total) XFAIL(XPGB_ERR_OUT_OF_RANGE, "packed pool needs %llu bytes, buffer holds %llu",
                               (unsigned long long)total, (unsigned long long)out_cap);
    // pass 2: encode every tensor into its record
    std::atomic<int> next{0};
    std::atomic<int> fail{0};
    std::vector<std::thread> pool_t;
    for (int t = 0; t < nthr; ++t)
      pool_t.emplace_back([&] {
        for (int i = next++; i < n_tensors; i = next++) {
          uint8_t* rec = static_cast<uint8_t*>(out) + rec_offsets[i];
          const uint64_t n = value_counts[i];
          const uint64_t sm16 = (n + 15) & ~15ull, bits16 = (bits_lens[i] + 8 + 15) & ~15ull;
          const uint64_t rb = xpgb_codec_record_bytes(n, bits_lens[i], chunk);
          memset(rec, 0, rb);
          size_t bl = 0;
          uint64_t bc = 0;
          int missing = -1;
          if (!codec_encode(words + first[i], n, lengths256, codes, rec, rec + sm16, bits_lens[i], &bl, &bc,
                            reinterpret_cast<uint32_t*>(rec + sm16 + bits16), chunk, &missing) ||
              bl != bits_lens[i] || bc != bit_counts[i])
            fail = 1;
        }
      });
    for (auto& th : pool_t) th.join();
    if (fail) XFAIL(XPGB_ERR, "codec pack: stream size mismatch");
  });
}

int xpgb_codec_index(const void* bits, uint64_t bits_len, uint64_t n, const uint8_t* lengths256, int32_t chunk,
                     uint32_t* index_out, uint64_t* consumed_bits) {
  return guard([&] {
    if (chunk <= 0 || chunk % 8) XFAIL(XPGB_ERR_CONFIG, "codec chunk must be a positive multiple of 8");
    size_t used = 0;
    const int r = codec_build_index(static_cast<const uint8_t*>(bits), bits_len, n, lengths256, chunk, index_out, &used);
    if (r == 1) XFAIL(XPGB_ERR_TRUNCATED_STREAM, "bitstream ended before all %llu values", (unsigned long long)n);
    if (r == 2) XFAIL(XPGB_ERR_INVALID_CODE, "no codeword matches a bit pattern in the stream");
    if (consumed_bits) *consumed_bits = used;
  });
}

int xpgb_codec_decode(const void* record_dev, uint64_t n, uint64_t bits_len, int32_t chunk, const uint8_t* lengths256,
                      void* out_dev, void* stream) {
  return guard([&] {
    if (chunk <= 0 || chunk % 8) XFAIL(XPGB_ERR_CONFIG, "codec chunk must be a positive multiple of 8");
    uint32_t codes[kCodecSymbols];
    if (!codec_canonical_codes(lengths256, codes)) XFAIL(XPGB_ERR_CONFIG, "invalid code lengths");
    CodecTable t;
    memcpy(t.len, lengths256, kCodecSymbols);
    const uint8_t* rec = static_cast<const uint8_t*>(record_dev);
    const uint64_t sm16 = (n + 15) & ~15ull, bits16 = (bits_len + 8 + 15) & ~15ull;
    launch_exp_decode(rec, reinterpret_cast<const uint32_t*>(rec + sm16),
                      reinterpret_cast<const uint32_t*>(rec + sm16 + bits16), n, chunk, t,
                      static_cast<uint16_t*>(out_dev), (cudaStream_t)stream);
    CKLAUNCH();
  });
}

uint64_t xpgb_fx4_scratch_bytes(uint64_t n) { return (n / kFxSeg + 1) * 4 + 1024 + 256; }

int xpgb_fx4_measure(const void* raw_dev, uint64_t n, void* scratch_dev, int32_t* base, uint64_t* n_escapes,
                     uint64_t* record_bytes, void* stream) {
  return guard([&] {
    if (n % kFxSeg) XFAIL(XPGB_ERR_CONFIG, "FX4 tensors hold a multiple of %d values", kFxSeg);
    int b = 0;
    uint64_t esc = 0;
    fx4_count(static_cast<const uint16_t*>(raw_dev), n, static_cast<uint32_t*>(scratch_dev), &b, &esc,
              (cudaStream_t)stream);
    CKLAUNCH();
    *base = b;
    if (n_escapes) *n_escapes = esc;
    if (record_bytes) *record_bytes = fx_layout(n, esc).total;
  });
}

int xpgb_fx4_encode(const void* raw_dev, uint64_t n, int32_t base, void* scratch_dev, void* record_dev, void* stream) {
  return guard([&] {
    if (n % kFxSeg) XFAIL(XPGB_ERR_CONFIG, "FX4 tensors hold a multiple of %d values", kFxSeg);
    if (base < 0 || base > kFxMaxBase) XFAIL(XPGB_ERR_OUT_OF_RANGE, "FX4 base %d outside [0, %d]", base, kFxMaxBase);
    fx4_encode(static_cast<const uint16_t*>(raw_dev), n, base, static_cast<uint32_t*>(scratch_dev),
               static_cast<uint8_t*>(record_dev), (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_fx4_decode(const void* record_dev, uint64_t n, int32_t base, void* out_dev, void* stream) {
  return guard([&] {
    if (n % kFxSeg) XFAIL(XPGB_ERR_CONFIG, "FX4 tensors hold a multiple of %d values", kFxSeg);
    launch_fx4_decode(static_cast<const uint8_t*>(record_dev), n, base, static_cast<uint16_t*>(out_dev),
                      (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_set_codec(xpgb_ctx* h, const void* pool, uint64_t pool_bytes, const uint64_t* rec_offsets,
                   const uint64_t* bits_lens, const uint8_t* lengths256, int32_t chunk, int32_t host_compressed) {
  return guard([&] {
    set_codec(&h->c, pool, pool_bytes, rec_offsets, bits_lens, lengths256, chunk, host_compressed != 0);
  });
}

int xpgb_hbm_bytes(xpgb_ctx* h, uint64_t* ring, uint64_t* staging, uint64_t* device_tier) {
  return guard([&] {
    Ctx* c = &h->c;
    // resident expert bytes: the ring arena (+ pinned blocks) and the shared experts
    *ring = (uint64_t)c->blocks * (c->s1 + c->s2) + (uint64_t)c->N * c->S * (c->s1 + c->s2);
    *staging = (uint64_t)c->n_stage * (c->stage_cap[0] + c->stage_cap[1]);
    if (c->d_index) {
      uint64_t entries = 0;
      const size_t nt = (size_t)c->N * c->E * 2;
      for (size_t ti = 0; ti < nt; ++ti) entries += ((((ti & 1) ? c->s2 : c->s1) / 2) + c->cchunk - 1) / c->cchunk;
      *staging += entries * 4;
    }
    uint64_t dt = 0;
    const size_t nt = (size_t)c->N * c->E * 2;
    for (size_t ti = 0; ti < nt && c->dev_tier; ++ti)
      if (c->backend[ti]) {
        const uint64_t raw = (ti & 1) ? c->s2 : c->s1;
        dt += (c->codec && fmt_of(c, ti) == 1) ? c->fx_bytes[ti]
              : c->codec      ? xpgb_codec_record_bytes(raw / 2, c->rec_bits[ti], c->cchunk)
                              : raw;
      }
    *device_tier = dt;
  });
}

}  // extern "C"

// Re-create the arena for a residency mask and ring cap: pinned experts get dedicated
// blocks (filled from the host pool), the ring gets 2 x (most streamed experts of any
// layer) blocks per kind, capped by ring_limit (sub-layer ring).
static void apply_residency(Ctx* c, std::vector<uint8_t> mask) {  // by value: callers pass c->pinned, which init_pools clears
  int n_pinned = 0, max_streamed = 0;
  for (int l = 0; l < c->N; ++l) {
    int streamed = 0;
    for (int e = 0; e < c->E; ++e) {
      n_pinned += mask[(size_t)l * c->E + e];
      streamed += !mask[(size_t)l * c->E + e];
    }
    max_streamed = std::max(max_streamed, streamed);
  }
  if (n_pinned && !c->host) XFAIL(XPGB_ERR_BACKEND_MISS, "pinning experts needs the host pool");
  const int D = depth_of(c);
  int ring = D * max_streamed;
  if (c->ring_limit > 0) ring = std::min(ring, c->ring_limit / D * D);
  std::vector<uint8_t> backend = c->backend;
  CK(cudaDeviceSynchronize());
  init_pools(c, ring, n_pinned);
  c->backend = backend;
  c->pinned = mask;
  int next = c->ring_blocks + 1;
  for (int l = 1; l <= c->N; ++l)
    for (int e = 0; e < c->E; ++e) {
      if (!mask[(size_t)(l - 1) * c->E + e]) continue;
      for (int kind = 1; kind <= 2; ++kind) {
        const int k = kind - 1;
        const size_t pi = (size_t)(l - 1) * c->E + e;
        c->free_ids[k].erase(next);
        c->blk[k][pi] = next;
        c->owner[k][next] = (int)pi;
        c->st[k][pi] = XPGB_PAGE_RESIDENT;
        c->bound += sigma_of(c, kind);
        const uint64_t off = pi * (c->s1 + c->s2) + (kind == 2 ? c->s1 : 0);
        CK(cudaMemcpy(block_ptr(c, kind, next), c->host + off, sigma_of(c, kind), cudaMemcpyHostToDevice));
      }
      ++next;
    }
  c->peak = c->bound;
  pt_upload(c);
  stage_device_tier(c);  // the device tier survives; re-stage it beside the new arena
}

extern "C" {

int xpgb_set_pinned(xpgb_ctx* h, const uint8_t* pinned_of) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->pool != XPGB_POOL_RING) XFAIL(XPGB_ERR_CONFIG, "pinned experts need a ring context");
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot pin experts during a session");
    std::vector<uint8_t> mask((size_t)c->N * c->E, 0);
    for (int l = 0; l < c->N; ++l)
      for (int e = 0; e < c->E; ++e)
        mask[(size_t)l * c->E + e] = pinned_of ? (pinned_of[(size_t)l * c->L + c->e_first + e] ? 1 : 0) : 0;
    apply_residency(c, mask);
  });
}

int xpgb_set_ring_experts(xpgb_ctx* h, int32_t ring_experts) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->pool != XPGB_POOL_RING) XFAIL(XPGB_ERR_CONFIG, "a sub-layer ring needs a ring context");
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot resize the ring during a session");
    if (ring_experts == 0 || ring_experts < -1 || (ring_experts > 0 && ring_experts < c->ring_depth))
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "ring of %d experts per kind: need >= the ring depth %d (or -1 for two layers)",
            ring_experts, c->ring_depth);
    c->ring_limit = ring_experts < 0 ? 0 : ring_experts;
    apply_residency(c, c->pinned);
  });
}

int xpgb_set_hazard_checks(xpgb_ctx* h, int32_t poison, int32_t skip_war_iteration, int32_t skip_war_layer) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change hazard checks during a session");
    c->poison = poison != 0;
    c->war_sab_it = skip_war_iteration;
    c->war_sab_layer = skip_war_layer;
  });
}

int xpgb_set_host_staging(xpgb_ctx* h, int32_t on) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change the host staging during a session");
    if (!c->codec || !c->host_codec) XFAIL(XPGB_ERR_CONFIG, "no compressed host tier");
    const size_t nt = (size_t)c->N * c->E * 2;
    if (!on)
      for (size_t ti = 0; ti < nt; ++ti)
        if (!c->backend[ti] && !c->pinned[ti / 2])
          XFAIL(XPGB_ERR_CONFIG, "tensor %zu is on the host tier: its records need the staging ring", ti);
    CK(cudaDeviceSynchronize());
    alloc_host_staging(c, on != 0);  // released: a host-tier record would fail loudly in materialize
  });
}

int xpgb_set_device_format(xpgb_ctx* h, int32_t format) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change the device-tier format during a session");
    if (format < 0 || format > 1) XFAIL(XPGB_ERR_OUT_OF_RANGE, "device-tier format %d: need 0 (Huffman) or 1 (FX4)", format);
    const size_t nt = (size_t)c->N * c->E * 2;
    if (c->tfmt.size() == nt && std::all_of(c->tfmt.begin(), c->tfmt.end(), [&](uint8_t f) { return f == format; }))
      return;
    CK(cudaDeviceSynchronize());
    c->tfmt.assign(nt, (uint8_t)format);
    if (c->codec) stage_device_tier(c);  // re-stage whatever is placed on the device tier
  });
}

int xpgb_set_device_formats(xpgb_ctx* h, const uint8_t* formats) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change the device-tier format during a session");
    if (!formats) XFAIL(XPGB_ERR_CONFIG, "formats is null");
    const size_t nt = (size_t)c->N * c->E * 2;
    for (size_t ti = 0; ti < nt; ++ti)
      if (formats[ti] > 1) XFAIL(XPGB_ERR_OUT_OF_RANGE, "tensor %zu: device-tier format %d: need 0 or 1", ti, (int)formats[ti]);
    if (c->tfmt.size() == nt && std::equal(c->tfmt.begin(), c->tfmt.end(), formats)) return;
    CK(cudaDeviceSynchronize());
    c->tfmt.assign(formats, formats + nt);
    if (c->codec) stage_device_tier(c);
  });
}

int xpgb_set_activation_planes(xpgb_ctx* h, int32_t planes) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change the activation planes during a session");
    if (planes != 1 && planes != 2) XFAIL(XPGB_ERR_OUT_OF_RANGE, "activation planes %d: need 1 or 2", planes);
    c->act_planes = planes;
  });
}

int xpgb_set_fused_decode(xpgb_ctx* h, int32_t mode) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot switch decode-into-GEMM during a session");
    if (mode < 0 || mode > 2) XFAIL(XPGB_ERR_OUT_OF_RANGE, "fused decode mode %d: need 0, 1 or 2", mode);
    c->fused_mode = mode;
  });
}

int xpgb_set_ring_depth(xpgb_ctx* h, int32_t depth) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change the ring depth during a session");
    if (depth < 1 || depth > kMaxRingDepth) XFAIL(XPGB_ERR_OUT_OF_RANGE, "ring depth %d: need 1..%d", depth, kMaxRingDepth);
    if (c->ring_limit > 0 && c->ring_limit < depth)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "ring depth %d exceeds the ring of %d experts", depth, c->ring_limit);
    c->ring_depth = depth;
    if (c->ring_limit > 0) apply_residency(c, c->pinned);
  });
}

int xpgb_fused_stats(xpgb_ctx* h, int64_t* launches, double* kernel_ns, int64_t* record_bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    *launches = (int64_t)c->fz_launches;
    *kernel_ns = c->fz_total_ns;
    *record_bytes = (int64_t)c->fz_total_bytes;
  });
}

int xpgb_decode_stats(xpgb_ctx* h, int64_t* launches, double* kernel_ns, int64_t* algo_bytes) {
  return guard([&] {
    Ctx* c = &h->c;
    *launches = (int64_t)c->dec_launches;
    *kernel_ns = c->dec_total_ns;
    *algo_bytes = (int64_t)c->dec_total_bytes;
  });
}

int xpgb_set_stage_buffers(xpgb_ctx* h, int32_t n_buffers) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot resize the staging ring during a session");
    if (n_buffers < 2 || n_buffers > kMaxStageBufs)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "%d staging buffers per kind: need 2..%d", n_buffers, kMaxStageBufs);
    CK(cudaDeviceSynchronize());
    for (int k = 0; k < 2; ++k) {
      for (int b = 0; b < kMaxStageBufs; ++b) {
        const bool want = b < n_buffers && c->stage_cap[k] > 0;
        if (want && !c->stage[k][b]) CK(cudaMalloc(&c->stage[k][b], c->stage_cap[k] + 256));
        if (!want && c->stage[k][b]) {
          CK(cudaFree(c->stage[k][b]));
          c->stage[k][b] = nullptr;
        }
      }
      c->stage_next[k] = 0;
    }
    c->n_stage = n_buffers;
  });
}

int xpgb_set_shared(xpgb_ctx* h, const void* host, uint64_t bytes, int32_t n_shared) {
  return guard([&] {
    Ctx* c = &h->c;
    if (c->sess && c->sess->active) XFAIL(XPGB_ERR, "cannot change shared experts during a session");
    if (n_shared < 0 || c->E + n_shared > kMaxExperts)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "shared experts %d outside [0, %d]", n_shared, kMaxExperts - c->E);
    if (n_shared >= kMaxTopK) XFAIL(XPGB_ERR_OUT_OF_RANGE, "shared experts %d leave no routed slot", n_shared);
    const uint64_t want = (uint64_t)c->N * n_shared * (c->s1 + c->s2);
    if (n_shared && (!host || bytes != want))
      XFAIL(XPGB_ERR_CONTAINER_FORMAT, "shared payload is %llu bytes, expected %llu", (unsigned long long)bytes,
            (unsigned long long)want);
    CK(cudaDeviceSynchronize());
    if (c->shared_w) cudaFree(c->shared_w);
    c->shared_w = nullptr;
    c->S = n_shared;
    c->cap_T = 0;  // plan rows and group counts change
    ensure_work(c, 16, std::min(c->L, 8) + c->S);
    if (!n_shared) return;
    // device layout: every gate/up block, then every down block (one TMA map per kind)
    const int nb = c->N * n_shared;
    CK(cudaMalloc(&c->shared_w, want));
    const uint8_t* src = static_cast<const uint8_t*>(host);
    for (int b = 0; b < nb; ++b) {
      CK(cudaMemcpy(c->shared_w + (uint64_t)b * c->s1, src + (uint64_t)b * (c->s1 + c->s2), c->s1,
                    cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->shared_w + (uint64_t)nb * c->s1 + (uint64_t)b * c->s2, src + (uint64_t)b * (c->s1 + c->s2) + c->s1,
                    c->s2, cudaMemcpyHostToDevice));
    }
    c->map_gu_sh = make_map(c->shared_w, (uint64_t)nb * 2 * c->F, c->H, kBM);
    c->map_dn_sh = make_map(c->shared_w + (uint64_t)nb * c->s1, (uint64_t)nb * c->H, c->F, kBM);
  });
}

int xpgb_set_shared_tokens(xpgb_ctx* h, int32_t first, int32_t count) {
  return guard([&] {
    Ctx* c = &h->c;
    if (first < 0) XFAIL(XPGB_ERR_OUT_OF_RANGE, "shared token range starts at %d", first);
    c->sh0 = first;
    c->sh1 = count < 0 ? 0x7fffffff : first + count;
  });
}

int xpgb_route(uint64_t seed, int32_t layer_first, int32_t layer_count, int32_t tokens, int32_t num_experts,
               int32_t top_k, int32_t* out_dev, void* stream) {
  return guard([&] {
    if (num_experts < 1 || num_experts > kMaxExperts)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "num_experts %d outside [1, %d]", num_experts, kMaxExperts);
    if (top_k < 1 || std::min(top_k, num_experts) > kMaxTopK)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "top_k %d outside [1, %d]", top_k, kMaxTopK);
    launch_route(seed, layer_first, layer_count, tokens, num_experts, top_k, out_dev, (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_layer_forward(xpgb_ctx* h, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens, int32_t top_k,
                       uint64_t router_seed, void* stream) {
  return guard([&] {
    Ctx* c = &h->c;
    if (layer < 1 || layer > c->N) XFAIL(XPGB_ERR_OUT_OF_RANGE, "layer %d outside [1, %d]", layer, c->N);
    if (top_k < 1) XFAIL(XPGB_ERR_OUT_OF_RANGE, "top_k must be >= 1");
    enqueue_layer(c, layer, x_dev, y_dev, tokens, top_k, router_seed, (cudaStream_t)stream);
  });
}

int xpgb_fault_get(xpgb_ctx* h, int32_t* faulted, char* msg, uint64_t cap) {
  return guard([&] {
    long long fw = 0;
    CK(cudaMemcpy(&fw, h->c.d_fault, sizeof(fw), cudaMemcpyDeviceToHost));
    *faulted = fw != 0;
    if (msg && cap) {
      std::string m;
      if (fw) {
        const int kind = (int)((fw >> 1) & 3), state = (int)((fw >> 3) & 7), expert = (int)((fw >> 8) & 0xFFFFFF),
                  layer = (int)(fw >> 32);
        if (kind == 3)  // an expert-parallel peer event (ep_p2p.cuh: ep_fault)
          m = fmt("expert-parallel peer rank %d %s", expert - 1,
                  state == 1 ? "faulted: its rows of this step are invalid" : "published no epoch within 20 s");
        else
          m = fmt("read through %s while %s", tid_str(layer, expert, kind).c_str(), state_name(state));
      }
      const size_t n = std::min<size_t>(m.size(), cap - 1);
      memcpy(msg, m.data(), n);
      msg[n] = 0;
    }
  });
}
int xpgb_fault_clear(xpgb_ctx* h) {
  return guard([&] { CK(cudaMemset(h->c.d_fault, 0, sizeof(long long))); });
}

int xpgb_run(xpgb_ctx* h, const xpgb_run_opts* opts, const float* x_dev, float* y_dev, xpgb_report* rep) {
  return guard([&] {
    if (!opts || !rep) XFAIL(XPGB_ERR, "null argument");
    run_impl(&h->c, opts, x_dev, y_dev, rep);
  });
}

int xpgb_session_begin(xpgb_ctx* h, const xpgb_run_opts* opts, float* acts_dev) {
  return guard([&] {
    if (!opts) XFAIL(XPGB_ERR, "null argument");
    session_begin(&h->c, opts, acts_dev);
  });
}
int xpgb_session_materialize(xpgb_ctx* h, int32_t step) {
  return guard([&] {
    try {
      session_materialize(&h->c, step);
    } catch (...) {
      session_abort(&h->c);
      throw;
    }
  });
}
int xpgb_session_acquire(xpgb_ctx* h, int32_t step, void* stream) {
  return guard([&] { session_acquire(&h->c, step, (cudaStream_t)stream); });
}
int xpgb_session_compute(xpgb_ctx* h, int32_t step) {
  return guard([&] {
    if (!session_of(&h->c).rs.acts) XFAIL(XPGB_ERR, "session has no activation buffer for built-in compute");
    session_compute(&h->c, step);
  });
}
int xpgb_session_release(xpgb_ctx* h, int32_t step, void* stream) {
  return guard([&] { session_release(&h->c, step, (cudaStream_t)stream); });
}
int xpgb_session_run_steps(xpgb_ctx* h, int32_t first, int32_t count, void* stream) {
  return guard([&] {
    Ctx* c = &h->c;
    if (!session_of(c).rs.acts) XFAIL(XPGB_ERR, "session has no activation buffer for built-in compute");
    if (count < 0) XFAIL(XPGB_ERR_OUT_OF_RANGE, "step count %d", count);
    try {
      for (int32_t g = first; g < first + count; ++g) {
        session_acquire(c, g, (cudaStream_t)stream);
        session_compute(c, g);
        session_release(c, g, (cudaStream_t)stream);
        session_materialize(c, g + 2);
      }
    } catch (...) {
      session_abort(c);
      throw;
    }
  });
}
int xpgb_session_end(xpgb_ctx* h, xpgb_report* rep) {
  return guard([&] {
    if (!rep) XFAIL(XPGB_ERR, "null argument");
    session_end(&h->c, rep);
  });
}
int xpgb_session_abort(xpgb_ctx* h) {
  return guard([&] { session_abort(&h->c); });
}
int xpgb_session_step(xpgb_ctx* h, int32_t step, int32_t* info) {
  return guard([&] {
    Session& ss = session_of(&h->c);
    if (!ss.active) XFAIL(XPGB_ERR, "no active session");
    if (step < 0 || step >= ss.steps) XFAIL(XPGB_ERR_OUT_OF_RANGE, "step %d outside [0, %d)", step, ss.steps);
    const Step& st = ss.sv[step];
    const int v[7] = {st.it, st.layer, st.w, st.e0, std::min(st.e1, h->c.E), st.first ? 1 : 0, st.last ? 1 : 0};
    memcpy(info, v, sizeof(v));
  });
}

int xpgb_session_info(xpgb_ctx* h, int32_t* steps_total, int32_t* steps_per_iteration, void** compute_stream) {
  return guard([&] {
    Session& ss = session_of(&h->c);
    if (!ss.active) XFAIL(XPGB_ERR, "no active session");
    if (steps_total) *steps_total = ss.steps;
    if (steps_per_iteration) *steps_per_iteration = ss.steps / std::max(1, ss.o.iterations);
    if (compute_stream) *compute_stream = (void*)h->c.s_comp;
  });
}

int xpgb_log_get(xpgb_ctx* h, xpgb_record* out, int32_t cap, int32_t* n) {
  return guard([&] {
    const auto& l = h->c.last_log;
    *n = (int32_t)l.size();
    if (out) memcpy(out, l.data(), std::min<size_t>(cap, l.size()) * sizeof(xpgb_record));
  });
}

int xpgb_set_expert_shard(xpgb_ctx* h, int32_t expert_first, int32_t expert_count) {
  return guard([&] {
    Ctx* c = &h->c;
    if (expert_first < 0 || expert_count < 1 || expert_first + expert_count > c->L)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "shard [%d, %d) outside [0, %d)", expert_first, expert_first + expert_count, c->L);
    CK(cudaDeviceSynchronize());
    if (c->host && c->host_owned) cudaFreeHost(c->host);
    if (c->host && c->host_registered) cudaHostUnregister(c->host);
    c->host = nullptr;
    c->host_owned = c->host_registered = false;
    c->e_first = expert_first;
    c->E = expert_count;
    c->cap_T = 0;  // force workspace re-creation with the new expert count
    init_pools(c);
    ensure_work(c, 16, std::min(c->L, 8) + c->S);
  });
}

static void experts_forward_range(Ctx* c, int layer, const void* rows_dev, long long lo_rows,
                                  const int32_t* offsets_dev, int n_rows, int e0, int e1, bool reduce, float* out_dev,
                                  cudaStream_t s) {
  if (layer < 1 || layer > c->N) XFAIL(XPGB_ERR_OUT_OF_RANGE, "layer %d outside [1, %d]", layer, c->N);
  if (e0 < 0 || e1 > c->E || e0 >= e1) XFAIL(XPGB_ERR_OUT_OF_RANGE, "expert range [%d, %d) outside [0, %d)", e0, e1, c->E);
  if (n_rows < 0 || n_rows > lo_rows)
    XFAIL(XPGB_ERR_OUT_OF_RANGE, "%d rows do not fit the %lld-row planes of the row buffer", n_rows, lo_rows);
  if (n_rows > c->cap_rows || !c->xp) ensure_work(c, std::max(n_rows, 1), 1);
  if (n_rows == 0) return;
  // the GEMMs read the caller's rows in place ([2][lo_rows][H]: hi plane, lo plane) through
  // tensor maps built once per buffer -- no copy into the context
  if (rows_dev != c->ep_rows_ptr || lo_rows != c->ep_lo_rows) {
    c->map_ep_x = make_map(rows_dev, 2 * lo_rows, c->H, kBoxRowsB);
    c->map_ep_x_pair = make_map(rows_dev, 2 * lo_rows, c->H, kBM);
    c->ep_rows_ptr = rows_dev;
    c->ep_lo_rows = lo_rows;
  }
  // rows per expert: under a session the expected share of the global batch (n_rows may be
  // an upper bound when the row count lives on the device), else n_rows spread evenly
  double per_group = (double)n_rows / std::max(1, c->E);
  int n_est = n_rows;
  if (c->sess && c->sess->active) {
    per_group = (double)c->sess->o.tokens * std::min(c->sess->o.top_k, c->L) / c->L;
    n_est = std::max(1, std::min(n_rows, (int)std::ceil(per_group * c->E)));
  }
  const int bn = pick_bn_rows(per_group);
  // an EP owner receives every rank's rows for its experts: groups of >= 128 rows run on
  // CTA pairs, exactly as in enqueue_window
  const bool pair = pair_gemm_supported(c->H, c->F) && (c->pair_mode == 1 || (c->pair_mode < 0 && per_group >= 128.0));
  // same for every window of the layer; the planes are n_rows apart, so part_rows bounds them
  const int splits = pair ? 1
                          : std::max(1, std::min<int>(pick_splits(c, n_est, 1, bn),
                                                      (int)(c->part_rows / std::max(1, n_rows))));
  GemmParams pg = gemm_params(c, layer, 1, offsets_dev, 1, false), pd = gemm_params(c, layer, 2, offsets_dev, splits, false);
  pg.act_lo_rows = lo_rows;  // x rows: the caller's planes; h rows: the context's
  pd.split_stride = (long long)n_rows * c->H;
  for (GemmParams* p : {&pg, &pd}) {  // window: groups [e0, e1), rows stay absolute
    p->offsets += e0;
    p->pt += e0;
    p->e_first += e0;
    p->E = p->E_routed = e1 - e0;
  }
  if (pair)
    launch_gemm_pair(true, c->map_ep_x_pair, c->map_gu, c->map_gu, pg, c->num_sms, s, c->pair_split);
  else
    launch_gate_up(c->map_gu, c->map_ep_x, c->map_gu, pg, bn, c->num_sms, s, lean_gemm(c));
  CKLAUNCH();
  if (pair)
    launch_gemm_pair(false, c->map_h_pair, c->map_dn, c->map_dn, pd, c->num_sms, s, c->pair_split);
  else
    launch_down(c->map_dn, c->map_h, c->map_dn, pd, bn, c->num_sms, s, lean_gemm(c));
  CKLAUNCH();
  c->ep_splits = splits;  // for a fused reduce + combine scatter (xpgb_ep_reduce_scatter)
  c->ep_split_stride = pd.split_stride;
  c->ep_rows = n_rows;
  if (reduce) {  // after the layer's last window: every row's split-K partials are final
    launch_reduce_rows(c->part, c->d_fault, out_dev, n_rows, c->H, splits, pd.split_stride, s);
    CKLAUNCH();
  }
}

int xpgb_experts_forward(xpgb_ctx* h, int32_t layer, const void* rows_dev, int64_t lo_rows,
                         const int32_t* offsets_dev, int32_t n_rows, float* out_dev, void* stream) {
  return guard([&] {
    experts_forward_range(&h->c, layer, rows_dev, lo_rows, offsets_dev, n_rows, 0, h->c.E, true, out_dev,
                          (cudaStream_t)stream);
  });
}

int xpgb_experts_forward_range(xpgb_ctx* h, int32_t layer, const void* rows_dev, int64_t lo_rows,
                               const int32_t* offsets_dev, int32_t n_rows, int32_t e0, int32_t e1, int32_t reduce,
                               float* out_dev, void* stream) {
  return guard([&] {
    experts_forward_range(&h->c, layer, rows_dev, lo_rows, offsets_dev, n_rows, e0, std::min(e1, h->c.E),
                          reduce != 0, out_dev, (cudaStream_t)stream);
  });
}

int xpgb_shared_forward(xpgb_ctx* h, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens, void* stream) {
  return guard([&] {
    Ctx* c = &h->c;
    if (layer < 1 || layer > c->N) XFAIL(XPGB_ERR_OUT_OF_RANGE, "layer %d outside [1, %d]", layer, c->N);
    if (!c->S || tokens <= 0) return;
    cudaStream_t s = (cudaStream_t)stream;
    const int S = c->S, T = tokens;
    if ((long long)T * S > c->cap_rows || !c->xp) ensure_work(c, T, S);
    // rows s*T + t hold token t for shared expert s; offsets [0, T, 2T, ...], written on the
    // stream (no host index, no synchronisation: this runs once per layer under EP)
    int32_t* d_pos = c->plan_pos[2];  // layer_forward's plan buffer doubles as scratch here
    int32_t* d_off = c->plan_off[2];
    launch_shared_plan(d_pos, d_off, T, S, s);
    CKLAUNCH();
    launch_gather(x_dev, d_pos, c->d_fault, c->xp, c->cap_rows, T, S, c->H, s);
    CKLAUNCH();
    const int bn = pick_bn_rows((double)T);
    GemmParams pg = gemm_params(c, layer, 1, d_off, 1), pd = gemm_params(c, layer, 2, d_off, 1);
    for (GemmParams* p : {&pg, &pd}) {  // only the shared groups
      p->E = S;
      p->E_routed = 0;
    }
    pd.split_stride = (long long)T * S * c->H;
    launch_gate_up(c->map_gu, c->map_xp, c->map_gu_sh, pg, bn, c->num_sms, s);
    CKLAUNCH();
    launch_down(c->map_dn, c->map_h, c->map_dn_sh, pd, bn, c->num_sms, s);
    CKLAUNCH();
    launch_combine(c->part, d_pos, c->d_fault, y_dev, T, S, 0, c->H, 1, pd.split_stride, 1.0f, nullptr, nullptr, 0, s,
                   true);
    CKLAUNCH();
  });
}

// ---------------------------------------------------------------- EP over peer memory
int xpgb_ep_window_alloc(uint64_t bytes, void** dptr, void* ipc_handle) {
  return guard([&] {
    CK(cudaMalloc(dptr, bytes));
    CK(cudaMemset(*dptr, 0, bytes));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, *dptr));
    memcpy(ipc_handle, &h, sizeof(h));
  });
}

int xpgb_ep_window_open(const void* ipc_handle, void** dptr) {
  return guard([&] {
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int xpgb_ep_window_close(void* dptr) {
  return guard([&] { CK(cudaIpcCloseMemHandle(dptr)); });
}

int xpgb_ep_window_free(void* dptr) {
  return guard([&] { CK(cudaFree(dptr)); });
}

int xpgb_ep_scatter_rows(const float* src_dev, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                         int32_t n, const int32_t* n_dev, int32_t hidden, int32_t to_bf16, int64_t lo_rows,
                         void* const* peer_rows, int32_t* const* peer_flags, int32_t world, int32_t rank, int32_t epoch,
                         const void* fault_dev, uint32_t* counter, void* stream) {
  return guard([&] {
    if (world < 1 || world > kMaxEpWorld || rank < 0 || rank >= world)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "rank %d of %d (at most %d ranks)", rank, world, kMaxEpWorld);
    if (hidden % 4) XFAIL(XPGB_ERR_OUT_OF_RANGE, "hidden_dim must be a multiple of 4");
    if (n < 0) XFAIL(XPGB_ERR_OUT_OF_RANGE, "negative row count");
    EpPeers peers{};
    peers.world = world;
    peers.rank = rank;
    for (int r = 0; r < world; ++r) {
      peers.rows[r] = peer_rows[r];
      peers.flags[r] = peer_flags[r];
    }
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    launch_ep_scatter(src_dev, src_rows, dst_rank, dst_row, n, n_dev, hidden, to_bf16 != 0, lo_rows, peers, epoch,
                      static_cast<const long long*>(fault_dev), counter, sms, (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_ep_reduce_scatter(xpgb_ctx* h, const int32_t* dst_rank, const int32_t* dst_row, int32_t n_rows,
                           const int32_t* n_dev, void* const* peer_rows, int32_t* const* peer_flags, int32_t world, int32_t rank,
                           int32_t epoch, uint32_t* counter, void* stream) {
  return guard([&] {
    Ctx* c = &h->c;
    if (world < 1 || world > kMaxEpWorld || rank < 0 || rank >= world)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "rank %d of %d (at most %d ranks)", rank, world, kMaxEpWorld);
    if (n_rows != c->ep_rows && n_rows > 0)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "%d rows, the last experts_forward_range computed %d", n_rows, c->ep_rows);
    EpPeers peers{};
    peers.world = world;
    peers.rank = rank;
    for (int r = 0; r < world; ++r) {
      peers.rows[r] = peer_rows[r];
      peers.flags[r] = peer_flags[r];
    }
    launch_ep_reduce_scatter(c->part, c->d_fault, c->ep_splits, c->ep_split_stride, dst_rank, dst_row, n_rows, n_dev,
                             c->H, peers, epoch, counter, c->num_sms, (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_ep_wait(const int32_t* flags_dev, int32_t world, int32_t epoch, void* fault_dev, void* stream) {
  return guard([&] {
    if (world < 1 || world > kMaxEpWorld) XFAIL(XPGB_ERR_OUT_OF_RANGE, "%d ranks (at most %d)", world, kMaxEpWorld);
    launch_ep_wait(flags_dev, world, epoch, static_cast<long long*>(fault_dev), (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int64_t xpgb_ep_plan_scratch_words(int32_t world, int32_t tokens, int32_t num_experts) {
  return ep_plan_scratch_words(world, tokens, num_experts);
}

int xpgb_ep_plan(const int32_t* routes_dev, int32_t tokens, int32_t world, int32_t rank, int32_t kk,
                 int32_t num_experts, int32_t* scratch_dev, const xpgb_ep_plan_bufs* out, void* stream) {
  return guard([&] {
    if (world < 1 || world > kMaxEpWorld || rank < 0 || rank >= world)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "rank %d of %d (at most %d ranks)", rank, world, kMaxEpWorld);
    if (kk < 1 || kk > num_experts || num_experts < world || tokens < 0)
      XFAIL(XPGB_ERR_OUT_OF_RANGE, "bad EP plan geometry (T=%d, kk=%d, L=%d, world=%d)", tokens, kk, num_experts, world);
    if (!out) XFAIL(XPGB_ERR, "null plan buffers");
    EpPlanOut o{out->src_rows, out->dst_rank, out->dst_row, out->ret_index, out->c_rank, out->c_row, out->to_arrival,
                out->from_arrival, out->offsets, out->counts};
    launch_ep_plan(routes_dev, tokens, world, rank, kk, num_experts, scratch_dev, o, (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_fault_set(xpgb_ctx* h, int64_t word) {
  return guard([&] {
    CK(cudaDeviceSynchronize());
    long long w = word;
    CK(cudaMemcpy(h->c.d_fault, &w, sizeof(w), cudaMemcpyHostToDevice));
  });
}

int xpgb_fault_ptr(xpgb_ctx* h, void** fault_dev) {
  return guard([&] {
    if (!fault_dev) XFAIL(XPGB_ERR, "null argument");
    *fault_dev = h->c.d_fault;
  });
}

int xpgb_combine_rows(const float* rows_dev, const int32_t* index_dev, int32_t tokens, int32_t kk, int32_t top_k,
                      int32_t hidden, float* y_dev, void* stream) {
  return guard([&] {
    if (hidden % 4) XFAIL(XPGB_ERR_OUT_OF_RANGE, "hidden_dim must be a multiple of 4");
    if (kk < 1 || kk > kMaxTopK || top_k < 1) XFAIL(XPGB_ERR_OUT_OF_RANGE, "kk %d outside [1, %d]", kk, kMaxTopK);
    static long long* zero = nullptr;
    if (!zero) {
      CK(cudaMalloc(&zero, sizeof(long long)));
      CK(cudaMemset(zero, 0, sizeof(long long)));
    }
    launch_combine(rows_dev, index_dev, zero, y_dev, tokens, kk, kk, hidden, 1, 0, (float)(1.0 / top_k), nullptr,
                   nullptr, 0, (cudaStream_t)stream);
    CKLAUNCH();
  });
}

int xpgb_profile_layer(xpgb_ctx* h, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens, int32_t top_k,
                       uint64_t router_seed, int32_t reps, xpgb_kernel_times* out) {
  return guard([&] {
    Ctx* c = &h->c;
    cudaStream_t s = c->s_comp;
    xpgb_kernel_times acc{};
    const int kt = slots_of(c, top_k);
    c->prof = true;
    for (int r = 0; r < std::max(1, reps); ++r) {
      enqueue_layer(c, layer, x_dev, y_dev, tokens, top_k, router_seed, s);
      CK(cudaStreamSynchronize(s));
      float ms[6];
      for (int i = 0; i < 6; ++i) CK(cudaEventElapsedTime(&ms[i], c->pev[i], c->pev[i + 1]));
      acc.plan_ns += ms[0] * 1e6;  // route + plan (one launch)
      acc.gather_ns += ms[1] * 1e6;
      acc.gate_up_ns += ms[3] * 1e6;
      acc.down_ns += ms[4] * 1e6;
      acc.combine_ns += ms[5] * 1e6;
    }
    c->prof = false;
    const double inv = 1.0 / std::max(1, reps);
    acc.route_ns *= inv; acc.plan_ns *= inv; acc.gather_ns *= inv;
    acc.gate_up_ns *= inv; acc.down_ns *= inv; acc.combine_ns *= inv;
    const int G = groups_of(c);
    std::vector<int32_t> offs(G + 1);
    CK(cudaMemcpy(offs.data(), c->plan_off[2] + (size_t)(layer - 1) * (G + 1), (G + 1) * 4,
                  cudaMemcpyDeviceToHost));
    long long active = 0, u1 = 0, u2 = 0;
    const int kk = std::min(top_k, c->L);
    const int bn = pick_bn(c, tokens, kk);
    for (int e = 0; e < G; ++e) {
      const int n = offs[e + 1] - offs[e];
      if (n <= 0) continue;
      ++active;
      u1 += (long long)((n + bn - 1) / bn) * ((c->F + kBM - 1) / kBM);
      const int bd = pick_bn_down(c, tokens, kk);
      u2 += (long long)((n + bd - 1) / bd) * ((c->H + kBM - 1) / kBM) * c->last_splits;
    }
    const long long pairs = offs[G];  // rows this device computes (local routed + shared)
    (void)kt;
    acc.gate_up_bytes = active * (long long)c->s1 + pairs * c->H * 2 + pairs * c->F * 2;
    acc.down_bytes = active * (long long)c->s2 + pairs * c->F * 2 + pairs * c->H * 4 * c->last_splits;
    acc.n_units_gate_up = (int32_t)u1;
    acc.n_units_down = (int32_t)u2;
    acc.down_splits = c->last_splits;
    c->last_times = acc;
    *out = acc;
  });
}

}  // extern "C"
