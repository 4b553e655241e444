/*
 * xpgb.h — C ABI of the B200-native expert-paging MoE layer (libxpgb.so).
 *
 * Drop-in boundary for the hot path of the reference package `xpg` 0.1.0
 * (/root/reference/pkg/src/xpg).  The reference has no FFI: its boundary is
 * duck-typed Python.  Every entry point below names the reference interface
 * it replaces (file:line); the Python host layer `paper_2604_02715_b200`
 * binds these with ctypes and re-exposes the reference's names.
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, ints.  Device pointers are
 *     `void*`/`float*` into CUDA global memory of the context's device;
 *     streams are `cudaStream_t` passed as `void*` (NULL = legacy stream).
 *   - Every function returns an xpgb_status; on failure a message is
 *     available from xpgb_last_error() (thread-local).
 *   - Ids follow the reference: layer in [1, N], expert in [1, L],
 *     kind 1 = GATE_UP (2F x H), kind 2 = DOWN (H x F), token index 0-based,
 *     block ids 1-based per kind.
 *   - One context per device; no hidden globals besides the error string.
 */
#ifndef XPGB_H_
#define XPGB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XPGB_ABI_VERSION 1

/* Status codes map 1:1 onto the reference exception tree (errors.py:4-74). */
typedef enum xpgb_status {
  XPGB_OK = 0,
  XPGB_ERR = 1,                    /* XpgError                */
  XPGB_ERR_OUT_OF_RANGE = 2,       /* OutOfRangeError         */
  XPGB_ERR_CONTAINER_FORMAT = 3,   /* ContainerFormatError    */
  XPGB_ERR_DOUBLE_MAP = 4,         /* DoubleMapError          */
  XPGB_ERR_POOL_EXHAUSTED = 5,     /* PoolExhaustedError      */
  XPGB_ERR_NOT_MAPPED = 6,         /* NotMappedError          */
  XPGB_ERR_PAGE_FAULT = 7,         /* PageFaultError          */
  XPGB_ERR_CAPACITY_EXCEEDED = 8,  /* CapacityExceededError   */
  XPGB_ERR_BACKEND_MISS = 9,       /* BackendMissError        */
  XPGB_ERR_INFEASIBLE_CONFIG = 10, /* InfeasibleConfigError   */
  XPGB_ERR_CONFIG = 11,            /* ConfigError             */
  XPGB_ERR_DEADLOCK = 12,          /* DeadlockError           */
  XPGB_ERR_CUDA = 13,              /* CUDA failure -> XpgError */
  XPGB_ERR_ODD_LENGTH = 14,        /* OddLengthError          */
  XPGB_ERR_EMPTY_HISTOGRAM = 15,   /* EmptyHistogramError     */
  XPGB_ERR_SYMBOL_NOT_IN_TABLE = 16, /* SymbolNotInTableError */
  XPGB_ERR_TRUNCATED_STREAM = 17,  /* TruncatedStreamError    */
  XPGB_ERR_INVALID_CODE = 18       /* InvalidCodeError        */
} xpgb_status;

/* Page states (paging.py:41-45). */
enum { XPGB_PAGE_UNMAPPED = 0, XPGB_PAGE_LOADING = 1, XPGB_PAGE_RESIDENT = 2, XPGB_PAGE_EVICTING = 3 };

/* Pool geometry of a context. */
enum {
  XPGB_POOL_RING = 0,     /* reference PageTable: 2 x L blocks per kind (paging.py:115-122) */
  XPGB_POOL_RESIDENT = 1  /* every tensor owns a block: resident_baseline (pipeline.py:216-230) */
};

/* ModelSpec (model.py:35-86).  H and F must be multiples of 8 (16-byte rows for TMA). */
typedef struct xpgb_spec {
  int32_t num_layers;        /* N >= 2 */
  int32_t experts_per_layer; /* L >= 1 */
  int32_t hidden_dim;        /* H */
  int32_t intermediate_dim;  /* F */
} xpgb_spec;

typedef struct xpgb_ctx xpgb_ctx;

/* Ordering-log record (pipeline.py:82-91); event codes below. */
enum {
  XPGB_EV_RECYCLE = 0,
  XPGB_EV_LOAD_START = 1,
  XPGB_EV_LOAD_DONE = 2,
  XPGB_EV_COMPUTE_START = 3,
  XPGB_EV_COMPUTE_DONE = 4,
  XPGB_EV_RUN_BEGIN = 5
};
typedef struct xpgb_record {
  int32_t t;                /* global order, from a device-side atomic counter */
  int32_t event;            /* XPGB_EV_* */
  int32_t iteration;
  int32_t layer;
  int32_t kind;             /* 1/2 for loads and recycles, -1 otherwise */
  int32_t target_iteration; /* recycle only, else -1 */
  int32_t target_layer;     /* recycle only, else -1 */
  int32_t group;            /* sub-layer ring window of the step (bits 0-15); recycles: the recycled
                               step's window in bits 16-31.  0 in the reference geometry. */
  int64_t wall_ns;          /* %globaltimer when the record was written */
} xpgb_record;

/* StreamedRunner.run options (pipeline.py:307-331, 403-483). */
typedef struct xpgb_run_opts {
  int32_t iterations;        /* >= 1 */
  int32_t tokens;            /* T (ForwardSpec.tokens_per_step) */
  int32_t top_k;             /* ForwardSpec.top_k */
  int32_t sequential;        /* 1: host-synchronous twin of mode="sequential"; 0: async streams ("threaded") */
  uint64_t router_seed;      /* ForwardSpec.router_seed reduced mod 2^64 */
  int32_t sabotage_iteration;/* (iteration, layer) whose RAW wait is skipped; 0 = none */
  int32_t sabotage_layer;
  const float* fetch_delay_s;   /* optional [N][L][2] seconds per tensor (delay_fn hook), host memory */
  const float* compute_delay_s; /* optional [iterations][N] seconds (compute_delay_fn hook), host memory */
  int32_t log_enable;        /* record the ordering log (default on) */
  int32_t profile;           /* 1: time every MoE kernel launch with CUDA events (report.kern_*,
                              * decoder / decode-into-GEMM stats); n >= 2: events around 1 in n
                              * decoder and decode-into-GEMM launches only (stats scaled to every
                              * launch; a light profile for timed runs -- use an odd n so both kinds
                              * are sampled) */
  int32_t fresh_inputs;      /* 1: every iteration starts from activations the caller wrote into acts_dev
                                (a serving session: step(acts) per decode step); 0: iteration i+1 consumes
                                iteration i's output, as run() does */
} xpgb_run_opts;

typedef struct xpgb_report {
  int64_t stall_ns;          /* compute stream blocked on RAW (RunReport.stall_seconds) */
  int64_t war_wait_ns;       /* copy streams blocked on WAR (RunReport.war_wait_seconds) */
  int64_t elapsed_ns;        /* first to last log record */
  int64_t arena_peak_bytes;  /* PageTable.arena_peak_bytes */
  int64_t h2d_bytes;         /* bytes paged in from the pinned host pool (wire bytes) */
  int64_t d2d_bytes;         /* raw bytes paged in from the device tier */
  int64_t copy_busy_ns[2];   /* per copy stream: sum of load-start..load-done spans */
  int32_t page_fault;        /* 1 if a compute read a non-resident page */
  int32_t n_records;
  /* opts.profile: mean device time per launch over the run (CUDA events on the compute stream) */
  double kern_gate_up_ns;
  double kern_down_ns;
  double kern_aux_ns;        /* plan + gather + combine per layer */
  int64_t gate_up_bytes;     /* mean algorithmic bytes per gate/up launch (weights of routed experts + rows) */
  int64_t down_bytes;
  int32_t down_splits;
  int32_t active_experts;    /* routed experts summed over the N layers of one iteration */
  int64_t decoded_bytes;     /* bf16 bytes produced by the GPU exponent decoder */
} xpgb_report;

/* ---------------------------------------------------------------- basics */
int xpgb_abi_version(void);
const char* xpgb_last_error(void);
/* Number of kernels this library launched since load (evidence counter). */
int64_t xpgb_kernel_launches(void);

/* Create a context on `device`.  pool = XPGB_POOL_RING (PageTable, paging.py:97-130)
 * or XPGB_POOL_RESIDENT (resident_baseline).  max_tokens sizes workspaces (grows lazily). */
int xpgb_create(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, xpgb_ctx** out);
/* Same, holding only experts [expert_first, expert_first + expert_count) of every layer from the
 * start (an expert-parallel rank): pools are sized for the shard, never for all L experts (a
 * DSv3 rank would otherwise allocate the whole 180 GB model transiently). */
int xpgb_create_shard(const xpgb_spec* spec, int32_t device, int32_t pool, int32_t max_tokens, int32_t expert_first,
                      int32_t expert_count, xpgb_ctx** out);
int xpgb_destroy(xpgb_ctx* ctx);
int xpgb_sync(xpgb_ctx* ctx);

/* ---------------------------------------------------------------- storage
 * WeightContainer payload (model.py:142-202) lives in a pinned host pool in
 * container order; StorageHierarchy.fetch (storage.py:228-243) copies from it. */
/* Exact-size pinned (page-locked, portable) host allocation, no context needed. */
int xpgb_pinned_alloc(uint64_t bytes, void** out);
int xpgb_pinned_free(void* ptr);
/* Container ingest (model.py:142-202 without the read copy): page-lock caller memory, e.g. an
 * mmap'd XPGW file, so the page-in DMAs straight from the page cache.  The range is widened to
 * whole pages; read_only = 1 for PROT_READ mappings (cudaHostRegisterReadOnly). */
int xpgb_host_register(void* ptr, uint64_t bytes, int32_t read_only);
int xpgb_host_unregister(void* ptr);
/* Allocate a pinned host pool of total_bytes; *host_ptr receives it for filling. */
int xpgb_host_pool_alloc(xpgb_ctx* ctx, void** host_ptr, uint64_t* bytes);
/* Use caller memory (cudaHostRegister'd here) as the host pool. */
int xpgb_host_pool_register(xpgb_ctx* ctx, void* host_ptr, uint64_t bytes);
/* Placement (plan_placement, storage.py:92-168): backend_of[((layer-1)*L + expert-1)*2 + kind-1]
 * = 0 host tier, 1 device tier.  Device-tier tensors are staged into HBM once, here. */
int xpgb_set_placement(xpgb_ctx* ctx, const uint8_t* backend_of);
/* StorageHierarchy.fetch: copy the exact sigma bytes of a tensor into dst (device memory) on stream. */
int xpgb_fetch(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, void* dst, uint64_t dst_bytes,
               void* stream);

/* ---------------------------------------------------------------- page table (paging.py:97-271) */
int xpgb_pt_map(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, int32_t* block_id);
int xpgb_pt_mark_resident(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind);
int xpgb_pt_unmap(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind);
int xpgb_pt_state(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, int32_t* state);
int xpgb_pt_block(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, int32_t* block_id);
int xpgb_pt_block_ptr(xpgb_ctx* ctx, int32_t kind, int32_t block_id, void** dptr, uint64_t* bytes);
int xpgb_pt_loading_view(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, void** dptr,
                         uint64_t* bytes);
/* read_page: copy a resident page's bytes to host memory (PageFault otherwise). */
int xpgb_pt_read(xpgb_ctx* ctx, int32_t layer, int32_t expert, int32_t kind, void* host_dst, uint64_t bytes);
int xpgb_pt_peak_bytes(xpgb_ctx* ctx, uint64_t* peak);
int xpgb_pt_pool_bytes(xpgb_ctx* ctx, uint64_t* bytes);
int xpgb_pt_check_consistency(xpgb_ctx* ctx);
/* Trace sink (paging.py:137-146): enable, then fetch newline-separated lines. */
int xpgb_pt_trace_enable(xpgb_ctx* ctx, int32_t enable);
int xpgb_pt_trace_get(xpgb_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed);
/* Map + fetch + mark_resident every tensor of the model (resident pools). */
int xpgb_make_resident(xpgb_ctx* ctx);

/* ---------------------------------------------------------------- exponent codec (codec.py:48-330)
 * Stream bytes are bit-identical to xpg's compress(); the chunk index (bit offset of every
 * `chunk`-value block) is B200 side metadata that lets the GPU decode one stream in parallel.
 * Packed record layout (all parts 16-byte aligned):
 *   [sign/mantissa plane: n][exponent stream: bits_len + 8 zero bytes][index: ceil(n/chunk) u32] */
int xpgb_codec_histogram(const void* data, uint64_t bytes, uint64_t* counts256, int32_t threads);
/* compress() of one tensor into caller buffers (host). */
int xpgb_codec_encode(const void* data, uint64_t bytes, const uint8_t* lengths256, void* sm_out, void* bits_out,
                      uint64_t bits_cap, uint64_t* bits_len, uint64_t* bit_count, uint32_t* index_out,
                      int32_t chunk);
/* Compress n_tensors consecutive tensors of a payload into packed records (multi-threaded,
 * host only).  out == NULL computes the layout only (pool_bytes, rec_offsets, bits_lens,
 * bit_counts: [n_tensors]); otherwise out (>= pool_bytes) receives the records.
 * place_order (nullable = payload order) lists tensor indices in the order their records
 * are laid out in the pool; the runtime stages runs of consecutive records with one copy,
 * so (layer, kind, expert) order lets a layer's small records travel together. */
int xpgb_codec_pack(const void* payload, int32_t n_tensors, const uint64_t* value_counts, const uint8_t* lengths256,
                    int32_t chunk, int32_t threads, const int32_t* place_order, void* out, uint64_t out_cap,
                    uint64_t* pool_bytes, uint64_t* rec_offsets, uint64_t* bits_lens, uint64_t* bit_counts);
/* Byte size of a packed record. */
uint64_t xpgb_codec_record_bytes(uint64_t n, uint64_t bits_len, int32_t chunk);
/* Rebuild the chunk index of a stream on the host, validating it like decompress()
 * (consumed_bits, nullable: the exact exponent bit count the stream codes):
 * TruncatedStreamError / InvalidCodeError statuses (codec.py:304-327). */
int xpgb_codec_index(const void* bits, uint64_t bits_len, uint64_t n, const uint8_t* lengths256, int32_t chunk,
                     uint32_t* index_out, uint64_t* consumed_bits);
/* decompress() on the GPU: packed record in device memory -> n bf16 words at out_dev. */
int xpgb_codec_decode(const void* record_dev, uint64_t n, uint64_t bits_len, int32_t chunk,
                      const uint8_t* lengths256, void* out_dev, void* stream);
/* FX4 records (B200 addition, fx4.cuh): a fixed-width exponent format for the compressed device
 * tier -- 4-bit offsets from a per-tensor base, escapes for exponents outside the 15-wide
 * window -- that the decode-into-GEMM kernel expands without a serial decode chain; lossless
 * like the exponent-Huffman record (codec.py:235-272), 12.1 bits per value instead of ~10.7.
 * n % 256 == 0.  measure: histogram -> base and escape count -> record bytes (synchronises
 * `stream`); encode: raw bf16 (device) -> record (device, record_bytes); decode: record ->
 * n bf16 words; base in [0, 240] (measure picks it).  scratch: xpgb_fx4_scratch_bytes(n) bytes of
 * device memory. */
uint64_t xpgb_fx4_scratch_bytes(uint64_t n);
int xpgb_fx4_measure(const void* raw_dev, uint64_t n, void* scratch_dev, int32_t* base, uint64_t* n_escapes,
                     uint64_t* record_bytes, void* stream);
int xpgb_fx4_encode(const void* raw_dev, uint64_t n, int32_t base, void* scratch_dev, void* record_dev, void* stream);
int xpgb_fx4_decode(const void* record_dev, uint64_t n, int32_t base, void* out_dev, void* stream);
/* Attach a packed model (records in container order, tensors of this context's shard) to the
 * context.  Device-tier tensors are then held compressed in HBM and decoded into ring blocks
 * (the reference's compressed device tier, storage.py:235-238); with host_compressed = 1 the
 * host tier also ships compressed records over PCIe and decodes them on the GPU. */
int xpgb_set_codec(xpgb_ctx* ctx, const void* pool, uint64_t pool_bytes, const uint64_t* rec_offsets,
                   const uint64_t* bits_lens, const uint8_t* lengths256, int32_t chunk, int32_t host_compressed);

/* Residency tier x > 0: experts with pinned_of[(layer-1)*L + expert-1]
 * = 1 stay RESIDENT in dedicated blocks for the context's lifetime; the schedule streams only the
 * others through a ring of 2 x (most streamed experts of any layer) blocks per kind.  Re-creates
 * the arena (no session may be active).  All-zero = the reference geometry. */
int xpgb_set_pinned(xpgb_ctx* ctx, const uint8_t* pinned_of);
/* Sub-layer ring (budgets below two layers, an extension of the reference): cap the ring at
 * ring_experts blocks per kind (>= 2; -1 = the reference's two layers).  A layer whose streamed
 * experts exceed ring_experts/2 is then scheduled as windows of ring_experts/2 streamed experts,
 * double-buffered in the two halves of the ring: window w+2 recycles window w's blocks after its
 * compute event (the reference's WAR rule one window at a time), each window's GEMMs read only
 * its experts, and the layer's combine runs after its last window.  Re-creates the arena. */
int xpgb_set_ring_experts(xpgb_ctx* ctx, int32_t ring_experts);
/* Windows in flight on a sub-layer ring (1..6, default 2 = double buffering; 1 = the next
 * window's decode waits for this window's compute, the link still runs ahead through the
 * staging ring): the ring's
 * ring_experts blocks per kind hold `depth` windows of ring_experts/depth experts, and window
 * g recycles window g-depth, so the loads of the next depth-1 windows overlap the compute of
 * the current one (the reference's two-layer WAR rule, generalised).  Callers keep the
 * reference's order -- materialize(0), materialize(1), materialize(g+2) after release(g) --
 * and the session materializes up to g+depth.  Ignored without a ring cap.  Re-creates the
 * arena. */
int xpgb_set_ring_depth(xpgb_ctx* ctx, int32_t depth);
/* Decode-into-GEMM (B200 addition to the compressed device tier, storage.py:143-168): mode 1
 * makes the builtin compute (xpgb_run, xpgb_session_compute) read device-tier experts'
 * records in place -- decoder warps inside the grouped GEMM expand them into the tensor-core
 * operand tiles -- instead of decoding each into its ring block first; the page table, the
 * ordering log and the results are unchanged (bit-identical).  Applies to decode-sized expert
 * groups (the 1-CTA GEMMs) when K of both projections is a multiple of the codec chunk.  Mode 0
 * (default) keeps every expert in the ring, as callers with their own compute need
 * (xpgb_experts_forward_range).  Mode 2 reads only FX4 records in place and decodes
 * exponent-Huffman device-tier records into the ring (a mixed device tier, where the Huffman
 * decoder's serial chain makes in-place decoding slower than decode-into-ring).  No session may
 * be active. */
int xpgb_set_fused_decode(xpgb_ctx* ctx, int32_t mode);
/* Activation planes the decode-sized (1-CTA) grouped GEMMs multiply: 2 (default) = the bf16 hi
 * and lo planes of every fp32 activation (fp32-like products: per-layer rel-L2 ~1e-5..5e-5 vs the
 * reference's fp32 forward), 1 = the hi plane only (bf16 activations: half the MMAs and half the
 * activation traffic; rel-L2 ~3e-3, inside the 1e-2 tolerance).  Streamed and resident runs of one
 * setting stay bit-identical; the CTA-pair prefill GEMMs always use both planes.  No session may
 * be active. */
int xpgb_set_activation_planes(xpgb_ctx* ctx, int32_t planes);
/* Record format of the compressed device tier: 0 = exponent-Huffman (default; the host pool's
 * records staged as they are, the reference's device tier, storage.py:143-168), 1 = FX4
 * (fx4.cuh; encoded on the GPU from the raw host pool when staged).  FX4 costs ~13% more HBM per
 * expert and decodes without a serial chain, so the decode-into-GEMM kernel runs near the
 * bandwidth of its compressed bytes.  Lossless either way.  Re-stages the device tier; no
 * session may be active. */
int xpgb_set_device_format(xpgb_ctx* ctx, int32_t fmt);
/* Per-tensor record format of the compressed device tier: formats[(layer * E + expert) * 2 +
 * kind] (kind 0 = gate/up, 1 = down), each 0 or 1 as in xpgb_set_device_format.  A mixed tier
 * lets a budget keep every streamed expert on the device tier -- FX4 for as many as fit, the
 * denser Huffman records for the rest -- instead of pushing the remainder to the host tier.
 * Entries of tensors not on the device tier are kept for when they are placed there.  Re-stages
 * the device tier; no session may be active. */
int xpgb_set_device_formats(xpgb_ctx* ctx, const uint8_t* formats);
/* Staging ring and device-resident chunk index of the compressed host tier: 1 allocates them
 * (the default once xpgb_set_codec(host_compressed = 1) ran), 0 releases them when the placement
 * leaves no tensor on the host tier (a budget plan that keeps every streamed expert on the device
 * tier gives that HBM back); a host-tier record streamed without them fails loudly. */
int xpgb_set_host_staging(xpgb_ctx* ctx, int32_t on);
/* Race hardening (debug; no reference counterpart -- the reference's sabotage control,
 * pipeline.py:369-370, covers RAW only).  poison != 0: every ring block a window maps is filled
 * with 0xFF bytes (bf16 NaN) on the copy stream before its load, so a GEMM that reads a block
 * whose load has not landed, or that a later window already recycled, produces NaNs.
 * skip_war_iteration/layer (0 = none): the load of that (iteration, layer) skips its WAR wait on
 * the compute of the step it recycles -- the WAR twin of opts.sabotage_iteration/layer.  No
 * session may be active. */
int xpgb_set_hazard_checks(xpgb_ctx* ctx, int32_t poison, int32_t skip_war_iteration, int32_t skip_war_layer);
/* Staging ring of the compressed host tier: n_buffers (2..16, default 4) buffers per kind of
 * min(largest record, 64 MB).  A staged copy waits only for its buffer's previous decode, never
 * for the arena's WAR event, so the link runs n_buffers-1 pieces ahead of the decoder -- across
 * device-tier windows that need no link at all.  Counted in xpgb_hbm_bytes' staging.  No session
 * may be active. */
int xpgb_set_stage_buffers(xpgb_ctx* ctx, int32_t n_buffers);
/* Exponent-decoder launches of the last run with opts.profile set: how many, their summed
 * device time (events on each launch's own decode stream) and their algorithmic bytes
 * (sign/mantissa + bitstream + chunk index read, bf16 written).  Zeros without profile. */
int xpgb_decode_stats(xpgb_ctx* ctx, int64_t* launches, double* kernel_ns, int64_t* algo_bytes);
/* Decode-into-GEMM launches of the last run with opts.profile set: how many, their summed device
 * time (events on the compute stream around each launch) and the compressed record bytes they
 * read in place.  Zeros without profile or without fused launches. */
int xpgb_fused_stats(xpgb_ctx* ctx, int64_t* launches, double* kernel_ns, int64_t* record_bytes);
/* Shared experts (DeepSeek-V3 style; absent from the reference, our convention): n_shared
 * always-on experts per layer that every token passes through after its routed experts,
 * weight 1.0 (the routed sum keeps its f32(1/top_k) scale).  host = N*n_shared*(sigma1+sigma2)
 * bytes in (layer, shared expert, kind) order; they stay resident in HBM and are never paged.
 * n_shared = 0 removes them.  Single-device contexts only (not the expert-parallel path). */
int xpgb_set_shared(xpgb_ctx* ctx, const void* host, uint64_t bytes, int32_t n_shared);
/* Step rows [first, first+count) pass through the shared experts (count < 0: every row, the
 * default).  An expert-parallel rank that also plans the other ranks' rows (global batch)
 * applies its replica of the shared experts to its own rows only. */
int xpgb_set_shared_tokens(xpgb_ctx* ctx, int32_t first, int32_t count);
/* Expert-weight HBM footprint of a context: ring/pool blocks (+ shared experts), codec
 * staging, device tier. */
int xpgb_hbm_bytes(xpgb_ctx* ctx, uint64_t* ring, uint64_t* staging, uint64_t* device_tier);

/* ---------------------------------------------------------------- compute */
/* routed_experts (pipeline.py:154-170) for layers [layer_first, layer_first+layer_count):
 * out_dev int32 [layer_count][T][min(top_k, L)], ascending 1-based ids. Stateless. */
int xpgb_route(uint64_t seed, int32_t layer_first, int32_t layer_count, int32_t tokens, int32_t num_experts,
               int32_t top_k, int32_t* out_dev, void* stream);
/* layer_forward (pipeline.py:192-208) through the device page table: every
 * routed expert of `layer` must be RESIDENT (else a page fault is recorded). */
int xpgb_layer_forward(xpgb_ctx* ctx, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens,
                       int32_t top_k, uint64_t router_seed, void* stream);
/* Device fault word: 0 = clean; fills a message like PageFaultError's. */
int xpgb_fault_get(xpgb_ctx* ctx, int32_t* faulted, char* msg, uint64_t cap);
int xpgb_fault_clear(xpgb_ctx* ctx);

/* ---------------------------------------------------------------- schedule (pipeline.py:299-483) */
/* StreamedRunner.run: x_dev/y_dev are [T][H] fp32 device buffers (y may alias x). */
int xpgb_run(xpgb_ctx* ctx, const xpgb_run_opts* opts, const float* x_dev, float* y_dev, xpgb_report* rep);
/* The same schedule one step at a time, so the compute of a step can be external
 * (e.g. expert-parallel dispatch/GEMM/combine over NCCL).  Step g = (iteration-1)*N + layer-1.
 * Order: begin; materialize(0); materialize(1); for g: acquire(g, s); <compute on s>;
 * release(g, s); materialize(g+2); end.  acts_dev (fp32 [T][H]) enables session_compute. */
int xpgb_session_begin(xpgb_ctx* ctx, const xpgb_run_opts* opts, float* acts_dev);
int xpgb_session_materialize(xpgb_ctx* ctx, int32_t step);  /* _materialize, pipeline.py:335-360 */
int xpgb_session_acquire(xpgb_ctx* ctx, int32_t step, void* stream); /* RAW wait + compute-start */
int xpgb_session_compute(xpgb_ctx* ctx, int32_t step);      /* built-in layer_forward of the step */
int xpgb_session_release(xpgb_ctx* ctx, int32_t step, void* stream); /* compute-done + WAR event */
/* Steps first .. first+count-1 with the built-in compute, each as acquire(g, s); compute(g);
 * release(g, s); materialize(g+2) -- one call per served iteration instead of four per step
 * (the host enqueue sits between a step's output readback and the next step's first kernels). */
int xpgb_session_run_steps(xpgb_ctx* ctx, int32_t first, int32_t count, void* stream);
int xpgb_session_end(xpgb_ctx* ctx, xpgb_report* rep);
int xpgb_session_abort(xpgb_ctx* ctx);
/* Shape of the active session's schedule and the stream the built-in compute runs on (the
 * caller orders its own H2D/D2H of acts_dev on it).  steps_per_iteration = N in the reference
 * geometry, N x windows with a sub-layer ring. */
int xpgb_session_info(xpgb_ctx* ctx, int32_t* steps_total, int32_t* steps_per_iteration, void** compute_stream);
/* Step `step` of the active session: info[7] = {iteration, layer, window, first local expert,
 * end local expert (exclusive, routed experts only), first window of its layer (0/1), last (0/1)}. */
int xpgb_session_step(xpgb_ctx* ctx, int32_t step, int32_t* info);
/* Ordering log of the last run (OrderingLog.records, pipeline.py:94-116). */
int xpgb_log_get(xpgb_ctx* ctx, xpgb_record* out, int32_t cap, int32_t* n);

/* ---------------------------------------------------------------- expert-parallel building blocks
 * (no reference counterpart).  A context may own a contiguous expert
 * shard [expert_first, expert_first+expert_count) of every layer. */
int xpgb_set_expert_shard(xpgb_ctx* ctx, int32_t expert_first, int32_t expert_count);
/* Grouped SwiGLU over rows already grouped by local expert:
 * rows_dev bf16 [2][lo_rows][H] -- the rows' hi plane bf16_rn(x), then their lo plane
 * bf16_rn(x - hi) lo_rows rows later (the activations reach the tensor cores as both planes,
 * so the expert math runs on x to ~2^-17 relative, as the reference's float32 x) -- read in
 * place; offsets_dev int32 [expert_count+1] device row ranges (n_rows <= lo_rows is an upper
 * bound of offsets[expert_count]); out_dev fp32 [n_rows][H] (expert output, unscaled).
 * Pages must be resident. */
int xpgb_experts_forward(xpgb_ctx* ctx, int32_t layer, const void* rows_dev, int64_t lo_rows,
                         const int32_t* offsets_dev, int32_t n_rows, float* out_dev, void* stream);

/* Ordered combine (pipeline.py:198-207) of rows returned by the expert owners:
 * y[t] = sum_{s ascending} rows[index[t][s]] * f32(1/top_k); index < 0 skips the slot.
 * rows fp32 [*][hidden], index int32 [tokens][kk], kk = number of routed slots. */
/* Shared experts of one layer on caller rows (the expert-parallel path: every rank applies its
 * replica to its own tokens after the routed combine): y[t] += sum_s shared_s(x[t]) in fp32,
 * shared experts in ascending order, weight 1.  x, y: device fp32 [tokens][H]. */
int xpgb_shared_forward(xpgb_ctx* ctx, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens, void* stream);
/* ---------------------------------------------------------------- EP exchange over peer memory
 * (SURVEY §8(e) fusion target; no reference counterpart).  Each rank allocates one window
 * (cudaMalloc'd, zeroed, exported as a 64-byte CUDA IPC handle), the ranks swap handles and
 * open each other's windows (NVLink P2P; the same device works too).  A layer's dispatch and
 * combine are then one scatter kernel each: row i of src (src_rows[i], or i when src_rows is
 * null) goes to row dst_row[i] of rank dst_rank[i]'s region peer_rows[dst_rank[i]] -- bf16
 * when to_bf16, else f32 -- and the kernel's last CTA releases `epoch` into slot `rank` of
 * every rank's flag array peer_flags[r] (int32[16]).  xpgb_ep_wait makes `stream` wait
 * (acquire) until all `world` slots of this rank's flags reach `epoch`.  counter: a device
 * uint32, zero, private to the call site.  peer_rows/peer_flags are host arrays of device
 * pointers (this rank's own window included). */
int xpgb_ep_window_alloc(uint64_t bytes, void** dptr, void* ipc_handle64);
int xpgb_ep_window_open(const void* ipc_handle64, void** dptr);
int xpgb_ep_window_close(void* dptr);
int xpgb_ep_window_free(void* dptr);
/* to_bf16: the rows land as their two bf16 planes (hi at dst_row, lo at dst_row + lo_rows of
 * the region).  n_dev (nullable): device row count (n is then an upper bound).  fault_dev
 * (nullable, xpgb_fault_ptr): when this rank's fault word is set, no rows are written and
 * every peer's fault word (int32 at index 32 of its flag array) is raised before the release.
 * xpgb_ep_wait is bounded: after 20 s without an epoch, or when a peer raised this rank's
 * fault word, it sets fault_dev (a "peer" fault, reported by xpgb_fault_get) instead of
 * trapping -- the rank's later kernels skip and its report carries the fault. */
int xpgb_ep_scatter_rows(const float* src_dev, const int32_t* src_rows, const int32_t* dst_rank, const int32_t* dst_row,
                         int32_t n, const int32_t* n_dev, int32_t hidden, int32_t to_bf16, int64_t lo_rows,
                         void* const* peer_rows, int32_t* const* peer_flags, int32_t world, int32_t rank, int32_t epoch,
                         const void* fault_dev, uint32_t* counter, void* stream);
int xpgb_ep_wait(const int32_t* flags_dev, int32_t world, int32_t epoch, void* fault_dev, void* stream);
/* Device pointer of the context's fault word (int64; 0 = no fault). */
int xpgb_fault_ptr(xpgb_ctx* ctx, void** fault_dev);
/* Test hook: overwrite the fault word (0 clears it; any other value makes the context's
 * kernels skip as after a page fault). */
int xpgb_fault_set(xpgb_ctx* ctx, int64_t word);
/* Per-step dispatch plan of one rank, built on the device from the global routing table
 * routes_dev int32 [world*tokens][kk] (xpgb_route's output: 1-based ids ascending per row) --
 * one launch, no host round trip, recomputed every step as the reference routes every forward
 * (pipeline.py:200-203).  Row positions follow expert_parallel.build_plan's canonical orders
 * (send order (owner, expert, token); expert-major order (expert, global token)); experts are
 * sharded contiguously and balanced (shard_bounds).  Buffers (device int32): src_rows,
 * dst_rank, dst_row, ret_index [tokens*kk]; c_rank, c_row, to_arrival, from_arrival
 * [world*tokens*kk] (n_own used); offsets [count+1]; counts [2*world+1] = rows sent to each
 * rank, rows received from each rank, n_own.  scratch_dev: xpgb_ep_plan_scratch_words int32. */
typedef struct xpgb_ep_plan_bufs {
  int32_t *src_rows, *dst_rank, *dst_row, *ret_index, *c_rank, *c_row, *to_arrival, *from_arrival, *offsets, *counts;
} xpgb_ep_plan_bufs;
int64_t xpgb_ep_plan_scratch_words(int32_t world, int32_t tokens, int32_t num_experts);
int xpgb_ep_plan(const int32_t* routes_dev, int32_t tokens, int32_t world, int32_t rank, int32_t kk,
                 int32_t num_experts, int32_t* scratch_dev, const xpgb_ep_plan_bufs* out, void* stream);
/* The combine fused with the down projection's split-K reduction: after
 * xpgb_experts_forward_range(..., reduce = 0) over a layer's last window, each of the n_rows
 * expert-major output rows is summed from ctx's partial planes and stored straight into
 * dst_rank[i]'s region at row dst_row[i] (f32); the last CTA releases `epoch` like
 * xpgb_ep_scatter_rows.  n_rows must be the rows of that experts_forward_range call. */
int xpgb_ep_reduce_scatter(xpgb_ctx* ctx, const int32_t* dst_rank, const int32_t* dst_row, int32_t n_rows,
                           const int32_t* n_dev, void* const* peer_rows, int32_t* const* peer_flags, int32_t world, int32_t rank,
                           int32_t epoch, uint32_t* counter, void* stream);

/* One window of a layer on pre-grouped rows (layout as xpgb_experts_forward): GEMMs of local
 * experts [e0, e1) only (rows stay absolute); reduce = 1 on the layer's last window writes
 * every row's output (split-K partials of all windows are final by then). */
int xpgb_experts_forward_range(xpgb_ctx* ctx, int32_t layer, const void* rows_dev, int64_t lo_rows,
                               const int32_t* offsets_dev, int32_t n_rows, int32_t e0, int32_t e1, int32_t reduce,
                               float* out_dev, void* stream);
int xpgb_combine_rows(const float* rows_dev, const int32_t* index_dev, int32_t tokens, int32_t kk, int32_t top_k,
                      int32_t hidden, float* y_dev, void* stream);

/* Per-kernel device timing of the last layer_forward/run (ns, CUDA events). */
typedef struct xpgb_kernel_times {
  double route_ns, plan_ns, gather_ns, gate_up_ns, down_ns, combine_ns;
  int64_t gate_up_bytes, down_bytes;  /* algorithmic bytes of the last launch */
  int32_t down_splits, n_units_gate_up, n_units_down;
} xpgb_kernel_times;
int xpgb_profile_layer(xpgb_ctx* ctx, int32_t layer, const float* x_dev, float* y_dev, int32_t tokens,
                       int32_t top_k, uint64_t router_seed, int32_t reps, xpgb_kernel_times* out);

#ifdef __cplusplus
}
#endif
#endif /* XPGB_H_ */
