// Decode-into-GEMM: the grouped SwiGLU expert GEMM reading a device-tier expert's weights
// straight from its compressed record (exponent-Huffman, codec.py:235-272 stream + chunk
// index) instead of from a bf16 ring block.
//
// The paged path without this kernel expands every device-tier expert into the ring first
// (k_exp_decode2 writes 2 B/value, the GEMM's TMA reads them back: 4 B/value of HBM traffic
// on top of the ~1.34 B/value record) and runs the decoder and the GEMM as two launches that
// compete for the SMs.  Here eight decoder warps per CTA expand the record into the UMMA A
// tiles in shared memory, in the 128-byte-swizzled K-major layout TMA would have produced,
// and the tensor cores consume them from there: HBM sees only the record and the activations.
//
// Unit = (expert, 256 weight rows, <= BN token rows, K range).  gate/up: the 256 rows are
// 128 gate rows and the matching 128 up rows (accumulators d0 / d0+128, SwiGLU epilogue as
// k_moe_gemm); down: 256 consecutive rows of W_down in two 128-row accumulators, fp32
// split-K partials.  A split's K range starts on a chunk boundary, so a decoder thread
// enters its row's stream once per unit (one chunk-index read) and then decodes the row
// continuously across stages and chunks -- the stream of one tensor row is contiguous.
//
// Warps (480 threads, one CTA per SM):
//   0      TMA producer of the activation tiles (hi and lo planes, moe_kernels.cuh)
//   1      TMEM allocator + MMA issuer
//   2..5   epilogue (TMEM lanes 32*(w%4)..)
//   14     FX4 only: TMA producer of the compressed stages (sign/mantissa + nibble rows)
//   6..13  decoders: thread d owns weight row d of the unit (tile d>>7, tile row d&127);
//          per 64-value stage it decodes 32 exponent pairs through the 12-bit pair table
//          (codec_dev.cuh) and writes 8 x 16 B into its swizzled smem row, then
//          fence.proxy.async + one mbarrier arrive per warp.
// The "full" barrier of a stage completes on the TMA bytes of the activations plus the
// eight decoder-warp arrivals.  The prologue repeats read_page's residency check
// (paging.py:228-237) on every routed expert's slot-table entry, as k_moe_gemm does.
#include <cuda_bf16.h>

#include <cstdlib>

#include "codec_dev.cuh"
#include "fx4.cuh"
#include "launch_count.h"
#include "moe_kernels.cuh"
#include "ptx_sm100.cuh"

namespace xpgb {

namespace {

constexpr int kDecWarps = 8;
constexpr int kDecThreads = 192 + 32 * kDecWarps + 32;  // 480: + the FX4 compressed-stage producer warp
constexpr int kDecRows = 256;                      // weight rows per unit (two 128-row A tiles)
constexpr int kDecThreads_dec = 32 * kDecWarps;    // decoder threads
constexpr int kRingBytes = 256;                    // per decoder thread: four 64-byte stream blocks

// FMT 0 (exponent-Huffman): decoded stages + the pair table and per-thread stream rings.
// FMT 1 (FX4): decoded stages + CST compressed stages the TMA fills -- per stage the unit's
// 2 x 128 rows of 64 sign/mantissa bytes (64-B swizzle) and 32 nibble bytes (32-B swizzle).
constexpr int kFxSmTile = 128 * 64, kFxNibTile = 128 * 32;
constexpr int kFxFenceFlag = 1 << 30;  // FX4 launches: bit in `chunk` -> proxy fence before a slot release
constexpr int kFxSpinFlag = 1 << 29;   // FX4 launches: bit in `chunk` -> MMA and decoders spin (no backoff)
constexpr int kFxNoDecFlag = 1 << 28;  // FX4 launches, timing A/B only: skip the decode math (wrong results)

constexpr int kFxCStage = 2 * kFxSmTile + 2 * kFxNibTile;  // 24 KB
#ifndef XPGB_FX_MAX_CST
#define XPGB_FX_MAX_CST 4
#endif
constexpr int kFxMaxCst = XPGB_FX_MAX_CST;  // compressed stages with the A tiles in TMEM (the smem they free)

// FMT 2: FX4 records, the decoded A tiles written to tensor memory (tcgen05.st) instead of
// shared memory, and the MMAs read A from there: shared memory then carries only the compressed
// stages and the activations (the smem path moves ~216 KB per 64-K stage -- the MMAs alone read
// each A tile twice, hi and lo planes -- and bounds the kernel, r2_t47: 405 us per Mixtral gate/up
// launch with the decode math switched off, 553 us with it).
template <int BN, int STAGES, int FMT = 0>
struct DecCfg {
  static constexpr int A_BYTES = kBM * kBK * 2;             // one 128 x 64 bf16 tile
  static constexpr int B_BYTES = BN * kBK * 2;              // one activation plane
  static constexpr int B_OFF = FMT == 2 ? 0 : 2 * A_BYTES;  // activations after the A tiles (smem A)
  static constexpr int STAGE = B_OFF + 2 * B_BYTES;         // [two A tiles +] hi/lo activations
  static constexpr int TMEM_COLS = 512;                     // 2 accumulator stages x 256 columns
  // accumulator columns per stage and the second accumulator's offset (up / W_down rows 128..255);
  // FMT 2 packs them at BN and keeps columns 384..511 for 2 stages x 2 decoded A tiles x 32
  static constexpr int ACC_W = FMT == 2 ? 2 * BN : 256;
  static constexpr int UP_OFF = FMT == 2 ? BN : 128;
  static constexpr int A_COL = 384;
  static_assert(FMT != 2 || (4 * BN <= A_COL && STAGES == 2), "TMEM-A tiles: BN <= 96, two stages");
  // activation stages in shared memory: with the A tiles in TMEM (two stages there) the
  // activations get their own deeper ring, so a stage's TMA load is issued BST - 1 stages ahead
  // of its MMAs instead of one (with two shared stages the L2 latency of every activation load
  // sat in the MMA loop: r2_t54, no unit saturated -- DRAM 42%, L2 33%, issue 50%)
  static constexpr int BST = FMT == 2 ? 4 : STAGES;
  static constexpr int TAB_BYTES = FMT ? (2 * kMaxExperts + 4) * 4 : (3 * kMaxExperts + 8) * 4;  // s_off, s_up (+ flag)
  static constexpr int DEC_TAB =
      FMT ? 0 : (((1 << kPairBits) * 4 + 3 * (kCodecMaxLen + 1) * 4 + kCodecSymbols + 15) & ~15);
  static constexpr int RING = FMT ? 0 : kDecThreads_dec * kRingBytes;  // per-decoder-thread bitstream rings
  // compressed stages (FX4): as many as fit beside the decoded stages, 2..4
  static constexpr int CST_FIT = (227 * 1024 - 1024 - 256 - TAB_BYTES - BST * STAGE) / kFxCStage;
  static constexpr int CST_MAX = FMT == 2 ? kFxMaxCst : 4;
  static constexpr int CST = FMT ? (CST_FIT > CST_MAX ? CST_MAX : CST_FIT) : 0;
  static_assert(!FMT || CST >= 2, "FX4 decode-GEMM needs two compressed stages");
  static constexpr int BAR_OFF = BST * STAGE + CST * kFxCStage;          // barriers, then the tables
  static constexpr int SMEM = BAR_OFF + 1024 + 256 + TAB_BYTES + DEC_TAB + RING;
  static_assert(SMEM <= 227 * 1024, "decode-GEMM stages exceed 227 KB");
};

// Offset arithmetic on the shared pointer itself: a round trip through uintptr_t loses the
// address space, and every table read through the result becomes a generic LD instead of LDS.
__device__ __forceinline__ uint8_t* align_1k(uint8_t* p) {
  return p + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(p)) & 1023u)) & 1023u);
}

__device__ __forceinline__ float silu_d(float g) { return g * (1.0f / (1.0f + __expf(-g))); }

// Generic-proxy smem writes -> visible to the tensor cores' async proxy.
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void st_smem_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// mbarrier wait for the warps that only feed or drain the decoders (TMA, MMA, epilogue): they
// back off between polls, so their spinning does not take issue slots and LSU bandwidth from
// the decoder warps on the same SM (ncu: 50 M polls per launch, each reloading the barrier
// address from local memory).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}

// The handoffs on the per-stage critical path (decoders -> MMA -> decoders) poll without a
// backoff when `spin` is set: a sleeping waiter adds up to ~2 x 64 ns per stage.
__device__ __forceinline__ void mbar_wait_role(uint64_t* bar, uint32_t parity, bool spin) {
  if (spin) mbar_wait(bar, parity);
  else mbar_wait_backoff(bar, parity);
}

// Branch-free stream window over a per-thread shared-memory ring of four 64-byte blocks
// (cp.async, bypassing L1).  Every lane of a warp refills at its own time, so a refill behind
// a branch made nearly every warp execute both paths (ncu: the refill branch diverged in
// 99.8% of warp executions); here a refill is a handful of predicated instructions.  The
// ring is topped up once per quad (8 values <= 8 words): while the read position sits in
// block B, blocks B+1 and B+2 are complete and B+3 is in flight, so no read waits.
struct PWindow {
  uint64_t win;
  int p;
  uint32_t nxt;     // next stream word (raw)
  uint32_t wi;      // absolute ring word index of the word after nxt
  uint32_t blk;     // block the fetches have reached (the next to fetch)
  uint32_t base;    // smem address of this thread's ring
  uint32_t sw;      // chunk swizzle
  const uint8_t* g; // global address of block `blk`
  __device__ __forceinline__ uint32_t word(uint32_t w) const {
    return lds32(base + ((((w >> 2) & 15) ^ sw) << 4) + ((w & 3) << 2));
  }
  __device__ __forceinline__ void fetch_if(bool pred) {  // block `blk` into its slot, predicated
    const uint32_t slot = blk & 3;
    const uint32_t pr = pred ? 1u : 0u;
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i)
      asm volatile(
          "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(
              base + (((slot * 4 + i) ^ sw) << 4)),
          "l"(g + 16 * i), "r"(pr)
          : "memory");
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q cp.async.commit_group;\n}\n" ::"r"(pr) : "memory");
    g += pred ? 64 : 0;
    blk += pred ? 1 : 0;
  }
  __device__ __forceinline__ void init(const uint32_t* bits, uint32_t bitpos, uint32_t ring, uint32_t swz) {
    base = ring;
    sw = swz;
    blk = 0;
    const uintptr_t a = reinterpret_cast<uintptr_t>(bits + (bitpos >> 5));
    g = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(15));
    const uint32_t w0 = (uint32_t)((a >> 2) & 3);
    fetch_if(true);
    fetch_if(true);
    fetch_if(true);
    fetch_if(true);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // blocks 0..2 complete
    win = ((uint64_t)bswap32(word(w0)) << 32) | bswap32(word(w0 + 1));
    nxt = word(w0 + 2);
    wi = w0 + 3;
    p = (int)(bitpos & 31);
  }
  // once per quad: the read position entered block wi/16; keep blocks up to wi/16 + 3 fetched
  __device__ __forceinline__ void top_up() {
    const bool need = blk < (wi >> 4) + 4;
    fetch_if(need);
    uint32_t pr = need ? 1u : 0u;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q cp.async.wait_group 1;\n}\n" ::"r"(pr) : "memory");
  }
  __device__ __forceinline__ void refill() {
    const bool r = p >= 32;
    const uint64_t wn = (win << 32) | bswap32(nxt);
    uint32_t ld = nxt;
    const uint32_t addr = base + ((((wi >> 2) & 15) ^ sw) << 4) + ((wi & 3) << 2);
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}\n"
                 : "+r"(ld)
                 : "r"(addr), "r"(r ? 1u : 0u)
                 : "memory");
    win = r ? wn : win;
    p = r ? p - 32 : p;
    nxt = ld;
    wi += r ? 1u : 0u;
  }
  __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)((win << p) >> (64 - kPairBits)); }
};

__device__ __forceinline__ void ldg_v4(uint4& v, const uint4* p) {
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
}

struct DUnit {
  int e, m0, row_begin, n_rows, split;
};

// Unit u -> (expert, 256-row weight tile, token tile, split); s_up: unit prefix per group.
__device__ __forceinline__ DUnit dec_unit(int u, const int* s_up, const int* s_off, int E, int bn, int splits) {
  int lo = 0, hi = E;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_up[mid] <= u) lo = mid; else hi = mid;
  }
  DUnit r;
  r.e = lo;
  const int local = u - s_up[lo];
  const int n = s_off[lo + 1] - s_off[lo];
  const int nt_count = (n + bn - 1) / bn;
  const int m = local / (splits * nt_count);
  const int rem = local % (splits * nt_count);
  r.split = rem / nt_count;
  const int nt = rem % nt_count;
  r.m0 = m * (kDecRows / 2);  // gate/up: feature tile of 128 (gate + up rows); down: see caller
  r.row_begin = s_off[lo] + nt * bn;
  r.n_rows = min(bn, n - nt * bn);
  return r;
}

}  // namespace

template <bool GU, int BN, int STAGES, int FMT>
__global__ void __maxnreg__(128)  // 480 threads x 128 registers (448 x 144 was refused at launch)
    k_moe_gemm_dec(const __grid_constant__ CUtensorMap map_b, GemmParams p, const DecTables* __restrict__ tabs,
                   int chunk) {
  using C = DecCfg<BN, STAGES, FMT>;
  constexpr int RFMT = FMT == 2 ? 1 : FMT;  // record format
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_1k(smem_raw);
  uint8_t* cstage = smem + C::BST * C::STAGE;  // FX4 compressed stages (CST of them)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::BST;
  uint64_t* tfull = empty + C::BST;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;  // FX4: compressed stage filled (TMA bytes)
  uint64_t* cempty = cfull + kFxMaxCst;  // FX4: compressed stage read by all decoder warps
  uint64_t* afull = cempty + kFxMaxCst;  // FMT 2: decoded A stage in TMEM written (decoder warps)
  uint64_t* aempty = afull + 2;          // FMT 2: decoded A stage read by the MMAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);
  int* s_off = reinterpret_cast<int*>(smem + C::BAR_OFF + 256);
  int* s_up = s_off + kMaxExperts + 1;
  int* s_flag = s_up + kMaxExperts + 1;
  uint32_t* s_pair = reinterpret_cast<uint32_t*>(s_off + 3 * kMaxExperts + 8);  // Huffman only (FMT 0)
  uint32_t* s_first = s_pair + (1 << kPairBits);
  int* s_count = reinterpret_cast<int*>(s_first + kCodecMaxLen + 1);
  int* s_rank = s_count + kCodecMaxLen + 1;
  uint8_t* s_sym = reinterpret_cast<uint8_t*>(s_rank + kCodecMaxLen + 1);
  uint8_t* s_ring = smem + C::BAR_OFF + 256 + C::TAB_BYTES + C::DEC_TAB;  // 16-byte aligned

  const int E = p.E;
  const int MT = GU ? (p.F + kBM - 1) / kBM : (p.H + kDecRows - 1) / kDecRows;
  const int S = GU ? 1 : p.splits;
  const uint32_t warp = warp_id_sync();
  const uint32_t lane = threadIdx.x & 31;

  // ---- prologue: unit prefix over the fused groups + page-table residency check
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
        if (n > 0 && e < p.E_routed && p.dec[e].sm && p.dec[e].fmt == (uint32_t)RFMT && ((p.dec_fmt_mask >> RFMT) & 1u)) {
          u = ((n + BN - 1) / BN) * MT * S;
          const int32_t ent = p.pt[e];
          if (pt_state(ent) != 2) {
            atomicCAS((unsigned long long*)p.fault, 0ull,
                      (unsigned long long)fault_pack(p.layer, p.e_first + e + 1, GU ? 1 : 2, pt_state(ent)));
            bad = true;
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
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < C::BST; ++s) {
      mbar_init(&full[s], FMT == 2 ? 1 : 1 + kDecWarps);  // FMT 2: activations only
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) { mbar_init(&afull[s], kDecWarps); mbar_init(&aempty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    for (int c = 0; c < kFxMaxCst; ++c) { mbar_init(&cfull[c], 1); mbar_init(&cempty[c], kDecWarps); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  if (FMT == 0 && warp >= 6 && warp < 6 + kDecWarps) {  // decoder tables -> smem
    const int t = threadIdx.x - 192;
    const uint4* src = reinterpret_cast<const uint4*>(tabs->pair);
    for (int i = t; i < (1 << kPairBits) / 4; i += 32 * kDecWarps) reinterpret_cast<uint4*>(s_pair)[i] = src[i];
    if (t <= kCodecMaxLen) {
      s_first[t] = tabs->first_code[t];
      s_count[t] = tabs->count[t];
      s_rank[t] = tabs->first_rank[t];
    }
    if (t < kCodecSymbols) s_sym[t] = tabs->sorted_sym[t];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int K = GU ? p.H : p.F;
  const int KB = K / kBK;
  // gate/up -> down overlap: the down launch may start on SMs this grid's tail leaves idle
  if (GU && p.unit_done && threadIdx.x == 0) griddep_launch_dependents();

  if (warp == 0) {
    // ---- activation tiles (hi, lo) by TMA
    if (lane == 0) {
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const DUnit un = dec_unit(u, s_up, s_off, E, BN, S);
        int kb0 = 0, kb1 = KB;
        if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
        const int nb = (un.n_rows + kBoxRowsB - 1) / kBoxRowsB;
        const uint32_t bytes = (p.act_lo ? 2 : 1) * nb * kBoxRowsB * kBK * 2;
        if (!GU && p.unit_done) {
          // this group's h rows: every gate/up unit of the group has stored them (release
          // counter), then order those generic-proxy stores before this thread's TMA reads
          const int n = s_off[un.e + 1] - s_off[un.e];
          const int need = ((n + BN - 1) / BN) * (p.F / kBM);
          for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.unit_done + un.e) : "memory");
            if (v >= need || *(volatile long long*)p.fault != 0) break;
            __nanosleep(200);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_backoff(&empty[stage], phase ^ 1);
          uint8_t* sb = smem + stage * C::STAGE + C::B_OFF;
          mbar_arrive_expect_tx(&full[stage], bytes);
          for (int i = 0; i < nb; ++i) {
            tma_load_2d(sb + i * kBoxRowsB * kBK * 2, &map_b, &full[stage], kb * kBK, un.row_begin + i * kBoxRowsB,
                        pol_b);
            if (p.act_lo)
              tma_load_2d(sb + C::B_BYTES + i * kBoxRowsB * kBK * 2, &map_b, &full[stage], kb * kBK,
                          (int)(un.row_begin + p.act_lo_rows) + i * kBoxRowsB, pol_b);
          }
          if (++stage == C::BST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: A tile 0 -> d0, A tile 1 -> d0 + 128, each against the hi and lo planes
    int stage = 0;       // activation (and, FMT 0/1, A) stage
    uint32_t phase = 0;
    int ast = 0;         // FMT 2: decoded A stage in TMEM
    uint32_t aph = 0;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const DUnit un = dec_unit(u, s_up, s_off, E, BN, S);
      int kb0 = 0, kb1 = KB;
      if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
      const uint32_t idesc = idesc_bf16_f32(kBM, (un.n_rows + 15) & ~15);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait_backoff(&tempty[acc], acc_par ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + acc * C::ACC_W;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait_role(&full[stage], phase, FMT >= 1 && (chunk & kFxSpinFlag));
        if constexpr (FMT == 2) mbar_wait_role(&afull[ast], aph, chunk & kFxSpinFlag);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + stage * C::STAGE);
          const uint32_t bbase = base + C::B_OFF;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t bdesc = sdesc_k_sw128(bbase + 32 * k);
            const uint64_t bdesc_lo = sdesc_k_sw128(bbase + C::B_BYTES + 32 * k);
            const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
            if constexpr (FMT == 2) {
              const uint32_t a0 = tmem + C::A_COL + ast * 64 + 8 * k, a1 = a0 + 32;
              umma_bf16_ts(d0, a0, bdesc, idesc, accum);
              if (p.act_lo) umma_bf16_ts(d0, a0, bdesc_lo, idesc, 1u);
              umma_bf16_ts(d0 + C::UP_OFF, a1, bdesc, idesc, accum);
              if (p.act_lo) umma_bf16_ts(d0 + C::UP_OFF, a1, bdesc_lo, idesc, 1u);
            } else {
              const uint64_t a0 = sdesc_k_sw128(base + 32 * k);
              const uint64_t a1 = sdesc_k_sw128(base + C::A_BYTES + 32 * k);
              umma_bf16(d0, a0, bdesc, idesc, accum);
              if (p.act_lo) umma_bf16(d0, a0, bdesc_lo, idesc, 1u);
              umma_bf16(d0 + 128, a1, bdesc, idesc, accum);
              if (p.act_lo) umma_bf16(d0 + 128, a1, bdesc_lo, idesc, 1u);
            }
          }
          umma_commit(&empty[stage]);
          if constexpr (FMT == 2) umma_commit(&aempty[ast]);
        }
        __syncwarp();
        if (++stage == C::BST) { stage = 0; phase ^= 1; }
        if (++ast == 2) { ast = 0; aph ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp < 6) {
    // ---- epilogue
    const int q = warp & 3;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const DUnit un = dec_unit(u, s_up, s_off, E, BN, S);
      const int acc = it & 1;
      const uint32_t acc_par = (it >> 1) & 1;
      mbar_wait_backoff(&tfull[acc], acc_par);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * C::ACC_W;
      if (GU) {
        const int r = un.m0 + q * 32 + lane;
        __nv_bfloat16* hcol = p.hbuf + (size_t)un.row_begin * p.F + r;
        const size_t lo_off = (size_t)p.h_lo_rows * p.F;
        for (int c0 = 0; c0 < un.n_rows; c0 += 16) {
          float g[16], v[16];
          tmem_ld16(tbase + c0, g);
          tmem_ld16(tbase + C::UP_OFF + c0, v);
          if (r < p.F) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < un.n_rows) {
                __nv_bfloat16 hi, lo;
                split_bf16(silu_d(g[i]) * v[i], &hi, &lo);
                hcol[(size_t)(c0 + i) * p.F] = hi;
                hcol[(size_t)(c0 + i) * p.F + lo_off] = lo;
              }
          }
        }
      } else {
        const int m0 = 2 * un.m0;  // 256-row tiles of W_down
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int r = m0 + half * 128 + q * 32 + lane;
          float* out = p.part + un.split * p.split_stride + (size_t)un.row_begin * p.H + r;
          for (int c0 = 0; c0 < un.n_rows; c0 += 16) {
            float v[16];
            tmem_ld16(tbase + half * C::UP_OFF + c0, v);
            if (r < p.H) {
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
  } else if (warp == 6 + kDecWarps) {
    // ---- FX4 compressed stages by TMA, on their own warp so they run CST stages ahead of the
    // decoders instead of queueing behind the activation loads' wait for a free decoded stage
    if (FMT >= 1 && lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // compressed weights: streamed once
      int cs = 0;
      uint32_t cph = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const DUnit un = dec_unit(u, s_up, s_off, E, BN, S);
        int kb0 = 0, kb1 = KB;
        if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
        const CUtensorMap* fxm = p.dec[un.e].maps;  // [sign/mantissa, nibbles]
        const int r0 = GU ? un.m0 : 2 * un.m0, r1 = GU ? p.F + un.m0 : 2 * un.m0 + kBM;
        for (int kb = kb0; kb < kb1; ++kb) {
          // the stage's compressed rows of both A tiles: 2 x 128 x 64 B of sign/mantissa bytes,
          // 2 x 128 x 32 B of nibbles (swizzled 64 / 32 B so the decoders' row reads spread banks)
          mbar_wait_backoff(&cempty[cs], cph ^ 1);
          uint8_t* cb = cstage + cs * kFxCStage;
          mbar_arrive_expect_tx(&cfull[cs], kFxCStage);
          tma_load_2d(cb, fxm, &cfull[cs], kb * kBK, r0, pol_w);
          tma_load_2d(cb + kFxSmTile, fxm, &cfull[cs], kb * kBK, r1, pol_w);
          tma_load_2d(cb + 2 * kFxSmTile, fxm + 1, &cfull[cs], kb * (kBK / 2), r0, pol_w);
          tma_load_2d(cb + 2 * kFxSmTile + kFxNibTile, fxm + 1, &cfull[cs], kb * (kBK / 2), r1, pol_w);
          if (++cs == C::CST) { cs = 0; cph ^= 1; }
        }
      }
    }
  } else {
    // ---- decoders: thread d owns weight row d of the unit
    // (FMT 2: a warp writes only its own TMEM lane quarter, warp id % 4, so its 32 rows are that
    // quarter of A tile (decoder warp / 4))
    const int dw = (threadIdx.x - 192) >> 5;
    const int a = FMT == 2 ? dw >> 2 : (threadIdx.x - 192) >> 7;
    const int lr = FMT == 2 ? (int)((warp & 3) * 32 + lane) : (threadIdx.x - 192) & 127;
    const int d = a * 128 + lr;
    const uint32_t sw = (uint32_t)(lr & 7);
    const CanonTabs ct{s_count, s_first, s_rank, s_sym, FMT == 0 ? tabs->maxlen : 0};
    int stage = 0;
    uint32_t phase = 0;
    int fcs = 0;        // FX4: compressed stage
    uint32_t fcph = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const DUnit un = dec_unit(u, s_up, s_off, E, BN, S);
      int kb0 = 0, kb1 = KB;
      if (!GU) split_kb(un.split, S, KB, &kb0, &kb1);
      const DecRec R = p.dec[un.e];
      const int wrow = GU ? (a ? p.F : 0) + un.m0 + lr : 2 * un.m0 + d;
      const bool valid = GU ? (un.m0 + lr < p.F) : (2 * un.m0 + d < p.H);
      const uint64_t v0 = (uint64_t)wrow * K + (uint64_t)kb0 * kBK;
      if constexpr (FMT == 0) {
      PWindow w;
      // sign/mantissa bytes: group g (16 values) of the stage lives in register sg; once
      // consumed, sg is reloaded with group g of the next stage -- one stage of lead, and no
      // register rotation (moving a register whose load is in flight waits for the load: ncu
      // put 11% of the samples on such a move).  g is warp-uniform, so the switches below are
      // uniform branches.  The row's bytes two stages further are prefetched into L2.
      const uint8_t* smp = R.sm + v0;  // next stage's sign/mantissa bytes
      const uint8_t* smend = R.sm + (uint64_t)wrow * K + (uint64_t)kb1 * kBK;
      uint4 s0 = make_uint4(0, 0, 0, 0), s1 = s0, s2 = s0, s3 = s0;
      if (valid) {
        w.init(R.bits, R.index[v0 / chunk] - R.bit_base, smem_u32(s_ring + d * kRingBytes), (uint32_t)(d & 7));
        const uint4* q4 = reinterpret_cast<const uint4*>(smp);
        s0 = __ldg(q4);
        s1 = __ldg(q4 + 1);
        s2 = __ldg(q4 + 2);
        s3 = __ldg(q4 + 3);
        smp += 64;
      }
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait_backoff(&empty[stage], phase ^ 1);
        if (valid) {
          if (smp + 128 < smend) asm volatile("prefetch.global.L2 [%0];" ::"l"(smp + 128));
          const uint32_t row = smem_u32(smem + stage * C::STAGE + a * C::A_BYTES + lr * 128);
          // 8 quads of 8 values (one 16-byte swizzled store each); the quad loop stays rolled so
          // the hot code fits the instruction cache (fully unrolled, 32 pair sites with their
          // slow paths made a 140 KB loop: ncu put 44% of the stall cycles on instruction fetch)
#pragma unroll 1
          for (uint32_t q = 0; q < 8; ++q) {
            w.top_up();
            uint4 cur;
            switch (q >> 1) {
              case 0: cur = s0; break;
              case 1: cur = s1; break;
              case 2: cur = s2; break;
              default: cur = s3; break;
            }
            const uint32_t sa = (q & 1) ? cur.z : cur.x, sb = (q & 1) ? cur.w : cur.y;
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if ((j & 1) == 0) w.refill();
              uint32_t e = s_pair[w.peek12()];
              const int len = (int)(e & 15u);
              if (__builtin_expect(len == 0, 0)) e = pair_slow(w, s_pair, ct);
              else w.p += len;
              const uint32_t dup = __byte_perm(j < 2 ? sa : sb, 0, (j & 1) ? 0x3322u : 0x1100u);
              o[j] = (dup & 0x807F807Fu) | (e & 0x7F807F80u);
            }
            st_smem_v4(row + ((q ^ sw) << 4), o[0], o[1], o[2], o[3]);
            if ((q & 1) && smp < smend) {  // group q/2 consumed: load the next stage's
              const uint4* nx = reinterpret_cast<const uint4*>(smp) + (q >> 1);
              // one load per case straight into its register (the compiler merged plain loads
              // into one temporary plus predicated moves, and the moves waited for the load)
              switch (q >> 1) {
                case 0: ldg_v4(s0, nx); break;
                case 1: ldg_v4(s1, nx); break;
                case 2: ldg_v4(s2, nx); break;
                default: ldg_v4(s3, nx); break;
              }
            }
          }
          smp += kBK;
          fence_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      } else {
      // FX4 records (fx4.cuh): the TMA warp stages each stage's sign/mantissa and nibble rows
      // in shared memory; a decoder thread reads its row there (6 x LDS.128), releases the
      // compressed stage, and expands 8 quads -- nibble codes sit at fixed positions, so the
      // pairs decode independently (no window, no table chain, no global load on the path)
      const uint8_t* escp = R.esc;
      const uint32_t bb = R.bit_base * 0x01010101u;
      if (valid) escp = R.esc + R.index[v0 / kFxSeg];
      const uint32_t sm_row = (uint32_t)(a * kFxSmTile + lr * 64), sm_sw = (uint32_t)((lr >> 1) & 3);
      const uint32_t nb_row = (uint32_t)(2 * kFxSmTile + a * kFxNibTile + lr * 32), nb_sw = (uint32_t)((lr >> 2) & 1);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&cfull[fcs], fcph);
        uint4 sv[4], nv[2];
        const uint32_t cb = smem_u32(cstage + fcs * kFxCStage);
        if (valid) {
#pragma unroll
          for (uint32_t g = 0; g < 4; ++g)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(sv[g].x), "=r"(sv[g].y), "=r"(sv[g].z), "=r"(sv[g].w)
                         : "r"(cb + sm_row + ((g ^ sm_sw) << 4))
                         : "memory");
#pragma unroll
          for (uint32_t g = 0; g < 2; ++g)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(nv[g].x), "=r"(nv[g].y), "=r"(nv[g].z), "=r"(nv[g].w)
                         : "r"(cb + nb_row + ((g ^ nb_sw) << 4))
                         : "memory");
          // release the slot as soon as this warp holds its rows, so the producer runs a full
          // CST stages ahead (releasing after the decode cost 6%); a use of every loaded register
          // makes the reads complete first -- releasing before they completed let the producer
          // overwrite rows still being read (wrong results at T = 256)
          const uint32_t all = sv[0].x ^ sv[0].y ^ sv[0].z ^ sv[0].w ^ sv[1].x ^ sv[1].y ^ sv[1].z ^ sv[1].w ^ sv[2].x ^
                               sv[2].y ^ sv[2].z ^ sv[2].w ^ sv[3].x ^ sv[3].y ^ sv[3].z ^ sv[3].w ^ nv[0].x ^ nv[0].y ^
                               nv[0].z ^ nv[0].w ^ nv[1].x ^ nv[1].y ^ nv[1].z ^ nv[1].w;
          asm volatile("" ::"r"(all));
        }
        if (chunk & kFxFenceFlag) fence_async_smem();  // A/B knob: the reads are already complete
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[fcs]);
        if (++fcs == C::CST) { fcs = 0; fcph ^= 1; }
        mbar_wait_role(FMT == 2 ? &aempty[stage] : &empty[stage], phase ^ 1, chunk & kFxSpinFlag);
        if constexpr (FMT == 2) {
          // the stage's 64 values of this row -> 32 registers (bf16 pairs, K order) -> TMEM
          // lane lr, columns A_COL + stage * 64 + a * 32 .. + 31; escapes patched in registers
          tc_fence_after();  // after the empty wait: the MMAs that read this stage are complete
          uint32_t o[32];
          const uint32_t bb7 = bb & 0x00FF00FFu;  // base at bytes 0 and 2: (code pair << 7) + (base pair << 7)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4& nq = nv[q >> 2];
            const uint32_t nw = (q & 3) == 0 ? nq.x : (q & 3) == 1 ? nq.y : (q & 3) == 2 ? nq.z : nq.w;
            const uint4& sq = sv[q >> 1];
            const uint32_t sa = (q & 1) ? sq.z : sq.x, sb = (q & 1) ? sq.w : sq.y;
            const uint32_t lo = nw & 0x0F0F0F0Fu, hi = (nw >> 4) & 0x0F0F0F0Fu;
            const uint32_t escf = ((lo + 0x01010101u) | (hi + 0x01010101u)) & 0x10101010u;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              // y = [lo_j, lo_j, hi_j, hi_j] (codes of values 2j, 2j+1); y * 128 + base pair puts
              // the two exponents at bits 7..14 and 23..30 (code + base <= 255: no carry out of a
              // field; the duplicate bytes land in bits the bit-select drops), and one bit-select
              // merges them with the sign/mantissa bytes: 4 ops per value pair
              const uint32_t y = __byte_perm(lo, hi, (uint32_t)(j | (j << 4) | ((4 + j) << 8) | ((4 + j) << 12)));
              const uint32_t ex = y * 128u + (bb7 << 7);
              const uint32_t dup = __byte_perm(j < 2 ? sa : sb, 0, (j & 1) ? 0x3322u : 0x1100u);
              o[4 * q + j] = (dup & 0x807F807Fu) | (ex & 0x7F807F80u);
            }
            // (one branch per stage instead of per quad: 15% slower, the unrolled patch block
            // changed the schedule of the whole stage)
            if (__builtin_expect(valid && escf != 0u, 0)) {
              // exponents outside the window, in value order: value v is half (v & 1) of word v / 2
#pragma unroll
              for (int v = 0; v < 8; ++v)
                if (((nw >> (4 * v)) & 15u) == 15u) {
                  const uint32_t sh = 7u + 16u * (uint32_t)(v & 1);
                  o[4 * q + (v >> 1)] = (o[4 * q + (v >> 1)] & ~(0xFFu << sh)) | ((uint32_t)*escp++ << sh);
                }
            }
          }
          if (!valid)
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = 0u;

          tmem_st32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(C::A_COL + stage * 64 + a * 32), o);
          tc_fence_before();  // the stores before the MMA warp's barrier wait
        } else if (valid && (chunk & kFxNoDecFlag)) {  // timing A/B: raw stores, no decode
          const uint32_t row = smem_u32(smem + stage * C::STAGE + a * C::A_BYTES + lr * 128);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            st_smem_v4(row + ((((uint32_t)q) ^ sw) << 4), sv[q >> 1].x, sv[q >> 1].y, nv[q >> 2].x, nv[q >> 2].y);
        } else if (valid) {
          const uint32_t row = smem_u32(smem + stage * C::STAGE + a * C::A_BYTES + lr * 128);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4& nq = nv[q >> 2];
            const uint32_t nw = (q & 3) == 0 ? nq.x : (q & 3) == 1 ? nq.y : (q & 3) == 2 ? nq.z : nq.w;
            const uint4& sq = sv[q >> 1];
            const uint32_t sa = (q & 1) ? sq.z : sq.x, sb = (q & 1) ? sq.w : sq.y;
            const uint32_t lo = nw & 0x0F0F0F0Fu, hi = (nw >> 4) & 0x0F0F0F0Fu;
            const uint32_t escf = ((lo + 0x01010101u) | (hi + 0x01010101u)) & 0x10101010u;
            const uint32_t le = lo + bb, he = hi + bb;
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t x = __byte_perm(le, he, (uint32_t)(j | ((4 + j) << 4)));
              const uint32_t ex = ((x & 0xFFu) << 7) | ((x >> 8) << 23);
              const uint32_t dup = __byte_perm(j < 2 ? sa : sb, 0, (j & 1) ? 0x3322u : 0x1100u);
              o[j] = (dup & 0x807F807Fu) | (ex & 0x7F807F80u);
            }
            const uint32_t qa = row + ((((uint32_t)q) ^ sw) << 4);
            st_smem_v4(qa, o[0], o[1], o[2], o[3]);
            if (__builtin_expect(escf != 0u, 0)) {
              // exponents outside the window, in value order: rewrite those values in place
#pragma unroll 1
              for (uint32_t v = 0; v < 8; ++v)
                if (((nw >> (4 * v)) & 15u) == 15u) {
                  const uint32_t sbyte = ((v < 4 ? sa : sb) >> (8 * (v & 3))) & 0xFFu;
                  const uint32_t bf = ((sbyte & 0x80u) << 8) | ((uint32_t)*escp++ << 7) | (sbyte & 0x7Fu);
                  asm volatile("st.shared.u16 [%0], %1;" ::"r"(qa + 2 * v), "h"((unsigned short)bf) : "memory");
                }
            }
          }
        }
        if constexpr (FMT != 2) fence_async_smem();  // the A tile's generic stores before the tensor cores' reads
        __syncwarp();
        if (lane == 0) mbar_arrive(FMT == 2 ? &afull[stage] : &full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
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

using DecKernel = void (*)(const CUtensorMap, GemmParams, const DecTables*, int);

// stage counts: the A tiles are produced on-chip, so a few stages cover the decoder/MMA overlap
#define XPGB_DEC_TILES(X) X(32, 3) X(48, 2) X(64, 2) X(80, 2) X(96, 2) X(128, 2)
// FX4: 2 decoded stages and up to 4 compressed ones (default), or 3 decoded stages and fewer
// compressed ones (XPGB_FX_STAGES=3, A/B)
#define XPGB_FX_TILES(X) X(32, 3) X(48, 2) X(64, 2) X(80, 2) X(96, 2) X(128, 2)
#define XPGB_FX_TILES3(X) X(32, 4) X(48, 3) X(64, 3) X(80, 3) X(96, 3) X(128, 2)
// FX4 with the decoded A tiles in tensor memory (FMT 2, the default for BN <= 96)
#define XPGB_FXT_TILES(X) X(32, 2) X(48, 2) X(64, 2) X(80, 2) X(96, 2)

template <bool GU, int BN, int ST, int FMT>
static void set_dec_attr() {
  cudaFuncSetAttribute(k_moe_gemm_dec<GU, BN, ST, FMT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       DecCfg<BN, ST, FMT>::SMEM);
}

void set_gemm_dec_attrs() {
#define XPGB_SET_DEC(BN, ST) set_dec_attr<true, BN, ST, 0>(); set_dec_attr<false, BN, ST, 0>();
#define XPGB_SET_FX(BN, ST) set_dec_attr<true, BN, ST, 1>(); set_dec_attr<false, BN, ST, 1>();
  XPGB_DEC_TILES(XPGB_SET_DEC)
  XPGB_FX_TILES(XPGB_SET_FX)
  XPGB_FX_TILES3(XPGB_SET_FX)
#define XPGB_SET_FXT(BN, ST) set_dec_attr<true, BN, ST, 2>(); set_dec_attr<false, BN, ST, 2>();
  XPGB_FXT_TILES(XPGB_SET_FXT)
#undef XPGB_SET_FXT
#undef XPGB_SET_DEC
#undef XPGB_SET_FX
}

// A unit's K range (a split_kb range: multiples of 256 values) must start on a chunk boundary.
bool gemm_dec_supported(int H, int F, int chunk) {
  return chunk >= kBK && 256 % chunk == 0 && H % 256 == 0 && F % 256 == 0 && H % kDecRows == 0 && F % kBM == 0;
}

void launch_gemm_dec(bool gate_up, const CUtensorMap& map_b, const GemmParams& p, const CodecTable& table, int chunk,
                     int bn, int grid, cudaStream_t s, bool fx4) {
  const DecTables* tabs = codec_device_tables(table, s);
  if (!tabs) return;
  static const bool fx3 = getenv("XPGB_FX_STAGES") && atoi(getenv("XPGB_FX_STAGES")) == 3;
  DecKernel kern = nullptr;
  int smem = 0;
#define XPGB_PICK_DEC(BN, ST)                                                            \
  if (bn == BN) {                                                                        \
    kern = gate_up ? k_moe_gemm_dec<true, BN, ST, 0> : k_moe_gemm_dec<false, BN, ST, 0>;  \
    smem = DecCfg<BN, ST>::SMEM;                                                         \
  }
#define XPGB_PICK_FX(BN, ST)                                                             \
  if (bn == BN) {                                                                        \
    kern = gate_up ? k_moe_gemm_dec<true, BN, ST, 1> : k_moe_gemm_dec<false, BN, ST, 1>;  \
    smem = DecCfg<BN, ST, 1>::SMEM;                                                      \
  }
#define XPGB_PICK_FXT(BN, ST)                                                            \
  if (bn == BN) {                                                                        \
    kern = gate_up ? k_moe_gemm_dec<true, BN, ST, 2> : k_moe_gemm_dec<false, BN, ST, 2>;  \
    smem = DecCfg<BN, ST, 2>::SMEM;                                                      \
  }
  static const bool fx_tmem = !(getenv("XPGB_FX_TMEM") && atoi(getenv("XPGB_FX_TMEM")) == 0);
  if (!fx4) {
    XPGB_DEC_TILES(XPGB_PICK_DEC)
  } else if (fx_tmem && !fx3 && bn <= 96) {
    XPGB_FXT_TILES(XPGB_PICK_FXT)
  } else if (fx3) {
    XPGB_FX_TILES3(XPGB_PICK_FX)
  } else {
    XPGB_FX_TILES(XPGB_PICK_FX)
  }
#undef XPGB_PICK_DEC
#undef XPGB_PICK_FX
#undef XPGB_PICK_FXT
  if (!kern) {
    kern = fx4 ? (gate_up ? k_moe_gemm_dec<true, 128, 2, 1> : k_moe_gemm_dec<false, 128, 2, 1>)
               : (gate_up ? k_moe_gemm_dec<true, 128, 2, 0> : k_moe_gemm_dec<false, 128, 2, 0>);
    smem = fx4 ? DecCfg<128, 2, 1>::SMEM : DecCfg<128, 2>::SMEM;
  }
  // FX4 ignores the Huffman chunk; its top bit carries the release-fence A/B (XPGB_FX_FENCE=0 drops it)
  static const bool fx_fence = !(getenv("XPGB_FX_FENCE") && atoi(getenv("XPGB_FX_FENCE")) == 0);
  static const bool fx_spin = getenv("XPGB_FX_SPIN") && atoi(getenv("XPGB_FX_SPIN")) != 0;
  static const bool fx_nodec = getenv("XPGB_FX_NODEC") && atoi(getenv("XPGB_FX_NODEC")) != 0;
  const int arg =
      fx4 ? ((fx_fence ? kFxFenceFlag : 0) | (fx_spin ? kFxSpinFlag : 0) | (fx_nodec ? kFxNoDecFlag : 0)) : chunk;
  if (!gate_up && p.unit_done) {  // overlaps the gate/up launch's tail (programmatic dependent launch)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kDecThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, map_b, p, tabs, arg);
  } else {
    kern<<<grid, kDecThreads, smem, s>>>(map_b, p, tabs, arg);
  }
  note_launch();
}

}  // namespace xpgb
