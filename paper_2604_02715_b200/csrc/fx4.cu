// FX4 device-tier format: encoder and standalone decoder (layout and rationale in fx4.cuh).
#include <algorithm>
#include <vector>

#include "fx4.cuh"
#include "launch_count.h"

namespace xpgb {

namespace {

__device__ __forceinline__ uint32_t exp_of(uint32_t w) { return (w >> 7) & 0xFFu; }

__global__ void k_fx4_hist(const uint16_t* __restrict__ raw, uint64_t n, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint4* p = reinterpret_cast<const uint4*>(raw);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n / 8; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = p[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      atomicAdd(&h[exp_of(w[k])], 1u);
      atomicAdd(&h[exp_of(w[k] >> 16)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// escapes per 256-value segment
__global__ void k_fx4_count(const uint16_t* __restrict__ raw, uint64_t n, int base, uint32_t* __restrict__ cnt) {
  const uint64_t seg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (seg >= n / kFxSeg) return;
  const uint4* p = reinterpret_cast<const uint4*>(raw + seg * kFxSeg);
  uint32_t c = 0;
  for (int i = 0; i < kFxSeg / 8; ++i) {
    const uint4 v = p[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c += (exp_of(w[k]) - (uint32_t)base) > 14u;
      c += (exp_of(w[k] >> 16) - (uint32_t)base) > 14u;
    }
  }
  cnt[seg] = c;
}

// exclusive scan of m counts into out[0..m] (out[m] = total), one CTA
__global__ void k_fx4_scan(const uint32_t* __restrict__ cnt, uint64_t m, uint32_t* __restrict__ out) {
  __shared__ uint32_t part[1024];
  const int t = threadIdx.x;
  const uint64_t per = (m + blockDim.x - 1) / blockDim.x;
  const uint64_t a0 = (uint64_t)t * per, a = a0 < m ? a0 : m, b = a + per < m ? a + per : m;
  uint32_t s = 0;
  for (uint64_t i = a; i < b; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    uint32_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const uint32_t x = part[i];
      part[i] = run;
      run += x;
    }
  }
  __syncthreads();
  uint32_t run = part[t];
  for (uint64_t i = a; i < b; ++i) {
    out[i] = run;
    run += cnt[i];
  }
  if (b == m && a < b) out[m] = run;
  if (m == 0 && t == 0) out[0] = 0;
}

// thread per segment: sign/mantissa bytes, nibbles, escapes
__global__ void k_fx4_write(const uint16_t* __restrict__ raw, uint64_t n, int base, const uint32_t* __restrict__ idx,
                            uint8_t* __restrict__ rec, FxLayout L) {
  const uint64_t seg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (seg >= n / kFxSeg) return;
  const uint4* p = reinterpret_cast<const uint4*>(raw + seg * kFxSeg);
  uint4* sm = reinterpret_cast<uint4*>(rec + seg * kFxSeg);
  uint2* nib = reinterpret_cast<uint2*>(rec + L.nib + seg * (kFxSeg / 2));
  uint8_t* esc = rec + L.esc + idx[seg];
  for (int g = 0; g < kFxSeg / 16; ++g) {  // 16 values per group
    const uint4 v0 = p[2 * g], v1 = p[2 * g + 1];
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t smw[4] = {0, 0, 0, 0}, nw[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t x = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      const uint32_t e = exp_of(x);
      const uint32_t sb = ((x >> 8) & 0x80u) | (x & 0x7Fu);
      smw[k >> 2] |= sb << (8 * (k & 3));
      uint32_t code = e - (uint32_t)base;
      if (code > 14u) {
        *esc++ = (uint8_t)e;
        code = 15u;
      }
      nw[k >> 3] |= code << (4 * (k & 7));
    }
    sm[g] = make_uint4(smw[0], smw[1], smw[2], smw[3]);
    nib[g] = make_uint2(nw[0], nw[1]);
  }
}

// thread per 16 values: coalesced sign/mantissa, nibble and bf16 accesses
__global__ void k_fx4_decode(const uint8_t* __restrict__ rec, uint64_t n, int base, FxLayout L,
                             uint16_t* __restrict__ out) {
  const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (g >= n / 16) return;
  const uint4 smv = reinterpret_cast<const uint4*>(rec)[g];
  const uint2 nv = reinterpret_cast<const uint2*>(rec + L.nib)[g];
  const uint32_t bb = (uint32_t)base * 0x01010101u;
  const uint32_t nw[2] = {nv.x, nv.y};
  const uint32_t smw[4] = {smv.x, smv.y, smv.z, smv.w};
  uint32_t o[8];
  uint32_t escm = 0;  // nonzero when the group holds an escape
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t lo = nw[h] & 0x0F0F0F0Fu, hi = (nw[h] >> 4) & 0x0F0F0F0Fu;
    // bytes equal to 15 are escapes: (x + 1) & 0x10 per byte
    const uint32_t el = ((lo + 0x01010101u) & 0x10101010u) >> 4, eh = ((hi + 0x01010101u) & 0x10101010u) >> 4;
    escm |= el | eh;
    const uint32_t le = lo + bb, he = hi + bb;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t x = __byte_perm(le, he, (uint32_t)(j | ((4 + j) << 4)));  // byte 0: le_j, byte 1: he_j
      const uint32_t ex = ((x & 0xFFu) << 7) | ((x >> 8) << 23);
      const int k = 4 * h + j;  // pair index
      const uint32_t dup = __byte_perm(smw[k >> 1], 0, (k & 1) ? 0x3322u : 0x1100u);
      o[k] = (dup & 0x807F807Fu) | (ex & 0x7F807F80u);
    }
  }
  if (escm) {
    // escapes before this group in its segment, then patch each escaped value
    const uint64_t seg = g * 16 / kFxSeg;
    uint32_t e = reinterpret_cast<const uint32_t*>(rec + L.idx)[seg];
    const uint32_t* nseg = reinterpret_cast<const uint32_t*>(rec + L.nib + seg * (kFxSeg / 2));
    for (uint64_t q = 0; q < (g * 16 - seg * kFxSeg) / 8; ++q) {
      const uint32_t w = nseg[q];
      const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
      e += __popc((lo + 0x01010101u) & 0x10101010u) + __popc((hi + 0x01010101u) & 0x10101010u);
    }
    const uint8_t* esc = rec + L.esc;
    for (int v = 0; v < 16; ++v) {
      if (((nw[v >> 3] >> (4 * (v & 7))) & 15u) != 15u) continue;
      const uint32_t ex = (uint32_t)esc[e++];
      const int k = v >> 1, sh = 16 * (v & 1);
      o[k] = (o[k] & ~(0xFFu << (7 + sh))) | (ex << (7 + sh));
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(out + 16 * g);
  dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

}  // namespace

void fx4_count(const uint16_t* raw, uint64_t n, uint32_t* scratch, int* base, uint64_t* n_esc, cudaStream_t s) {
  uint32_t* hist = scratch;  // 256 entries, then the segment counts
  cudaMemsetAsync(hist, 0, 256 * 4, s);
  k_fx4_hist<<<148 * 4, 256, 0, s>>>(raw, n, hist);
  note_launch();
  std::vector<uint32_t> h(256);
  cudaMemcpyAsync(h.data(), hist, 256 * 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  uint64_t best = 0;
  int b = 0;
  // 15-wide window with the most values; base <= 240 so base + 15 (an escape's code) still fits
  // a byte -- the decoders add the base to four codes at once, and a carry would reach the next
  for (int lo = 0; lo <= kFxMaxBase; ++lo) {
    uint64_t c = 0;
    for (int k = 0; k < 15; ++k) c += h[lo + k];
    if (c > best) {
      best = c;
      b = lo;
    }
  }
  *base = b;
  *n_esc = n - best;
}

void fx4_encode(const uint16_t* raw, uint64_t n, int base, uint32_t* scratch, uint8_t* rec, cudaStream_t s) {
  const uint64_t ns = n / kFxSeg;
  const FxLayout L0 = fx_layout(n, 0);
  uint32_t* cnt = scratch + 256;
  uint32_t* idx = reinterpret_cast<uint32_t*>(rec + L0.idx);  // the record's own escape index
  const unsigned blocks = (unsigned)((ns + 255) / 256);
  if (ns) {
    k_fx4_count<<<blocks, 256, 0, s>>>(raw, n, base, cnt);
    note_launch();
  }
  k_fx4_scan<<<1, 1024, 0, s>>>(cnt, ns, idx);
  note_launch();
  uint32_t total = 0;
  cudaMemcpyAsync(&total, idx + ns, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const FxLayout L = fx_layout(n, total);
  if (ns) {
    k_fx4_write<<<blocks, 256, 0, s>>>(raw, n, base, idx, rec, L);
    note_launch();
  }
}

void launch_fx4_decode(const uint8_t* rec, uint64_t n, int base, uint16_t* out, cudaStream_t s) {
  if (!n) return;
  const FxLayout L = fx_layout(n, 0);  // offsets before the escape bytes do not depend on the count
  const uint64_t groups = n / 16;
  k_fx4_decode<<<(unsigned)((groups + 255) / 256), 256, 0, s>>>(rec, n, base, L, out);
  note_launch();
}

}  // namespace xpgb
