// Microbenchmark: kernel reads of pinned host memory (zero-copy) vs cudaMemcpyAsync H2D.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const int4* __restrict__ src, int4* __restrict__ dst, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}
int main() {
  const size_t n = 1ull << 30;
  void *h, *d;
  cudaHostAlloc(&h, n, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaMalloc(&d, n);
  memset(h, 1, n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy H2D: %.1f GB/s\n", n / ms / 1e6);
  }
  int grids[] = {16, 32, 64, 148, 296, 592, 1184};
  int blocks[] = {256, 512};
  for (int bi = 0; bi < 2; ++bi)
  for (int g : grids) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); rd<<<g, blocks[bi]>>>((const int4*)h, (int4*)d, n / 16); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("kernel zero-copy grid=%d block=%d: %.1f GB/s\n", g, blocks[bi], n / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
