// Zero-copy read bandwidth of pinned host memory from SMs (PCIe), by load depth / grid.
#include <cstdio>
#include <cuda_runtime.h>
template <int DEPTH>
__global__ void zc_read(const uint4* __restrict__ src, uint4* dst, size_t n16, int chunk16) {
  // each CTA reads contiguous chunks of chunk16 16-B words; each thread DEPTH loads in flight
  const size_t nchunks = n16 / chunk16;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint4* p = src + c * chunk16;
    for (int i0 = 0; i0 < chunk16; i0 += blockDim.x * DEPTH) {
      uint4 v[DEPTH];
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        const int i = i0 + d * blockDim.x + threadIdx.x;
        v[d] = (i < chunk16) ? p[i] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) { acc.x ^= v[d].x; acc.y ^= v[d].y; acc.z ^= v[d].z; acc.w ^= v[d].w; }
    }
  }
  if (acc.x == 0x12345678u) dst[threadIdx.x] = acc;
}
template <int DEPTH>
void run(const uint4* src, uint4* dst, size_t bytes, int grid, int threads, int chunk) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  zc_read<DEPTH><<<grid, threads>>>(src, dst, bytes / 16, chunk / 16);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) zc_read<DEPTH><<<grid, threads>>>(src, dst, bytes / 16, chunk / 16);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("depth %2d grid %5d threads %4d chunk %7d: %.1f GB/s\n", DEPTH, grid, threads, chunk,
         3.0 * bytes / (ms / 1e3) / 1e9);
}
// random 4-KB blocks over the whole buffer (the page-in pattern): one block per warp-iteration
__global__ void zc_rand(const uint4* __restrict__ src, uint4* dst, size_t nblk, int per_cta) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < per_cta; k += nw * 4) {
    uint4 v[4][8];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      unsigned long long h = (unsigned long long)(blockIdx.x * per_cta + k + d * nw) * 0x9E3779B97F4A7C15ull;
      const size_t b = (h >> 20) % nblk;
      const uint4* p = src + b * 256;
#pragma unroll
      for (int i = 0; i < 8; ++i) v[d][i] = p[i * 32 + lane];
    }
#pragma unroll
    for (int d = 0; d < 4; ++d)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc.x ^= v[d][i].x;
  }
  if (acc.x == 0x12345678u) dst[threadIdx.x] = acc;
}
int main() {
  const size_t bytes = 512ull << 20;
  void* h; cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  memset(h, 1, bytes);
  void* d; cudaHostGetDevicePointer(&d, h, 0);
  uint4* dst; cudaMalloc(&dst, 1 << 20);
  const uint4* s = (const uint4*)d;
  run<8>(s, dst, bytes, 148 * 8, 256, 4096);
  run<8>(s, dst, bytes, 148 * 8, 256, 65536);
  run<16>(s, dst, bytes, 148 * 8, 256, 65536);
  run<16>(s, dst, bytes, 148 * 4, 512, 65536);
  run<32>(s, dst, bytes, 148 * 4, 256, 65536);
  run<4>(s, dst, bytes, 148 * 16, 128, 4096);
  run<16>(s, dst, bytes, 148, 1024, 1 << 20);
  run<16>(s, dst, bytes, 296, 1024, 1 << 20);
  run<8>(s, dst, bytes, 64, 256, 1 << 20);
  run<8>(s, dst, bytes, 32, 256, 1 << 20);
  for (size_t gb : {1ull, 8ull, 32ull}) {
    const size_t big = gb << 30;
    void* hb;
    if (cudaHostAlloc(&hb, big, cudaHostAllocMapped) != cudaSuccess) { printf("alloc %zu GB failed\n", gb); break; }
    memset(hb, 1, big);
    void* db; cudaHostGetDevicePointer(&db, hb, 0);
    const int per = 256, grid = 148 * 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    zc_rand<<<grid, 256>>>((const uint4*)db, dst, big / 4096, per);
    cudaEventRecord(a);
    zc_rand<<<grid, 256>>>((const uint4*)db, dst, big / 4096, per);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("random 4KB blocks over %zu GB: %.1f GB/s\n", gb, (double)grid * per * 4096 / (ms / 1e3) / 1e9);
    cudaFreeHost(hb);
  }
  return 0;
}
