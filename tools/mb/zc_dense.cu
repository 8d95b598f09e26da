// Zero-copy read rate of pinned host memory in the dense-rung pattern: per task a
// contiguous run of 4-KB key blocks and the matching value blocks of one unit,
// 4 warps per CTA, each warp one block (K + V, 16 x 16 B per lane) at a time or
// DEPTH blocks in flight; against the DMA rate of the same bytes.
#include <cstdio>
#include <cuda_runtime.h>
template <int DEPTH>
__global__ void zc_dense(const uint4* __restrict__ k, const uint4* __restrict__ v, size_t unit_blocks,
                         int units, int splits, uint4* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int task = blockIdx.x; task < units * splits; task += gridDim.x) {
    const int u = task / splits, sp = task % splits;
    const size_t bps = unit_blocks / splits;
    const size_t b0 = (size_t)u * unit_blocks + sp * bps;
    for (size_t b = warp * DEPTH; b < bps; b += 4 * DEPTH) {
      uint4 t[DEPTH][16];
#pragma unroll
      for (int d = 0; d < DEPTH; ++d)
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          t[d][g] = v[(b0 + b + d) * 256 + g * 32 + lane];
          t[d][8 + g] = k[(b0 + b + d) * 256 + g * 32 + lane];
        }
#pragma unroll
      for (int d = 0; d < DEPTH; ++d)
#pragma unroll
        for (int g = 0; g < 16; ++g) acc.x ^= t[d][g].x ^ t[d][g].w;
    }
  }
  if (acc.x == 0x12345678u) sink[threadIdx.x] = acc;
}
int main() {
  const size_t unit_blocks = 8192, units_total = 256, bytes = units_total * unit_blocks * 4096;  // 8.6 GB each
  void *hk, *hv;
  if (cudaHostAlloc(&hk, bytes, cudaHostAllocMapped) || cudaHostAlloc(&hv, bytes, cudaHostAllocMapped)) {
    printf("alloc failed\n");
    return 1;
  }
  memset(hk, 1, bytes);
  memset(hv, 2, bytes);
  uint4 *dk, *dv, *sink;
  cudaHostGetDevicePointer((void**)&dk, hk, 0);
  cudaHostGetDevicePointer((void**)&dv, hv, 0);
  cudaMalloc(&sink, 1 << 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int units = 12;
  for (int splits : {32, 128}) {
    for (int grid : {148 * 4, 148 * 8}) {
      for (int depth : {1, 2}) {
        // units spread over the 256 (every 21st), as Rung-3 units are
        const uint4* kk = dk + (size_t)7 * unit_blocks * 256;
        const uint4* vv = dv + (size_t)7 * unit_blocks * 256;
        auto run = [&]() {
          if (depth == 1) zc_dense<1><<<grid, 128>>>(kk, vv, unit_blocks, units, splits, sink);
          else zc_dense<2><<<grid, 128>>>(kk, vv, unit_blocks, units, splits, sink);
        };
        run();
        cudaEventRecord(a);
        run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("zero-copy dense pattern: %d units x 64 MB (K+V), splits %3d, grid %4d, depth %d: %.1f GB/s\n",
               units, splits, grid, depth, (double)units * unit_blocks * 8192 / (ms / 1e3) / 1e9);
      }
    }
  }
  void* d;
  cudaMalloc(&d, (size_t)units * unit_blocks * 8192);
  cudaEventRecord(a);
  for (int u = 0; u < units; ++u) {
    cudaMemcpyAsync((char*)d + (size_t)u * unit_blocks * 8192, (char*)hk + (size_t)(7 + u) * unit_blocks * 4096,
                    unit_blocks * 4096, cudaMemcpyHostToDevice);
    cudaMemcpyAsync((char*)d + (size_t)u * unit_blocks * 8192 + unit_blocks * 4096,
                    (char*)hv + (size_t)(7 + u) * unit_blocks * 4096, unit_blocks * 4096, cudaMemcpyHostToDevice);
  }
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("DMA of the same bytes: %.1f GB/s\n", (double)units * unit_blocks * 8192 / (ms / 1e3) / 1e9);
  return 0;
}
