// Microbenchmark: read-only streaming of 4608-B records with per-warp TMA
// (cp.async.bulk) rings, the access pattern of k_pass_a, with no compute.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_20868_b200/csrc/common.cuh"
using namespace ckv;
template <int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32) k_stream(const uint8_t* base, int nblk_per_cta, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* stage = sm;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + WARPS * STAGES * REC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < WARPS * STAGES; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* cb = base + (size_t)blockIdx.x * nblk_per_cta * REC;
  const int nmine = (nblk_per_cta - warp + WARPS - 1) / WARPS;
  if (lane == 0)
    for (int s = 0; s < STAGES && s < nmine; ++s) {
      mbar_expect_tx(&bar[warp * STAGES + s], REC);
      bulk_g2s(stage + (warp * STAGES + s) * REC, cb + (size_t)(warp + WARPS * s) * REC, REC, &bar[warp * STAGES + s]);
    }
  float acc = 0.f;
  for (int i = 0; i < nmine; ++i) {
    const int s = i % STAGES;
    mbar_wait(&bar[warp * STAGES + s], (i / STAGES) & 1);
    acc += reinterpret_cast<const float*>(stage + (warp * STAGES + s) * REC)[lane];
    __syncwarp();
    if (lane == 0 && i + STAGES < nmine) {
      mbar_expect_tx(&bar[warp * STAGES + s], REC);
      bulk_g2s(stage + (warp * STAGES + s) * REC, cb + (size_t)(warp + WARPS * (i + STAGES)) * REC, REC, &bar[warp * STAGES + s]);
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}
template <int WARPS, int STAGES>
void run(const uint8_t* d, size_t nrec, float* sink, size_t pad = 0) {
  const int per = 256;
  const int grid = (int)(nrec / per);
  const size_t smem = WARPS * STAGES * REC + WARPS * STAGES * 8 + pad;
  cudaFuncSetAttribute(k_stream<WARPS, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k_stream<WARPS, STAGES><<<grid, WARPS * 32, smem>>>(d, per, sink);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_stream<WARPS, STAGES><<<grid, WARPS * 32, smem>>>(d, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<WARPS, STAGES>, WARPS * 32, smem);
  printf("warps %d stages %d: %.3f ms  %.1f GB/s  (CTAs/SM %d)  err=%s\n", WARPS, STAGES, best,
         (double)grid * per * REC / best / 1e6, occ, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t nrec = 2097152;  // 9.66 GB as in C3
  uint8_t* d; float* sink;
  cudaMalloc(&d, nrec * REC); cudaMemset(d, 1, nrec * REC); cudaMalloc(&sink, 4);
  run<4, 2>(d, nrec, sink, 56 * 1024 - 4 * 2 * REC);  // 4 CTAs/SM: 32 records in flight / SM
  run<4, 2>(d, nrec, sink, 75 * 1024 - 4 * 2 * REC);  // 3 CTAs/SM: 24
  run<4, 2>(d, nrec, sink, 110 * 1024 - 4 * 2 * REC);  // 2 CTAs/SM: 16
  run<4, 3>(d, nrec, sink, 56 * 1024 - 4 * 3 * REC);  // 4 CTAs/SM: 48
  run<4, 3>(d, nrec, sink, 75 * 1024 - 4 * 3 * REC);  // 3 CTAs/SM: 36
  return 0;
}
