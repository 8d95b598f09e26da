// Exploration spot check (fallback.py:202-227, harness.py:262-269).
//
// The reference samples count = min(|tail|, round(rate * N_B)) positions of
// the ascending tail list with the workload's host Philox generator
// (rng.choice(len(tail), count, replace=False)); the draws depend only on the
// tail size, so the host draws them after reading K' back and the device maps
// position -> block (the pos-th non-promoted full block), rescoring it on the
// FP16 originals (orig_block) against its Phase-1 scores (phase1_block):
// a gap above Delta + epsilon_guard is a Rung-4 canary event.
#include "step.cuh"

namespace ckv {

__global__ void __launch_bounds__(128) k_explore(StepArgs a) {
  extern __shared__ __align__(16) uint32_t sh[];
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  const ckv_policy& pol = a.pol;
  const int h = blockIdx.x, u = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nh = st.n_heads;
  const size_t hu = (size_t)u * nh + h;
  const int n = st.explore_n[hu];
  if (n <= 0) return;
  const int nb = c.n_blocks[u];
  const int W = (nb + 31) / 32;
  uint32_t* fb = sh;               // [W] promoted bitmap
  uint32_t* pre = sh + W;          // [W] tail blocks before word w
  __shared__ __align__(16) float qh[H * D];
  __shared__ int fail;
  for (int i = tid; i < W; i += blockDim.x) fb[i] = 0u;
  for (int i = tid; i < H * D; i += blockDim.x) {
    const int hh = i / D;
    qh[i] = (hh < nh) ? (float)(st.q[((size_t)u * nh + hh) * D + (i % D)] * 0.08838834764831845) : 0.f;
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  const int kp = st.cert[hu].k_star;
  const int32_t* ord = st.order + hu * st.kcap;
  for (int i = tid; i < kp; i += blockDim.x) atomicOr(&fb[ord[i] >> 5], 1u << (ord[i] & 31));
  __syncthreads();
  if (tid == 0) {  // exclusive prefix of tail counts per 32-block word
    int run = 0;
    for (int w = 0; w < W; ++w) {
      pre[w] = run;
      const uint32_t valid = (w == W - 1 && (nb & 31)) ? ((1u << (nb & 31)) - 1u) : 0xffffffffu;
      run += __popc(~fb[w] & valid);
    }
  }
  __syncthreads();
  QFrag f;
  load_qfrag(f, qh, lane);
  QFrag16 f16;
  load_qfrag16(f16, qh, lane);
  const HeadState& hs = *reinterpret_cast<const HeadState*>(st.head_state + hu * CKV_HEAD_FLOATS);
  const double thr = (double)hs.delta + pol.epsilon_guard;
  const size_t ubk = (size_t)u * c.max_blocks;
  const int32_t* pos = st.explore_pos + hu * st.ecap;
  for (int i = warp; i < n; i += blockDim.x / 32) {
    // block id of tail position pos[i]: binary search the word, then the bit
    const int p = pos[i];
    int lo = 0, hi = W - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    uint32_t m = ~fb[lo];
    int r = p - (int)pre[lo];
    while (r-- > 0) m &= m - 1u;
    const int b = lo * 32 + __ffs(m) - 1;
    if (lane == 0 && !c.tier2_valid[ubk + b]) atomicOr(&c.status[CKV_ST_TIER2], 1);
    const BlockScores q = phase1_block(f, c.tier1 + (ubk + b) * REC, c.kscale_max[ubk + b], lane);
    const float2 o = orig_block(f16, reinterpret_cast<const uint4*>(c.tier2_k + (ubk + b) * B * D), lane);
    float gap = fmaxf(fabsf(o.x - q.s0), fabsf(o.y - q.s1));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 4));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 8));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 16));
    if (lane == h && !((double)gap <= thr)) fail = 1;
  }
  __syncthreads();
  if (tid == 0 && fail) {
    ckv_cert& ct = st.cert[hu];
    ct.flags |= CKV_F_EXPLORE;
    ct.returned_kind = 2;
  }
}


cudaError_t launch_explore(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st,
                           int host_max_blocks, cudaStream_t s) {
  StepArgs a{*c, *st, *pol};
  const int W = (host_max_blocks + 31) / 32;
  k_explore<<<dim3(st->n_heads, c->n_units), 128, 2 * W * 4, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace ckv
