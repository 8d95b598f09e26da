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

constexpr int XP_WARPS = 4;
constexpr int XP_STAGES = 3;
constexpr int XP_KEY = OFF_VCODES;  // key codes + scale + offset: the head of the record
constexpr int XP_STAGE = XP_KEY + B * D * 2;  // + the FP16 original key tile

struct ExploreSmem {
  uint8_t stage[XP_WARPS][XP_STAGES][XP_STAGE];
  uint64_t bar[XP_WARPS][XP_STAGES];
  float qh[H * D];
};

// One CTA per (unit, q-head).  The sampled tail positions are mapped to block
// ids first (promoted bitmap + per-word tail prefix), then every warp streams
// its blocks through a 3-stage ring of bulk copies -- the key part of the
// Tier-1 record (3 KB) and the FP16 original key tile (4 KB) per block -- and
// compares the Phase-1 scores (phase1_block) with the original-key scores
// (orig_block): a gap above Delta + epsilon_guard is a canary event.
__global__ void __launch_bounds__(XP_WARPS * 32) k_explore(StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ExploreSmem& S = *reinterpret_cast<ExploreSmem*>(smem_raw);
  uint32_t* fb = reinterpret_cast<uint32_t*>(smem_raw + sizeof(ExploreSmem));  // [W] promoted
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_EXPLORE);
  const ckv_policy& pol = a.pol;
  const int h = blockIdx.x, u = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nh = st.n_heads;
  const size_t hu = (size_t)u * nh + h;
  const int n = st.explore_n[hu];
  if (n <= 0) return;
  const int nb = c.n_blocks[u];
  const int W = (nb + 31) / 32;
  uint32_t* pre = fb + W;                                    // [W] tail blocks before word w
  int32_t* blk = reinterpret_cast<int32_t*>(pre + W);        // [n] sampled block ids
  __shared__ int fail;
  for (int i = tid; i < W; i += blockDim.x) fb[i] = 0u;
  for (int i = tid; i < H * D; i += blockDim.x) {
    const int hh = i / D;
    S.qh[i] = (hh < nh) ? (float)(st.q[((size_t)u * nh + hh) * D + (i % D)] * 0.08838834764831845) : 0.f;
  }
  if (tid == 0) {
    fail = 0;
    for (int w = 0; w < XP_WARPS; ++w)
      for (int s = 0; s < XP_STAGES; ++s) mbar_init(&S.bar[w][s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int kp = st.cert[hu].k_star;
  const int32_t* ord = st.order + hu * st.kcap;
  for (int i = tid; i < kp; i += blockDim.x) atomicOr(&fb[ord[i] >> 5], 1u << (ord[i] & 31));
  __syncthreads();
  if (warp == 0) {  // exclusive prefix of the tail counts per 32-block word
    int carry = 0;
    for (int w0 = 0; w0 < W; w0 += 32) {
      const int w = w0 + lane;
      int cnt = 0;
      if (w < W) {
        const uint32_t valid = (w == W - 1 && (nb & 31)) ? ((1u << (nb & 31)) - 1u) : 0xffffffffu;
        cnt = __popc(~fb[w] & valid);
      }
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (w < W) pre[w] = carry + x - cnt;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
  // tail position -> block: binary search the word, then the bit
  const int32_t* pos = st.explore_pos + hu * st.ecap;
  for (int i = tid; i < n; i += blockDim.x) {
    const int p = pos[i];
    int lo = 0, hi = W - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)pre[mid] <= p) lo = mid; else hi = mid - 1;
    }
    uint32_t m = ~fb[lo];
    int r = p - (int)pre[lo];
    while (r-- > 0) m &= m - 1u;
    blk[i] = lo * 32 + __ffs(m) - 1;
  }
  __syncthreads();
  const size_t ubk = (size_t)u * c.max_blocks;
  const int nmine = (n > warp) ? (n - warp + XP_WARPS - 1) / XP_WARPS : 0;
  auto issue = [&](int i, int s) {
    const int b = blk[warp + XP_WARPS * i];
    mbar_expect_tx(&S.bar[warp][s], XP_STAGE);
    bulk_g2s(S.stage[warp][s], c.tier1 + (ubk + b) * REC, XP_KEY, &S.bar[warp][s]);
    bulk_g2s(S.stage[warp][s] + XP_KEY, c.tier2_k + (ubk + b) * B * D, B * D * 2, &S.bar[warp][s]);
  };
  if (lane == 0)
    for (int s = 0; s < XP_STAGES && s < nmine; ++s) issue(s, s);
  QFrag f;
  load_qfrag(f, S.qh, lane);
  QFrag16 f16;
  load_qfrag16(f16, S.qh, lane);
  const HeadState& hs = *reinterpret_cast<const HeadState*>(st.head_state + hu * CKV_HEAD_FLOATS);
  const double thr = (double)hs.delta + pol.epsilon_guard;
  bool bad = false;
  for (int i = 0; i < nmine; ++i) {
    const int s = i % XP_STAGES;
    const int b = blk[warp + XP_WARPS * i];
    if (lane == 0 && !c.tier2_valid[ubk + b]) atomicOr(&c.status[CKV_ST_TIER2], 1);
    mbar_wait(&S.bar[warp][s], (uint32_t)(i / XP_STAGES) & 1u);
    const uint8_t* st8 = S.stage[warp][s];
    const BlockScores q = phase1_block(f, st8, c.kscale_max[ubk + b], lane);
    const float2 o = orig_block(f16, reinterpret_cast<const uint4*>(st8 + XP_KEY), lane);
    float gap = fmaxf(fabsf(o.x - q.s0), fabsf(o.y - q.s1));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 4));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 8));
    gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 16));
    bad |= (lane == h && !((double)gap <= thr));
    __syncwarp();  // every lane is done with the stage before it is refilled
    if (lane == 0 && i + XP_STAGES < nmine) issue(i + XP_STAGES, s);
  }
  if (bad) fail = 1;
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
  const size_t smem = sizeof(ExploreSmem) + (size_t)2 * W * 4 + (size_t)st->ecap * 4;
  cudaError_t e = set_max_dyn_smem(k_explore, (int)smem);
  if (e != cudaSuccess) return e;
  k_explore<<<dim3(st->n_heads, c->n_units), XP_WARPS * 32, smem, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace ckv
