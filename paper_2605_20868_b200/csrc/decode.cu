// The certified decode step on device.
//
//   pass A  (k_pass_a)  streams every unit's Tier-1 once (TMA bulk copies into
//                       a per-warp smem ring): Phase-1 INT8 scores on the
//                       tensor cores, per-block log-mass l'_b, Delta_b, and a
//                       *speculative* Phase-2 online-softmax attend over all
//                       blocks with quantized scores and INT4 values.
//   select  (k_select)  per q-head: lse, radix top-K, coverage K*, Rung 1,
//                       tail mass, Rung 2 value promotions, tail part of
//                       E_val, the promoted / value work list.
//   pass B  (k_pass_b)  per q-head over the work list only: original-key
//                       scores from Tier-2, phase-2 log-mass of promoted
//                       blocks, canary gap, and the additive correction that
//                       turns the speculative attend into the mask-gated one.
//   combine (k_combine) per q-head: merge, output, ranking / boundary /
//                       canary monitors, E_key / E_val, rung flags.
//
// Every additive decomposition is over blocks, so the result equals the
// reference's single mask-gated pass (attention.py:227-300) up to fp32
// rounding.
#include <cstdlib>
#include "step.cuh"

namespace ckv {

// =============================================================================
// pass A
// =============================================================================
#ifndef PA_WARPS_CFG
#define PA_WARPS_CFG 4
#endif
constexpr int PA_WARPS = PA_WARPS_CFG;

// A warp's ring refills a stage only after computing on it, so a record costs
// (latency + compute) / stages.  Many waves of CTAs (C3: 16) run three stages
// (1.4% faster pass A there); a few (the kv1 proxy: 2) two, where three measured
// 4% slower.  4 CTAs x 56.4 KB per SM
// fit only with q' staged in the last warp's last stage, which is filled once
// the fragments are built.
template <int STG>
struct PassASmem {
  static constexpr bool QALIAS = STG >= 3;
  uint8_t stage[PA_WARPS][STG][REC];
  uint64_t bar[PA_WARPS][STG];
  float pbuf[PA_WARPS][H][B];  // p' of the block, tokens permuted (vmeta order)
  float qh[QALIAS ? 1 : H * D];
};
static_assert(H * D * 4 <= REC, "q' staging fits one stage");
constexpr int PA_DEEP_WAVES = 4;  // waves of CTAs from which three stages pay

// (PVFrag / pv_frag / pv_block_sub: step.cuh)

#ifndef PA_MINB
#define PA_MINB 4
#endif
template <int PA_STAGES>
__global__ void __launch_bounds__(PA_WARPS * 32, PA_MINB) k_pass_a(StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using Smem = PassASmem<PA_STAGES>;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_PASS_A);
  const int u = a.u0 + blockIdx.y, sp = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nh = st.n_heads;
  const int nb = c.n_blocks[u];
  pdl_trigger();  // the selection may launch as this grid's last CTAs start
  int32_t* flow_cnt = st.flow ? st.flow + FLOW_PA_CNT * c.n_units + u : nullptr;
  int32_t* flow_done = st.flow ? st.flow + FLOW_PA_DONE * c.n_units + u : nullptr;
  // balanced partition of the unit's blocks over its splits (pa_splits)
  const int nsp = min(a.nsplit, nb);
  if (sp >= nsp) {
    if (flow_cnt) flow_arrive(flow_cnt, flow_done, gridDim.x, st.epoch);
    return;
  }
  const int b0 = (int)((long long)sp * nb / nsp);
  const int b1 = (int)((long long)(sp + 1) * nb / nsp);

  float* qh = Smem::QALIAS ? reinterpret_cast<float*>(S.stage[PA_WARPS - 1][PA_STAGES - 1]) : S.qh;
  for (int i = tid; i < H * D; i += blockDim.x) {
    int h = i / D;
    qh[i] = (h < nh) ? (float)(st.q[((size_t)u * nh + h) * D + (i % D)] * 0.08838834764831845)
                     : 0.f;
  }
  if (tid == 0) {
    for (int w = 0; w < PA_WARPS; ++w)
      for (int s = 0; s < PA_STAGES; ++s) mbar_init(&S.bar[w][s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int span = b1 - b0;
  const int nmine = (span > warp) ? (span - warp + PA_WARPS - 1) / PA_WARPS : 0;
  const uint8_t* ubase = c.tier1 + (size_t)u * c.max_blocks * REC;
  const float* smax_u = c.kscale_max + (size_t)u * c.max_blocks;
#ifdef PA_EVICT_FIRST
  // the Tier-1 stream is read once: evict it first so what selection and pass B
  // read next (l'_b, split states, score stash) stays in L2
  const uint64_t pol_ef = evict_first_policy();
#define PA_G2S(dst, src, bar) bulk_g2s_hint(dst, src, REC, bar, pol_ef)
#else
#define PA_G2S(dst, src, bar) bulk_g2s(dst, src, REC, bar)
#endif
  // the ring's first copies (all but the stage holding q'), then the fragments
  const bool last_w = warp == PA_WARPS - 1;
  if (lane == 0) {
    for (int s = 0; s < PA_STAGES && s < nmine; ++s) {
      if (Smem::QALIAS && last_w && s == PA_STAGES - 1) break;
      int b = b0 + warp + PA_WARPS * s;
      mbar_expect_tx(&S.bar[warp][s], REC);
      PA_G2S(S.stage[warp][s], ubase + (size_t)b * REC, &S.bar[warp][s]);
    }
  }
  QFrag f;
  load_qfrag(f, qh, lane);
  if (Smem::QALIAS) {
    fence_proxy_async();  // q' (generic writes) before the bulk copy that overwrites it
    __syncthreads();
  }
  if (Smem::QALIAS && last_w && lane == 0 && PA_STAGES - 1 < nmine) {
    const int s = PA_STAGES - 1;
    mbar_expect_tx(&S.bar[warp][s], REC);
    PA_G2S(S.stage[warp][s], ubase + (size_t)(b0 + warp + PA_WARPS * s) * REC, &S.bar[warp][s]);
  }

  const int h = lane & 3;
  const int t0 = lane >> 2;
  const int pi0 = 4 * (t0 >> 1) + (t0 & 1);  // permuted positions of tokens t0, t0 + 8
  const int pi1 = pi0 + 2;
  const int hb = lane >> 3;                  // head of this lane's B column
  const bool lo_lane = (lane >> 2) & 1;
  const int Sx = value_exp(c.v_max[u]);
  const float p2S = pow2f(Sx);
  float m_run = ninf(), l_run = 0.f, dmax = 0.f;
  float acc[NG][4], accz[4];
#pragma unroll
  for (int g = 0; g < NG; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
  accz[0] = accz[1] = accz[2] = accz[3] = 0.f;

  float* lm1 = st.lm1 + ((size_t)u * nh + (h < nh ? h : 0)) * c.max_blocks;
  // stash threshold of this lane's head: the previous step's largest tail l' minus a
  // margin (+inf before the first step or without a stash)
  float sthr = __int_as_float(0x7f800000);
  if (st.stash && h < nh) {
    const HeadState& hp = *reinterpret_cast<const HeadState*>(st.head_state + ((size_t)u * nh + h) * CKV_HEAD_FLOATS);
    if (hp.kprime > 0) sthr = hp.tailmax - st.stash_margin;
  }
  float* stash_u = st.stash ? st.stash + (size_t)u * c.max_blocks * 64 : nullptr;

  float smax_nxt = (nmine > 0) ? __ldg(smax_u + b0 + warp) : 0.f;
  for (int i = 0; i < nmine; ++i) {
    const int s = i % PA_STAGES;
    const uint32_t par = (uint32_t)(i / PA_STAGES) & 1u;
    const int b = b0 + warp + PA_WARPS * i;
    const float smax = smax_nxt;  // loaded one iteration ahead
    if (i + 1 < nmine) smax_nxt = __ldg(smax_u + b + PA_WARPS);
    mbar_wait(&S.bar[warp][s], par);
    const uint8_t* rec = S.stage[warp][s];

    // ---- phase 1: scores, block statistics --------------------------------
    BlockScores r = phase1_block(f, rec, smax, lane);
    float bm = fmaxf(r.s0, r.s1);
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
    const float e0 = fast_exp(r.s0 - bm), e1 = fast_exp(r.s1 - bm);
    float bs = e0 + e1;
    bs += __shfl_xor_sync(0xffffffffu, bs, 4);
    bs += __shfl_xor_sync(0xffffffffu, bs, 8);
    bs += __shfl_xor_sync(0xffffffffu, bs, 16);
    bool cand = false;
    if (lane < nh) {
      const float lb = bm + __logf(bs);
      lm1[b] = lb;
      cand = lb > sthr;
    }
    // likely promoted for some head: keep that head's scores for pass B
    const uint32_t smask = stash_u ? (__ballot_sync(0xffffffffu, cand) & 0xfu) : 0u;
    if (smask) {
      if ((smask >> h) & 1u) {
        stash_u[(size_t)b * 64 + h * 16 + t0] = r.s0;
        stash_u[(size_t)b * 64 + h * 16 + t0 + 8] = r.s1;
      }
      if (lane == 0) st.stash_epoch[(size_t)u * c.max_blocks + b] = (st.epoch << 4) | (int)smask;
    }
    dmax = fmaxf(dmax, r.delta);
    const float m_new = fmaxf(m_run, bm);
    const float alpha = fast_exp(m_run - m_new);
    const float beta = fast_exp(bm - m_new) * p2S;
    l_run = l_run * alpha + bs * beta;
    m_run = m_new;
    S.pbuf[warp][h][pi0] = e0 * beta;
    S.pbuf[warp][h][pi1] = e1 * beta;
    // rescale this lane's accumulators (all belong to head l%4)
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        acc[g][0] *= alpha; acc[g][1] *= alpha; acc[g][2] *= alpha; acc[g][3] *= alpha;
      }
      accz[0] *= alpha; accz[1] *= alpha; accz[2] *= alpha; accz[3] *= alpha;
    }
    __syncwarp();

    // ---- speculative phase 2 on the tensor cores -----------------------------
    PVFrag F;
    pv_frag(F, *reinterpret_cast<const float4*>(&S.pbuf[warp][hb][4 * (lane & 3)]), lo_lane);
    pv_block_sub(acc, accz, F, rec, lane);
    __syncwarp();
    // refill the stage: it is only ever read by this warp's generic loads (all
    // consumed before the __syncwarp above) and written by the bulk copy, so no
    // proxy fence is needed (write-after-read, no generic writes to order)
    if (lane == 0 && i + PA_STAGES < nmine) {
      mbar_expect_tx(&S.bar[warp][s], REC);
      PA_G2S(S.stage[warp][s], ubase + (size_t)(b + PA_WARPS * PA_STAGES) * REC, &S.bar[warp][s]);
    }
  }

  // ---- per-lane outputs: O[c][h] = (acc * 2^24 + offset sum) * 2^-S ----------
  const float oz = accz[0] + accz[1];  // group l/4, head l%4
  const float inv = pow2f(-Sx);
  // ---- merge the four warps of the CTA, write the split state ---------------
  __syncthreads();
  float* mw = reinterpret_cast<float*>(S.stage);        // [warp][h][4]: m, l, dmax
  float* ow = mw + PA_WARPS * H * 4;                     // [warp][h][D]
  if (lane < H) {
    mw[(warp * H + lane) * 4 + 0] = m_run;
    mw[(warp * H + lane) * 4 + 1] = l_run * inv;
    mw[(warp * H + lane) * 4 + 2] = dmax;
  }
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const float zg = __shfl_sync(0xffffffffu, oz, 4 * g + h);
    const int c0 = 16 * g + t0;
    ow[(warp * H + h) * D + c0] = fmaf(acc[g][0] + acc[g][1], 16777216.f, zg) * inv;
    ow[(warp * H + h) * D + c0 + 8] = fmaf(acc[g][2] + acc[g][3], 16777216.f, zg) * inv;
  }
  __syncthreads();
  for (int ch = tid; ch < D; ch += PA_WARPS * 32) {
  for (int hh = 0; hh < H; ++hh) {
    float M = ninf(), dm = 0.f;
    for (int w = 0; w < PA_WARPS; ++w) {
      M = fmaxf(M, mw[(w * H + hh) * 4 + 0]);
      dm = fmaxf(dm, mw[(w * H + hh) * 4 + 2]);
    }
    float L = 0.f, O = 0.f;
    if (M != ninf()) {
      for (int w = 0; w < PA_WARPS; ++w) {
        const float mwv = mw[(w * H + hh) * 4 + 0];
        if (mwv == ninf()) continue;
        const float sc = fast_exp(mwv - M);
        L += mw[(w * H + hh) * 4 + 1] * sc;
        O += ow[(w * H + hh) * D + ch] * sc;
      }
    }
    float* outp = st.split_state + (((size_t)u * st.n_splits + sp) * H + hh) * CKV_SPLIT_FLOATS;
    if (ch == 0) {
      outp[0] = M;
      outp[1] = L;
      outp[2] = dm;
      outp[3] = 0.f;
    }
    outp[4 + ch] = O;
  }
  }
  if (flow_cnt) flow_arrive(flow_cnt, flow_done, gridDim.x, st.epoch);
}

// =============================================================================
// select
// =============================================================================
constexpr int SEL_THREADS = 256;
constexpr int SEL_MAXSORT = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* total) {
  // 512 threads; returns exclusive prefix of v, writes the block total
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (int)(blockDim.x >> 5)) wsum[lane] = w;
    if (lane == (int)(blockDim.x >> 5) - 1) *total = w;
  }
  __syncthreads();
  int before = (warp > 0) ? wsum[warp - 1] : 0;
  int r = before + x - v;
  __syncthreads();
  return r;
}

// Block reductions: every warp folds the per-warp partials itself, lane w taking
// warp w's, with the same xor butterfly (addition is commutative, so all threads
// hold the same bits), two barriers per call.
__device__ __forceinline__ double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum_d(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
  t = warp_sum_d(t);
  __syncthreads();
  return t;
}

__device__ __forceinline__ float block_max_f(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : ninf();
  t = warp_max(t);
  __syncthreads();
  return t;
}

// two maxima in one barrier round (red: 2 x 32 floats)
__device__ __forceinline__ float2 block_max_f2(float a, float b, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_max(a);
  b = warp_max(b);
  if (lane == 0) {
    red[warp] = a;
    red[32 + warp] = b;
  }
  __syncthreads();
  const bool in = lane < (int)(blockDim.x >> 5);
  const float ta = warp_max(in ? red[lane] : ninf()), tb = warp_max(in ? red[32 + lane] : ninf());
  __syncthreads();
  return make_float2(ta, tb);
}

// The small fields first, then the arrays; the radix histogram and the coverage
// prefix are live in different phases and share storage.  The union builder at
// the end (last q-head CTA of a unit) uses everything from `big` on as its bitmap
// scratch: sel_body_bytes() sizes the dynamic allocation for it.
struct SelSmem {
  float qv[D];
  float ps[B];
  int wsum[32];
  int wsum2[32];
  int misc[16];
  uint32_t krange[2];
  double redd[40];
  float redf[40];
  union {
    int hist[2048];                       // radix-select histogram
    double cum[SEL_MAXSORT];              // coverage prefix (after the sort)
  } __align__(16);
  unsigned long long cand[SEL_MAXSORT];   // candidates (block order)
  unsigned long long sortk[SEL_MAXSORT];  // candidates sorted descending
};
__host__ __device__ inline size_t sel_body_bytes(int max_blocks) {
  const size_t ub = (size_t)2 * H * ((max_blocks + 31) / 32) * 4;  // build_union's bitmaps
  const size_t need = offsetof(SelSmem, hist) + ub;
  const size_t body = need > sizeof(SelSmem) ? need : sizeof(SelSmem);
  return (body + 15) & ~(size_t)15;
}

// Phase profile of k_select (build with -DCKV_SELPROF; tools/selprof.py): thread 0
// of every CTA adds globaltimer deltas between barrier-fenced markers.
#ifdef CKV_SELPROF
__device__ unsigned long long g_selprof[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define SELPROF(i) do { __syncthreads(); if (threadIdx.x == 0) { unsigned long long t_ = gtimer(); atomicAdd(&g_selprof[i], t_ - t_prev); t_prev = t_; } __syncthreads(); } while (0)
extern "C" void ckv_debug_selprof(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_selprof, sizeof(g_selprof)); }
#else
#define SELPROF(i) do {} while (0)
#endif

template <int KPT, int NT>
#ifndef SEL_MINB
#define SEL_MINB 4  // 64 registers (some spills) but 32 warps per SM: measured faster than 2
#endif
__global__ void __launch_bounds__(NT, NT == 256 ? SEL_MINB : (NT == 512 ? 2 : 1)) k_select(StepArgs a) {
#ifdef CKV_SELPROF
  unsigned long long t_prev = gtimer();
#endif
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SelSmem& S = *reinterpret_cast<SelSmem*>(smem_raw);
  const ckv_cache& c = a.c;
  uint32_t* fmask = reinterpret_cast<uint32_t*>(smem_raw + sel_body_bytes(c.max_blocks));
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_SELECT);
  const ckv_policy& pol = a.pol;
  const int h = blockIdx.x, u = a.u0 + blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nh = st.n_heads;
  const int nb = c.n_blocks[u];
  const int pl = c.partial_len[u];
  const size_t hu = (size_t)u * nh + h;
  const float* lm = st.lm1 + hu * c.max_blocks;
  HeadState& hs = *reinterpret_cast<HeadState*>(st.head_state + hu * CKV_HEAD_FLOATS);
  pdl_trigger();
  if (st.flow) flow_wait(st.flow + FLOW_PA_DONE * c.n_units + u, st.epoch);  // this unit's pass A
#ifdef CKV_SELPROF
  t_prev = gtimer();  // the profile starts once the unit's pass A is done
#endif

  // the eta annotations (tail pass) and this head's pass-A split states (merge) are
  // needed later: start pulling them into L2 now
  if (tid == 0) {
    prefetch_l2(c.eta + (size_t)u * c.max_blocks, (uint32_t)nb * 4u);
    prefetch_l2(st.split_state + (size_t)u * st.n_splits * H * CKV_SPLIT_FLOATS,
                (uint32_t)min(a.nsplit, nb) * H * CKV_SPLIT_FLOATS * 4u);
  }
  // ---- this thread's blocks tid + NT * j (j < KPT): order keys of l'_b in
  // registers; strided ownership keeps every load coalesced
#define BJ(j) (tid + NT * (j))
  uint32_t kk[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) kk[j] = (BJ(j) < nb) ? okey(__ldcg(lm + BJ(j))) : 0u;

  // ---- the pass-A split states, loaded right away (their latency overlaps the
  // keys'): thread (g, d) merges splits g, g + SG, ... online, the SG group
  // partials are combined after the barrier below
  constexpr int SG = NT / D;
  const int nsp = min(a.nsplit, nb);
  float* mrg = reinterpret_cast<float*>(S.cand);  // [SG][D] O, then [SG] m, l, delta (free until the gather)
  {
    const int g = tid / D, d = tid % D;
    const float* spb = st.split_state + (((size_t)u * st.n_splits) * H + h) * CKV_SPLIT_FLOATS;
    float m_t = ninf(), l_t = 0.f, o_t = 0.f, d_t = 0.f;
    constexpr int MU = KPT <= 16 ? 4 : 1;  // splits in flight per thread (register budget)
    for (int s0 = g; s0 < nsp; s0 += SG * MU) {
      float m[MU], l[MU], dl[MU], o[MU];
#pragma unroll
      for (int q = 0; q < MU; ++q) {
        const float* sp = spb + (size_t)(s0 + q * SG) * H * CKV_SPLIT_FLOATS;
        const bool ok = s0 + q * SG < nsp;
        m[q] = ok ? sp[0] : ninf();
        l[q] = ok ? sp[1] : 0.f;
        dl[q] = ok ? sp[2] : 0.f;
        o[q] = ok ? sp[4 + d] : 0.f;
      }
#pragma unroll
      for (int q = 0; q < MU; ++q) {
        d_t = fmaxf(d_t, dl[q]);
        if (m[q] != ninf()) {
          const float mn = fmaxf(m_t, m[q]);
          const float a0 = (m_t == ninf()) ? 0.f : expf(m_t - mn), a1 = expf(m[q] - mn);
          l_t = fmaf(l_t, a0, l[q] * a1);
          o_t = fmaf(o_t, a0, o[q] * a1);
          m_t = mn;
        }
      }
    }
    mrg[g * D + d] = o_t;
    if (d == 0) {
      mrg[SG * D + g] = m_t;
      mrg[SG * D + SG + g] = l_t;
      mrg[SG * D + 2 * SG + g] = d_t;
    }
  }
  if (tid < D) S.qv[tid] = (float)(st.q[hu * D + tid] * 0.08838834764831845);
  for (int i = tid; i < (c.max_blocks + 31) / 32; i += NT) fmask[i] = 0u;
  __syncthreads();
  if (tid < D) {  // combine the SG group partials of the pass-A splits
    float M = ninf(), dm = 0.f;
#pragma unroll
    for (int g = 0; g < SG; ++g) {
      M = fmaxf(M, mrg[SG * D + g]);
      dm = fmaxf(dm, mrg[SG * D + 2 * SG + g]);
    }
    float L = 0.f, O = 0.f;
    if (M != ninf()) {
#pragma unroll
      for (int g = 0; g < SG; ++g) {
        const float mg = mrg[SG * D + g];
        const float sc = (mg == ninf()) ? 0.f : expf(mg - M);
        L = fmaf(mrg[SG * D + SG + g], sc, L);
        O = fmaf(mrg[g * D + tid], sc, O);
      }
    }
    hs.oA[tid] = O;
    if (tid == 0) {
      hs.mA = M;
      hs.lA = L;
      hs.delta = dm;
    }
  }

  SELPROF(1);
  // ---- partial block on originals (attention.py:98-104) ------------------------
  for (int t = warp; t < pl; t += NT / 32) {
    const uint16_t* pk = c.partial_k + ((size_t)u * B + t) * D;
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      acc = fmaf(__half2float(__ushort_as_half(pk[lane * 4 + j])), S.qv[lane * 4 + j], acc);
    acc = warp_sum(acc);
    if (lane == 0) S.ps[t] = acc;
  }
  __syncthreads();
  float mp = ninf(), lp = 0.f;
  for (int t = 0; t < pl; ++t) mp = fmaxf(mp, S.ps[t]);
  for (int t = 0; t < pl; ++t) lp += expf(S.ps[t] - mp);
  const float lmp = (pl > 0) ? mp + logf(lp) : ninf();
  if (tid < D) {
    float acc = 0.f;
    for (int t = 0; t < pl; ++t)
      acc = fmaf(expf(S.ps[t] - mp),
                 __half2float(__ushort_as_half(c.partial_v[((size_t)u * B + t) * D + tid])), acc);
    hs.np_[tid] = acc;
  }

  SELPROF(2);
  if (tid == 0) {
    hs.mp = mp;
    hs.lp = lp;
  }
  SELPROF(3);
  // ---- lse over l'_b and the partial (attention.py:170-179) ------------------------
  // (with the key range the radix select starts from: one barrier round)
  float lmax = lmp;
  uint32_t kmn_r = 0xffffffffu, kmx_r = 0u;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    if (BJ(j) < nb) {
      lmax = fmaxf(lmax, ukey(kk[j]));
      kmn_r = min(kmn_r, kk[j]);
      kmx_r = max(kmx_r, kk[j]);
    }
  }
  lmax = warp_max(lmax);
  kmn_r = __reduce_min_sync(0xffffffffu, kmn_r);
  kmx_r = __reduce_max_sync(0xffffffffu, kmx_r);
  if (lane == 0) {
    S.redf[warp] = lmax;
    S.wsum[warp] = (int)kmn_r;
    S.wsum2[warp] = (int)kmx_r;
  }
  __syncthreads();
  {
    const bool in = lane < NT / 32;
    lmax = warp_max(in ? S.redf[lane] : ninf());
    kmn_r = __reduce_min_sync(0xffffffffu, in ? (uint32_t)S.wsum[lane] : 0xffffffffu);
    kmx_r = __reduce_max_sync(0xffffffffu, in ? (uint32_t)S.wsum2[lane] : 0u);
  }
  if (tid == 0) {  // read again by the radix select (behind block_sum_d's barriers)
    S.krange[0] = kmn_r;
    S.krange[1] = kmx_r;
  }
  float sef = 0.f;
  const float lmax2 = lmax * 1.4426950408889634f;
#pragma unroll
  for (int j = 0; j < KPT; ++j)
    sef += (BJ(j) < nb) ? ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lmax2)) : 0.f;
  double se = block_sum_d((double)sef, S.redd);
  if (pl > 0) se += exp((double)lmp - (double)lmax);
  const double lse = (double)lmax + log(se);
  const float lsef = (float)lse;
  const double pmass = (pl > 0) ? exp((double)lmp - lse) : 0.0;
  // the reference orders fp64 masses exp(l' - lse) (attention.py:183): masses that
  // underflow to exactly 0 there (l' - lse < -745.13) tie and keep block order, so
  // the selection gives all of them one key just below every other key
  const uint32_t zk = okey((float)(lse - 745.1332191019412));
  auto skey = [&](int j) -> uint32_t { return kk[j] < zk ? zk - 1u : kk[j]; };

  SELPROF(4);
  // ---- top K_sel blocks by l' (ties -> lower index) -------------------------------
  // T = the K_sel-th largest key by a 3-digit (11/11/10 bit) radix select over
  // shared histograms, then the candidates (all keys > T, the first keys == T
  // in block order) are sorted descending by (key, -block) with a bitonic sort.
  // the sorted prefix covers every block that can be promoted (K' <= 2 K_max
  // with rung 1); the largest tail key comes from a reduction below
  const int kwant = pol.rung1_enabled ? 2 * pol.k_max : pol.k_max;
  const int ksel = min(nb, min(kwant, SEL_MAXSORT));
#ifndef SEL_SORTCAP
#define SEL_SORTCAP 384
#endif
  const int sort_cap = max(ksel, SEL_SORTCAP);  // candidates allowed into the rank sort
  int n_sorted = 0;
  if (ksel > 0) {
    // digits of (key - min key), 11 bits at a time from the top of the occupied
    // range, so the first histogram spreads over the keys actually present
    // skey is monotone in the key: the range of skey is skey of the key range
    const uint32_t kmn = S.krange[0] < zk ? zk - 1u : S.krange[0];
    const uint32_t kmx = S.krange[1] < zk ? zk - 1u : S.krange[1];
    const int nbits = (kmx > kmn) ? 32 - __clz(kmx - kmn) : 0;
    // Radix passes until the keys >= the current bin's lower edge number at
    // most SEL_MAXSORT (normally one pass): those are the candidates, sorted
    // below.  Only when a single key value holds too many blocks does the
    // exact K_sel-th key T and its tie rule (lower block index first) apply.
    uint32_t prefix = 0, pmask = 0;
    int need = ksel, above = 0, n_cand = nb;
    bool exact = nb > sort_cap;
    for (int top = nbits; top > 0 && exact;) {
      const int shift = max(top - 11, 0);
      const int nbins = 1 << (top - shift);
      for (int i = tid; i < 2048; i += NT) S.hist[i] = 0;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const uint32_t rel = skey(j) - kmn;
        const bool in = BJ(j) < nb && (rel & pmask) == prefix;
        if (in) atomicAdd(&S.hist[(rel >> shift) & (uint32_t)(nbins - 1)], 1);
      }
      __syncthreads();
      // suffix counts from the top bin down: thread t owns bins [hi-per, hi)
      const int per = (nbins + NT - 1) / NT;
      const int hi_bin = nbins - tid * per;
      int loc = 0;
      for (int i = 1; i <= per; ++i)
        if (hi_bin - i >= 0) loc += S.hist[hi_bin - i];
      const int before = block_excl_scan(loc, S.wsum, &S.misc[8]);  // count in higher bins
      if (before < need && before + loc >= need) {
        int run = before;
        for (int i = 1; i <= per; ++i) {
          const int cnt = S.hist[hi_bin - i];
          if (run + cnt >= need) {
            S.misc[0] = hi_bin - i;
            S.misc[1] = run;
            S.misc[2] = cnt;
            break;
          }
          run += cnt;
        }
      }
      __syncthreads();
      const uint32_t dgt = (uint32_t)S.misc[0];
      const int run = S.misc[1], binc = S.misc[2];
      __syncthreads();
      above += run;
      need -= run;
      prefix |= dgt << shift;
      pmask |= (uint32_t)(nbins - 1) << shift;
      top = shift;
      if (above + binc <= sort_cap) {
        exact = false;
        n_cand = above + binc;
      }
    }
    SELPROF(8);
    const uint32_t T = kmn + prefix;
    if (!exact) {
      // candidates: every key >= T (the lower edge of the last bin), block order
      int nc = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) nc += (BJ(j) < nb && skey(j) >= T);
      int pc = block_excl_scan(nc, S.wsum, &S.misc[3]);
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const int b = BJ(j);
        if (b < nb && skey(j) >= T)
          S.cand[pc++] = ((unsigned long long)skey(j) << 32) |
                         (unsigned long long)(0xffffffffu - (uint32_t)b);
      }
      n_sorted = n_cand;
    } else {
      // T is the K_sel-th largest key itself: all keys > T, then the first == T
      // in block order; blocks run j-major (BJ), so one scan per j (rare path)
      int ngt = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) ngt += (BJ(j) < nb && skey(j) > T);
      int pg = block_excl_scan(ngt, S.wsum, &S.misc[2]);
      const int tot_gt = S.misc[2];
#pragma unroll
      for (int j = 0; j < KPT; ++j)
        if (BJ(j) < nb && skey(j) > T)
          S.cand[pg++] = ((unsigned long long)skey(j) << 32) |
                         (unsigned long long)(0xffffffffu - (uint32_t)BJ(j));
      int taken = tot_gt;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        if (taken >= ksel) continue;  // uniform across the block
        const bool eq = BJ(j) < nb && skey(j) == T;
        const int pos = taken + block_excl_scan((int)eq, S.wsum, &S.misc[3]);
        const int cnt = S.misc[3];
        if (eq && pos < ksel)
          S.cand[pos] = ((unsigned long long)skey(j) << 32) |
                        (unsigned long long)(0xffffffffu - (uint32_t)BJ(j));
        taken += cnt;
      }
      n_sorted = ksel;
    }
    __syncthreads();
    SELPROF(10);
    // rank sort (composite keys are distinct): position = #greater; the
    // candidate list is read as broadcast 16-byte pairs (a thread per candidate
    // measured faster than warp-cooperative variants)
    // (a thread per candidate, the list read as broadcast 16-byte pairs: measured
    // faster than splitting a candidate's count over several lanes)
    const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(S.cand);
    for (int i = tid; i < n_sorted; i += NT) {
      const unsigned long long x = S.cand[i];
      int r = 0;
      int j = 0;
#pragma unroll 4
      for (; j + 1 < n_sorted; j += 2) {
        const ulonglong2 y = c2[j >> 1];
        r += (y.x > x) + (y.y > x);
      }
      if (j < n_sorted) r += (S.cand[j] > x);
      S.sortk[r] = x;
    }
    __syncthreads();
  }

  SELPROF(5);
  // ---- coverage K, clamp, rung 1 (attention.py:180-203, fallback.py:134-138) --------
  for (int i = tid; i < n_sorted; i += NT) {
    S.cum[i] = (double)expf(ukey((uint32_t)(S.sortk[i] >> 32)) - lsef);
  }
  __syncthreads();
  // prefix sum in fp64 along the mass order: 32-entry chunks scanned by the warps
  // in parallel, then each chunk adds the carry pmass + T_0 + ... + T_{c-1} summed
  // in chunk order (the same operations as one warp walking the chunks)
  const int nchk = (n_sorted + 31) / 32;
  double* ctot = S.redd;  // chunk totals (<= 32)
  for (int ch = warp; ch < nchk; ch += NT / 32) {
    const int i = ch * 32 + lane;
    double x = (i < n_sorted) ? S.cum[i] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < n_sorted) S.cum[i] = x;
    if (lane == 31) ctot[ch] = x;
  }
  if (tid == 0) S.misc[4] = -1;
  __syncthreads();
  for (int ch = warp; ch < nchk; ch += NT / 32) {
    double carry = pmass;
    for (int c2 = 0; c2 < ch; ++c2) carry += ctot[c2];
    const int i = ch * 32 + lane;
    if (i < n_sorted) S.cum[i] = carry + S.cum[i];
  }
  __syncthreads();
  for (int i = tid; i < n_sorted; i += NT)
    if (S.cum[i] >= pol.tau_cov && (i == 0 || S.cum[i - 1] < pol.tau_cov)) S.misc[4] = i + 1;
  __syncthreads();
  if (tid == 0) {
    int kcov = S.misc[4];
    if (kcov < 0 && n_sorted == nb) kcov = nb;
    int kstar;
    if (nb == 0) {
      kstar = 0;
      kcov = 0;
    } else {
      const int kc_eff = (kcov < 0) ? 0x3fffffff : kcov;
      kstar = min(max(kc_eff, pol.k_min), min(pol.k_max, nb));
    }
    int kp = kstar;
    if (pol.rung1_enabled) kp = min(2 * kstar, nb);
    S.misc[4] = kcov;
    S.misc[5] = kstar;
    S.misc[6] = kp;
  }
  __syncthreads();
  const int kcov = S.misc[4], kstar = S.misc[5], kp = S.misc[6];
  int32_t* order = st.order + hu * st.kcap;
  for (int i = tid; i < kp; i += NT) {
    const int b = (int)(0xffffffffu - (uint32_t)(S.sortk[i] & 0xffffffffull));
    order[i] = b;
    atomicOr(&fmask[b >> 5], 1u << (b & 31));
  }
  __syncthreads();

  SELPROF(6);
  // ---- tail mass, rung 2, E_val tail (fallback.py:141-161, certifier.py:153-160) ----
  const bool r2 = pol.rung2_enabled != 0;
  const bool greedy = r2 && pol.greedy_value_budget >= 0.0;
  // greedy budget mode: promote in descending p*eta (ties -> lower index) while the
  // residual exceeds the budget; realised as a threshold T on the contribution key
  // (all keys > T, plus the first `take` keys == T in block order)
  // this thread's eta values, vector-loaded up front (one latency, not KPT)
  const float* eta = c.eta + (size_t)u * c.max_blocks;
  const float lse2 = lsef * 1.4426950408889634f;
  uint32_t gT = 0xffffffffu;
  int take = 0;
  float etv[KPT];  // greedy mode only (the threshold path loads eta in chunks)
  if (greedy) {
#pragma unroll
    for (int j = 0; j < KPT; ++j) etv[j] = (BJ(j) < nb) ? __ldg(eta + BJ(j)) : 0.f;
  }
  if (greedy && nb > 0) {
    double tot = 0.0;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (BJ(j) < nb) tot += (double)(ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lse2)) * etv[j]);
    tot = block_sum_d(tot, S.redd);
    const double need = tot - pol.greedy_value_budget;
    if (need > 0.0) {
      uint32_t lo = 0u;
      unsigned long long hi = 0x100000000ull;
      while (hi - lo > 1ull) {
        const uint32_t mid = (uint32_t)((lo + hi) >> 1);
        double g = 0.0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
          if (BJ(j) >= nb) continue;
          const float cj = ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lse2)) * etv[j];
          if (__float_as_uint(cj) >= mid) g += (double)cj;
        }
        g = block_sum_d(g, S.redd);
        if (g >= need) lo = mid;
        else hi = mid;
      }
      gT = lo;
      double ggt = 0.0;
      int neq = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        if (BJ(j) >= nb) continue;
        const float cj = ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lse2)) * etv[j];
        if (__float_as_uint(cj) > gT) ggt += (double)cj;
        neq += (__float_as_uint(cj) == gT);
      }
      ggt = block_sum_d(ggt, S.redd);
      const int eq_before = block_excl_scan(neq, S.wsum, &S.misc[9]);
      const double cT = (double)__uint_as_float(gT);
      int m = (cT > 0.0) ? (int)ceil((need - ggt) / cT) : 0;
      m = max(0, min(m, S.misc[9]));
      take = m - eq_before;  // how many of this thread's == T blocks are promoted
    }
  }
  // masses p_b = exp(l'_b - lse): fp32 via MUFU ex2, per-thread sums in fp32,
  // across threads in fp64
  const float vtol = (float)pol.v_tol;
  float atf = 0.f, etf = 0.f, tmx = ninf();
  int nv = 0;
  uint32_t vb[(KPT + 31) / 32];
#pragma unroll
  for (int w = 0; w < (KPT + 31) / 32; ++w) vb[w] = 0u;
  auto account = [&](int j, bool valid, float pf, float pe, bool inV) {
    const bool inF = valid && ((fmask[BJ(j) >> 5] >> (BJ(j) & 31)) & 1u);
    atf += inF ? 0.f : pf;
    tmx = fmaxf(tmx, (valid && !inF) ? ukey(kk[j]) : ninf());
    etf += (inF || inV) ? 0.f : pe;
    nv += inV;
    vb[j >> 5] |= (uint32_t)inV << (j & 31);
  };
  if (greedy) {
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      const bool valid = BJ(j) < nb;
      const float pf = valid ? ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lse2)) : 0.f;
      const float pe = pf * etv[j];
      const uint32_t ck = __float_as_uint(pe);
      const bool inV = valid && (gT != 0xffffffffu) && (ck > gT || (ck == gT && take-- > 0));
      account(j, valid, pf, pe, inV);
    }
  } else {
    // eta in chunks of 8 blocks per thread: bounded register pressure (the
    // memory clobber keeps the compiler from hoisting every load to the top)
#pragma unroll
    for (int j0 = 0; j0 < KPT; j0 += 8) {
      float ev[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) ev[jj] = (BJ(j0 + jj) < nb) ? __ldg(eta + BJ(j0 + jj)) : 0.f;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = j0 + jj;
        const bool valid = BJ(j) < nb;
        const float pf = valid ? ex2_approx(fmaf(ukey(kk[j]), 1.4426950408889634f, -lse2)) : 0.f;
        const float pe = pf * ev[jj];
        account(j, valid, pf, pe, r2 && valid && (pe > vtol));
      }
      asm volatile("" ::: "memory");
    }
  }
  // tail max, the two fp64 sums and the value-list scan in one barrier round; every
  // thread folds the per-warp partials in warp order (the order block_sum_d uses)
  double at, et;
  int vo, n_v;
  {
    const float tw = warp_max(tmx);  // largest phase-1 log-mass over the tail
    const double aw = warp_sum_d((double)atf), ew = warp_sum_d((double)etf);
    int x = nv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 0) {
      S.redf[warp] = tw;
      S.redd[warp] = aw;
      S.cum[warp] = ew;  // (free after the coverage scan)
    }
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    const bool in = lane < NT / 32;
    const float tm = warp_max(in ? S.redf[lane] : ninf());
    const double ta = warp_sum_d(in ? S.redd[lane] : 0.0), te = warp_sum_d(in ? S.cum[lane] : 0.0);
    int sc = in ? S.wsum[lane] : 0;  // inclusive scan of the warp counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += y;
    }
    const int tot = __shfl_sync(0xffffffffu, sc, 31);
    const int before = (warp > 0) ? __shfl_sync(0xffffffffu, sc, warp - 1) : 0;
    __syncthreads();
    tmx = tm;
    at = ta;
    et = te;
    vo = before + x - nv;
    n_v = tot;
  }
  {
    int32_t* vlist = st.vlist + hu * c.max_blocks;
    int pv = vo;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if ((vb[j >> 5] >> (j & 31)) & 1u) vlist[pv++] = BJ(j);
  }
  if (tid == 0) {
    hs.lse = lse;
    hs.alpha_hat = (kp >= nb) ? 0.0 : at;
    hs.e_tail = et;
    hs.partial_mass = pmass;
    hs.tailmax = (kp < nb) ? tmx : ninf();
    hs.kprime = kp;
    hs.kstar0 = kstar;
    hs.n_v = n_v;
    hs.k_cov = kcov;
    ckv_cert& ct = st.cert[hu];
    ct.partial_mass = pmass;
    ct.k_star = kp;
    ct.k_star0 = kstar;
    ct.k_coverage = kcov;
    ct.n_value_promoted = n_v;
    uint32_t fl = CKV_F_ACTIVE;
    if (pol.rung1_enabled && kp != kstar) fl |= CKV_F_RUNG1;
    if (n_v > 0) fl |= CKV_F_RUNG2;
    if (kcov != kstar) fl |= CKV_F_CLAMPED;
    ct.flags = fl;
  }
  SELPROF(7);
  // the last q-head of the unit to finish builds the unit's union work list
  if (st.unit_done) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(&st.unit_done[u], 1);
      last = (prev == nh - 1);
      if (last) st.unit_done[u] = 0;
      __threadfence();
    }
    __syncthreads();
    if (last) build_union(c, st, u, reinterpret_cast<uint32_t*>(S.hist), S.wsum);
    if (last) SELPROF(9);
    if (last && st.flow) {  // the unit's selection and union list are published
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release_gpu(st.flow + FLOW_SEL_DONE * c.n_units + u, st.epoch);
    }
  }
}

// =============================================================================
// kernel-backend plugin (pure.py:16-66) -- parity surface, not the hot path
// =============================================================================
__global__ void k_block_logmass(const double* s, const int64_t* bnd, int nb, double* bmax,
                                double* bsum, double* lmass) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int64_t lo = bnd[i], hi = bnd[i + 1];
  double m = -INFINITY;
  for (int64_t t = lo; t < hi; ++t) m = fmax(m, s[t]);
  double acc = 0.0;
  for (int64_t t = lo; t < hi; ++t) acc += exp(s[t] - m);
  bmax[i] = m;
  bsum[i] = acc;
  lmass[i] = m + log(acc);
}

__global__ void k_fused_attend(const float* s, const float* v, const int64_t* bnd, int nb, int d,
                               float* out, float* ml) {
  float m = -INFINITY, l = 0.f;
  const int ch = threadIdx.x;
  float o = 0.f;
  for (int i = 0; i < nb; ++i) {
    const int64_t lo = bnd[i], hi = bnd[i + 1];
    float mn = m;
    for (int64_t t = lo; t < hi; ++t) mn = fmaxf(mn, s[t]);
    const float sc = expf(m - mn);
    float w = 0.f;
    o *= sc;
    for (int64_t t = lo; t < hi; ++t) {
      const float p = expf(s[t] - mn);
      w += p;
      if (ch < d) o = fmaf(p, v[t * d + ch], o);
    }
    l = l * sc + w;
    m = mn;
  }
  if (ch < d) out[ch] = o / l;
  if (ch == 0) {
    ml[0] = m;
    ml[1] = l;
  }
}

// Clears the step's per-step status words before its kernels run: the Tier-2
// loss flag and (fused LRU accounting) the per-unit page stats.  A programmatic
// dependent of the previous kernel on the stream (which may still read them).
__global__ void k_step_begin(int32_t* status, int32_t* ps, int n_ps) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) status[CKV_ST_TIER2] = 0;
  for (int i = threadIdx.x; i < n_ps; i += blockDim.x) ps[i] = 0;
}

// =============================================================================
// launchers
// =============================================================================
cudaError_t launch_union(const ckv_cache*, const ckv_policy*, const ckv_step*, int, int, cudaStream_t);
cudaError_t launch_passb(const ckv_cache*, const ckv_policy*, const ckv_step*, const PageView&, int, int,
                         bool, bool, cudaStream_t);
cudaError_t launch_scratch(const ckv_cache*, const ckv_step*, const ckv_scratch*, int, int, cudaStream_t);

// a scratch that holds every block and has no HBM slots needs no separate LRU
// pass: pass B decides hit / miss per union item (same counts as k_lru_fast)
static bool lru_fused(const ckv_cache* c, const ckv_scratch* sc) {
  return lru_ring(c->max_blocks, sc->key_capacity) == 0 && lru_ring(c->max_blocks, sc->value_capacity) == 0 &&
         sc->key_capacity > 0 && sc->value_capacity > 0 && !sc->key_slots && !sc->value_slots &&
         !knobs().separate_lru;
}

// Everything after pass A for units [u0, u0 + nu): selection, the union work
// list, LRU scratch (+ page-in), pass B, combine.
static cudaError_t launch_tail(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st,
                               const ckv_scratch* sc, int host_max_blocks, int u0, int nu,
                               int nsplit, bool finish, cudaStream_t s) {
  StepArgs a{*c, *st, *pol, PageView{}, u0, 0, nsplit};
  const size_t smS = sel_body_bytes(c->max_blocks) + ((c->max_blocks + 31) / 32) * 4;
  const int nbh = host_max_blocks;  // selection only touches the filled blocks
  // few (unit, head) CTAs (e.g. 8-way KV-head sharding): 1024 threads per head, so
  // each CTA's serial phases are shorter; otherwise 256 threads, 4 CTAs per SM
  const long long plan_u = st->plan_units > 0 ? st->plan_units : nu;
  // variant: keys per thread x threads per (unit, head) CTA.  Few CTAs (e.g. 8-way
  // KV-head sharding): 1024 threads, so the serial phases of each CTA are short;
  // many: 256 threads and 4 CTAs per SM up to 8192 blocks, 512 threads beyond
  // (more keys per thread would spill)
  int kpt, nt;
  if (knobs().sel_kpt > 0) {
    kpt = knobs().sel_kpt;
    nt = knobs().sel_nt;
  } else if (plan_u * st->n_heads <= 2 * 148) {
    nt = 1024;
    kpt = nbh <= 1024 * 8 ? 8 : (nbh <= 1024 * 16 ? 16 : 32);
  } else if (nbh <= SEL_THREADS * 32) {
    nt = SEL_THREADS;
    kpt = nbh <= SEL_THREADS * 8 ? 8 : (nbh <= SEL_THREADS * 16 ? 16 : 32);
  } else {
    nt = 512;
    kpt = nbh <= 512 * 32 ? 32 : 64;
  }
  const dim3 gs(st->n_heads, nu);
  const bool pdl = st->flow != nullptr;  // overlaps pass A's last wave (flow_wait per unit)
  cudaError_t le = cudaErrorInvalidConfiguration;
#define SEL_CASE(K, T) \
  if (kpt == K && nt == T) le = launch_k(pdl, k_select<K, T>, gs, dim3(T), smS, s, a); else
  SEL_CASE(8, 1024) SEL_CASE(16, 1024) SEL_CASE(32, 1024)
  SEL_CASE(8, 256) SEL_CASE(16, 256) SEL_CASE(32, 256) SEL_CASE(64, 256) SEL_CASE(128, 256)
  SEL_CASE(16, 512) SEL_CASE(32, 512) SEL_CASE(64, 512) {}
#undef SEL_CASE
  if (le != cudaSuccess) return le;
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (!st->unit_done) {  // otherwise built by the last selection CTA of each unit
    e = launch_union(c, pol, st, u0, nu, s);
    if (e != cudaSuccess) return e;
  }
  PageView pv{};
  bool pdl_b = st->unit_done != nullptr;  // pass B directly behind the selection
  if (sc) {
    const bool fuse = lru_fused(c, sc);
    pdl_b = pdl_b && fuse;
    if (fuse) {  // page_stats zeroed before pass A (launch_decode)
      pv.fused = 1;
      pv.klru = sc->key_lru;
      pv.vlru = sc->value_lru;
      pv.counters = sc->counters;
      pv.page_stats = st->page_stats;
    } else {
      e = launch_scratch(c, st, sc, u0, nu, s);  // LRU accounting (+ side-stream page-in into slots)
      if (e != cudaSuccess) return e;
    }
    pv.kslots = sc->key_slots;
    pv.vslots = sc->value_slots;
    pv.kcap = sc->key_capacity;
    pv.vcap = sc->value_capacity;
    pv.kstride = lru_words(c->max_blocks, sc->key_capacity);
    pv.vstride = lru_words(c->max_blocks, sc->value_capacity);
    pv.kslot_of = sc->key_lru + lru_slot_offset(c->max_blocks, sc->key_capacity);
    pv.vslot_of = sc->value_lru + lru_slot_offset(c->max_blocks, sc->value_capacity);
  }
  return launch_passb(c, pol, st, pv, u0, nu, pdl_b, finish, s);
}

// Optional unit chunks (CKV_CHUNKS=n): pass A of chunk k+1 runs while the
// tail of chunk k runs on a second, high-priority stream.  Units are
// independent, so the result is identical to one launch over all units.  Off
// by default: pass A fills every SM's register file (4 x 128 threads x 126
// registers), so tail CTAs displace pass-A CTAs instead of filling gaps
// (measured at C3: 1 chunk 2.47 ms, 2 chunks 2.53, 4 chunks 2.69).
static int decode_chunks(int n_units) {
  int n = knobs().chunks;
  if (n_units < 16) n = 1;
  return max(1, min(n, n_units));
}

// Pass-A splits per unit: a balanced partition of the unit's blocks whose CTA
// count (units x splits) fills the SMs' pass-A slots in whole waves -- a last
// wave that is half empty costs up to 1 / (2 x waves) of the stream (14% at 32
// units x 128K).  Splits of 64..512 blocks; the fewest splits of <= 256 blocks
// that keep >= 97% of the slots busy, else the best-filled count.
static int pa_splits(long long units, int nb, int cap, int sms) {
  if (nb <= 0) return 1;
  const long long slots = (long long)sms * PA_MINB;
  const int lo = max(1, (nb + 511) / 512), base = max(1, (nb + 255) / 256);
  const int hi = max(1, min(cap, (nb + 63) / 64));
  int best = min(base, hi);
  double best_eff = -1.0;
  for (int s = lo; s <= hi; ++s) {
    const long long ctas = units * s;
    const long long waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (s >= base && eff >= 0.97) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// whether launch_decode runs the step as a dataflow (see flow_wait / flow_arrive)
bool decode_flow(const ckv_cache* c, const ckv_step* st) {
  return st->flow && st->unit_done && !st->queue && decode_chunks(c->n_units) == 1;
}

cudaError_t launch_decode(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st,
                          const ckv_scratch* sc, int host_max_blocks, bool finish, cudaStream_t s) {
  g_launches = 0;
  const size_t smA2 = sizeof(PassASmem<2>), smA3 = sizeof(PassASmem<3>);
  set_max_dyn_smem(k_pass_a<2>, (int)smA2);
  set_max_dyn_smem(k_pass_a<3>, (int)smA3);
  {
    const int smS = (int)(sel_body_bytes(c->max_blocks) + ((c->max_blocks + 31) / 32) * 4);
    set_max_dyn_smem(k_select<8, 1024>, smS);
    set_max_dyn_smem(k_select<16, 1024>, smS);
    set_max_dyn_smem(k_select<32, 1024>, smS);
    set_max_dyn_smem(k_select<8, SEL_THREADS>, smS);
    set_max_dyn_smem(k_select<16, SEL_THREADS>, smS);
    set_max_dyn_smem(k_select<32, SEL_THREADS>, smS);
    set_max_dyn_smem(k_select<64, SEL_THREADS>, smS);
    set_max_dyn_smem(k_select<128, SEL_THREADS>, smS);
    set_max_dyn_smem(k_select<16, 512>, smS);
    set_max_dyn_smem(k_select<32, 512>, smS);
    set_max_dyn_smem(k_select<64, 512>, smS);
  }
  const int U = c->n_units;
  const int nch = decode_chunks(U);
  const int per = (U + nch - 1) / nch;
  const int nsplit = pa_splits(st->plan_units > 0 ? st->plan_units : U, host_max_blocks, st->n_splits,
                               dev_state().sms);
  const int nsplit_used = min(nsplit, host_max_blocks);
  cudaStream_t s2 = (nch > 1) ? dev_state().tail : s;
  cudaError_t e = cudaSuccess;
  {  // the step's per-step words: Tier-2 loss (reported per step), the fused LRU's page stats
    int32_t* ps = (sc && lru_fused(c, sc)) ? st->page_stats : nullptr;
    e = launch_k(true, k_step_begin, dim3(1), dim3(256), 0, s, c->status, ps, ps ? 4 * U : 0);
    ++g_launches;
    if (e != cudaSuccess) return e;
  }
  // the kernel dataflow needs the selection to build the union list and one
  // unit chunk per step (the chunked overlap puts events between the kernels)
  ckv_step stf = *st;
  if (!decode_flow(c, st)) stf.flow = nullptr;
  st = &stf;
  if (st->prof_begin) cudaEventRecord(reinterpret_cast<cudaEvent_t>(st->prof_begin), s);
  cudaEvent_t evs[64];
  int nev = 0;
  for (int k = 0; k < nch; ++k) {
    const int u0 = k * per, nu = min(per, U - u0);
    if (nu <= 0) break;
    StepArgs a{*c, *st, *pol, PageView{}, u0, 0, nsplit};
    if (nsplit_used > 0 || st->flow) {  // with the dataflow every unit's pass A must publish
      // behind k_step_begin (k == 0, no event in between) as a programmatic dependent:
      // that kernel does not trigger early, so pass A starts when it has finished
      const bool pdl = k == 0 && !st->prof_begin;
      const long long ctas = (long long)max(nsplit_used, 1) * nu;
      if (ctas >= PA_DEEP_WAVES * (long long)dev_state().sms * PA_MINB)
        e = launch_k(pdl, k_pass_a<3>, dim3(max(nsplit_used, 1), nu), dim3(PA_WARPS * 32), smA3, s, a);
      else
        e = launch_k(pdl, k_pass_a<2>, dim3(max(nsplit_used, 1), nu), dim3(PA_WARPS * 32), smA2, s, a);
      ++g_launches;
      if (e != cudaSuccess) break;
    }
    if (k == nch - 1 || u0 + nu >= U) {
      if (st->prof_end) cudaEventRecord(reinterpret_cast<cudaEvent_t>(st->prof_end), s);
    }
    if (nch > 1) {
      cudaEventCreateWithFlags(&evs[nev], cudaEventDisableTiming);
      cudaEventRecord(evs[nev], s);
      cudaStreamWaitEvent(s2, evs[nev], 0);
      ++nev;
    }
    e = launch_tail(c, pol, st, sc, host_max_blocks, u0, nu, nsplit, finish && nch == 1, s2);
    if (e != cudaSuccess) break;
  }
  if (nch > 1) {
    cudaEventCreateWithFlags(&evs[nev], cudaEventDisableTiming);
    cudaEventRecord(evs[nev], s2);
    cudaStreamWaitEvent(s, evs[nev], 0);
    ++nev;
    for (int i = 0; i < nev; ++i) cudaEventDestroy(evs[i]);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_block_logmass(const double* sc, const int64_t* bnd, int nb, double* bm,
                                 double* bs, double* lm, cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  k_block_logmass<<<(nb + 127) / 128, 128, 0, s>>>(sc, bnd, nb, bm, bs, lm);
  return cudaGetLastError();
}
cudaError_t launch_fused_attend(const float* sc, const float* v, const int64_t* bnd, int nb, int d,
                                float* out, float* ml, cudaStream_t s) {
  int th = ((d + 31) / 32) * 32;
  if (th < 32) th = 32;
  k_fused_attend<<<1, th, 0, s>>>(sc, v, bnd, nb, d, out, ml);
  return cudaGetLastError();
}

}  // namespace ckv
