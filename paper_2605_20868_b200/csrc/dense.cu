// Rung 3 / Rung 4 terminal fallback on device (fallback.py:230-255,
// harness.py:271-281, 362-372):
//
//   k_resolve      step-wide (per rung4 group of units) Rung 4: a canary or
//                  numeric flag anywhere makes every head of the group dense;
//                  builds the compact list of units that need a dense pass.
//   k_dense        exact softmax attention over the FP16 originals (full
//                  blocks from Tier-2 + the partial block), fp32, split over
//                  the sequence; the four q-heads of a unit share each K/V read.
//                  The last split CTA of a unit to finish merges the splits and
//                  overwrites the fast-path output of every dense head.
#include "step.cuh"

namespace ckv {

constexpr int DN_MAXSPLIT = 256;  // splits per dense unit (merge buffer)
#ifndef DN_SPLITS
#define DN_SPLITS 128
#endif
constexpr int DN_WARPS = 4;

struct DenseArgs {
  ckv_cache c;
  ckv_step st;
  int32_t resolved;  // the step was resolved by the last combine CTA: wait for its epoch
  int32_t n_dsplit;  // splits per dense unit of this launch (set on device from the count)
  int32_t blk_per_split;  // (unused)
  PageView pv;  // HBM scratch slots (Tier-2 in host RAM): resident blocks are read from HBM
};

__device__ __forceinline__ float dninf() { return __int_as_float(0xff800000); }


// every head whose certificate requests Rung 4 flags its unit's group
__global__ void k_group_flags(DenseArgs a) {
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_FLAGS);
  const int nh = st.n_heads;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.c.n_units * nh) return;
  if (st.cert[i].flags & (CKV_F_CANARY | CKV_F_NUMERIC | CKV_F_EXPLORE)) {
    const int g = rung4_group_of(st, i / nh);
    if (g >= 0 && g < st.n_groups) atomicOr(&st.group_flags[g], 1);
  }
}

// a flagged group returns dense for all its heads; list the units needing a dense pass
__global__ void k_resolve(DenseArgs a) {
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_RESOLVE);
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.c.n_units) return;
  const int nh = st.n_heads;
  const int g = rung4_group_of(st, u);
  const bool any4 = (g >= 0 && g < st.n_groups) && st.group_flags[g] != 0;
  int mask = 0;
  for (int h = 0; h < nh; ++h) {
    ckv_cert& ct = st.cert[(size_t)u * nh + h];
    if (any4) ct.returned_kind = 2;
    if (ct.returned_kind != 0) mask |= 1 << h;
  }
  if (mask) {
    const int slot = atomicAdd(&st.dense_list[0], 1);
    st.dense_list[1 + a.c.n_units + slot] = u | (mask << 24);
  }
}

// Merge the splits of one dense item and overwrite the output of its dense
// heads (run by the last split CTA of the item to finish).
__device__ void dense_merge_item(const DenseArgs& a, int item, float* scratch) {
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  const int e = st.dense_list[1 + c.n_units + item];
  const int u = e & 0xffffff, mask = (e >> 24) & 0xf;
  const int nh = st.n_heads;
  const int tid = threadIdx.x;
  const int pl = c.partial_len[u];
  const int ns = a.n_dsplit;
  // (scratch: the CTA's K/V stage buffers, free once its blocks are consumed)
  float (*sm_m)[DN_MAXSPLIT] = reinterpret_cast<float (*)[DN_MAXSPLIT]>(scratch);
  float (*sm_sc)[DN_MAXSPLIT] = reinterpret_cast<float (*)[DN_MAXSPLIT]>(scratch + H * DN_MAXSPLIT);
  __shared__ float red[H][4];
  const float* p0 = st.dense_part + ((size_t)item * st.n_dsplit_cap * H) * 132;
  // per-split maxima -> per-head frame, splits spread over the threads
  for (int i = tid; i < ns * H; i += blockDim.x) sm_m[i % H][i / H] = __ldcg(p0 + (size_t)i * 132);
  __syncthreads();
  if (tid < H * 32) {
    const int h = tid >> 5, l = tid & 31;
    float m = dninf();
    for (int s = l; s < ns; s += 32) m = fmaxf(m, sm_m[h][s]);
    m = warp_max(m);
    if (l == 0) red[h][0] = m;
  }
  __syncthreads();
  for (int i = tid; i < ns * H; i += blockDim.x) {
    const int h = i % H, s = i / H;
    const HeadState& hs =
        *reinterpret_cast<const HeadState*>(st.head_state + ((size_t)u * nh + (h < nh ? h : 0)) * CKV_HEAD_FLOATS);
    const float M = (pl > 0) ? fmaxf(red[h][0], hs.mp) : red[h][0];
    sm_sc[h][s] = (sm_m[h][s] == dninf()) ? 0.f : expf(sm_m[h][s] - M);
  }
  __syncthreads();
  for (int h = 0; h < nh; ++h) {
    if (!((mask >> h) & 1)) continue;
    const HeadState& hs =
        *reinterpret_cast<const HeadState*>(st.head_state + ((size_t)u * nh + h) * CKV_HEAD_FLOATS);
    const float M = (pl > 0) ? fmaxf(red[h][0], hs.mp) : red[h][0];
    float L = 0.f, O = 0.f;
#pragma unroll 8
    for (int s = 0; s < ns; ++s) {
      const float* p = p0 + (s * H + h) * 132;
      const float sc = sm_sc[h][s];
      L += __ldcg(p + 1) * sc;
      O += __ldcg(p + 4 + tid) * sc;
    }
    if (pl > 0) {
      const float sc = expf(hs.mp - M);
      L += hs.lp * sc;
      O += hs.np_[tid] * sc;
    }
    st.out[((size_t)u * nh + h) * D + tid] = O / L;
  }
}

// Called by every split CTA of a dense item once its state is written: the
// last one merges (device-scope counter, reset for the next step).
__device__ __forceinline__ void dense_split_done(const DenseArgs& a, int item, float* scratch) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    int* done = a.st.dense_list + 1 + item;
    const int prev = atomicAdd(done, 1);
    last = (prev == a.n_dsplit - 1);
    if (last) *done = 0;
    __threadfence();
  }
  __syncthreads();
  if (last) dense_merge_item(a, item, scratch);
}

constexpr int DN_STAGES = 2;
struct DenseSmem {
  uint8_t stg[DN_WARPS][DN_STAGES][2][B * D * 2];  // per warp: ring of (key tile, value tile)
  uint64_t bar[DN_WARPS][DN_STAGES];
  float qh[H * D];
  float w[DN_WARPS][H][B];  // softmax weights x 2^14, tokens permuted (B-fragment order)
};

// Exact attention over the full blocks of one split of a flagged unit; all
// four q-heads share every K/V read.  Scores come from orig_block (FP16 keys
// x hi/lo-split q' on the tensor cores, fp32 accumulate); P.V runs on the
// tensor cores too: A = the fragment-ordered FP16 values (exact), B = the
// weights as an fp16 hi/lo pair (column 2h + part), fp32 accumulation.  The
// partial block is added in the merge from the state k_select computed.
__global__ void __launch_bounds__(DN_WARPS * 32) k_dense(DenseArgs a_in) {
  extern __shared__ __align__(128) uint8_t dn_smem[];
  DenseSmem& S = *reinterpret_cast<DenseSmem*>(dn_smem);
  // a warp's split partials (O, then m / l) go to its own stage buffers once it
  // has consumed its blocks; the merge scratch is the whole stage area
  auto ow = [&](int w) { return reinterpret_cast<float (*)[D]>(S.stg[w][0][0]); };
  auto mw = [&](int w) { return reinterpret_cast<float (*)[2]>(S.stg[w][0][0] + H * D * 4); };
  float* mscratch = reinterpret_cast<float*>(S.stg);
  DenseArgs a = a_in;
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_DENSE);
  if (a.resolved) flow_wait(flow_step(st.flow, c.n_units, FLOW_RESOLVED), st.epoch);
  // persistent over (item, split) tasks; the split count adapts to the number of
  // dense units so that a few of them still spread over every SM
  const int count = st.dense_list[0];
  if (count == 0) return;
  if (threadIdx.x == 0) {
    for (int w = 0; w < DN_WARPS; ++w)
      for (int s = 0; s < DN_STAGES; ++s) mbar_init(&S.bar[w][s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int kb = 0;  // blocks this warp has pushed through its ring (stage / parity across tasks)
  // ~384 tasks in all: long splits (little merge work) when many units are dense,
  // up to DN_SPLITS per unit when only a few are (latency-bound otherwise)
  if (st.dense_splits > 0) {
    a.n_dsplit = min(st.n_dsplit_cap, st.dense_splits);
  } else if (count <= (int)gridDim.x) {  // one wave of tasks
    a.n_dsplit = min(st.n_dsplit_cap, min(DN_SPLITS, (int)gridDim.x / count));
  } else {  // the split count with the fewest waves per unit of work (ties -> fewer splits)
    int best = 1;
    long long bw = (count + gridDim.x - 1) / gridDim.x;  // waves x best, compared as fractions
    for (int n = 2; n <= 16 && n <= st.n_dsplit_cap; ++n) {
      const long long w = ((long long)count * n + gridDim.x - 1) / gridDim.x;
      if (w * best < bw * n) {
        best = n;
        bw = w;
      }
    }
    a.n_dsplit = best;
  }
  for (int task = blockIdx.x; task < count * a.n_dsplit; task += gridDim.x) {
  const int item = task / a.n_dsplit, sp = task % a.n_dsplit;
  const int e = st.dense_list[1 + c.n_units + item];
  const int u = e & 0xffffff;
  const int nh = st.n_heads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = c.n_blocks[u];
  const int bps = max(1, (nb + a.n_dsplit - 1) / a.n_dsplit);
  const int b0 = sp * bps, b1 = min(nb, b0 + bps);
  float* outp = st.dense_part + (((size_t)item * st.n_dsplit_cap + sp) * H) * 132;
  fence_proxy_async();  // this thread's generic smem writes before the next bulk copies
  __syncthreads();  // the previous task is done with S (stages, partials, merge)
  if (b0 >= b1) {
    for (int i = tid; i < H * 132; i += blockDim.x) outp[i] = (i % 132 == 0) ? dninf() : 0.f;
    dense_split_done(a, item, mscratch);
    continue;
  }
  const size_t ubk = (size_t)u * c.max_blocks;
  // a block already paged into an HBM slot this or an earlier step (its bytes are
  // the Tier-2 bytes) is read from the slot instead of over PCIe from host Tier-2
  const PageView& pv = a.pv;
  const int32_t* kslot = pv.kslots ? pv.kslot_of + (size_t)u * pv.kstride : nullptr;
  const int32_t* vslot = pv.vslots ? pv.vslot_of + (size_t)u * pv.vstride : nullptr;
  // this warp's blocks b0 + warp + 4 i stream through a DN_STAGES ring of bulk copies
  const int nmine = (b1 - b0 > warp) ? (b1 - b0 - warp + DN_WARPS - 1) / DN_WARPS : 0;
  auto issue = [&](int i) {  // lane 0
    const int b = b0 + warp + DN_WARPS * i;
    const int s2 = (kb + i) % DN_STAGES;
    const int ksl = kslot ? kslot[b] : -1, vsl = vslot ? vslot[b] : -1;
    const uint16_t* ks = (ksl >= 0) ? pv.kslots + ((size_t)u * pv.kcap + ksl) * B * D : c.tier2_k + (ubk + b) * B * D;
    const uint16_t* vs = (vsl >= 0) ? pv.vslots + ((size_t)u * pv.vcap + vsl) * B * D : c.tier2_v + (ubk + b) * B * D;
    mbar_expect_tx(&S.bar[warp][s2], 2 * B * D * 2);
    bulk_g2s(S.stg[warp][s2][0], ks, B * D * 2, &S.bar[warp][s2]);
    bulk_g2s(S.stg[warp][s2][1], vs, B * D * 2, &S.bar[warp][s2]);
  };
  if (lane == 0)  // the ring's first copies, before the query setup they do not need
    for (int i = 0; i < DN_STAGES && i < nmine; ++i) issue(i);
  for (int i = tid; i < H * D; i += blockDim.x) {
    const int h = i / D;
    S.qh[i] = (h < nh) ? (float)(st.q[((size_t)u * nh + h) * D + (i % D)] * 0.08838834764831845) : 0.f;
  }
  // Tier-2 must hold every block we read (cache.py:138-142)
  for (int b = b0 + tid; b < b1; b += blockDim.x)
    if (!c.tier2_valid[(size_t)u * c.max_blocks + b]) atomicOr(&c.status[CKV_ST_TIER2], 1);
  __syncthreads();
  QFrag16 f16;
  load_qfrag16(f16, S.qh, lane);
  const int h = lane & 3, t0 = lane >> 2;
  const int pi0 = 4 * (t0 >> 1) + (t0 & 1), pi1 = pi0 + 2;
  const int hb = lane >> 3;
  const bool lo_lane = (lane >> 2) & 1;
  float m_h = dninf(), l_h = 0.f;
  float acc[NG][4];
#pragma unroll
  for (int g = 0; g < NG; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
  for (int i = 0; i < nmine; ++i) {
    const int s2 = (kb + i) % DN_STAGES;
    mbar_wait(&S.bar[warp][s2], (uint32_t)((kb + i) / DN_STAGES) & 1u);
    const uint4* kf = reinterpret_cast<const uint4*>(S.stg[warp][s2][0]);
    const uint4* vf = reinterpret_cast<const uint4*>(S.stg[warp][s2][1]);
    uint4 av[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) av[g] = vf[g * 32 + lane];
    const float2 s = orig_block(f16, kf, lane);
    __syncwarp();  // every lane has read the stage: refill it
    if (lane == 0 && i + DN_STAGES < nmine) issue(i + DN_STAGES);
    float bmx = fmaxf(s.x, s.y);
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 4));
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 8));
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 16));
    const float m_new = fmaxf(m_h, bmx);
    const float alpha = (m_h == dninf()) ? 0.f : expf(m_h - m_new);
    m_h = m_new;
    const float w0 = expf(s.x - m_h), w1 = expf(s.y - m_h);
    l_h = l_h * alpha + w0 + w1;
    S.w[warp][h][pi0] = w0 * 16384.f;
    S.w[warp][h][pi1] = w1 * 16384.f;
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        acc[g][0] *= alpha; acc[g][1] *= alpha; acc[g][2] *= alpha; acc[g][3] *= alpha;
      }
    }
    __syncwarp();
    uint32_t h01, l01, h23, l23;
    const float4 p4 = *reinterpret_cast<const float4*>(&S.w[warp][hb][4 * (lane & 3)]);
    split_h2(p4.x, p4.y, h01, l01);
    split_h2(p4.z, p4.w, h23, l23);
    const uint32_t bb0 = lo_lane ? l01 : h01, bb1 = lo_lane ? l23 : h23;
#pragma unroll
    for (int g = 0; g < NG; ++g) mma_f16r(acc[g], av[g].x, av[g].y, av[g].z, av[g].w, bb0, bb1);
    __syncwarp();
  }
  kb += nmine;
  l_h += __shfl_xor_sync(0xffffffffu, l_h, 4);
  l_h += __shfl_xor_sync(0xffffffffu, l_h, 8);
  l_h += __shfl_xor_sync(0xffffffffu, l_h, 16);
  if (lane < H) {
    mw(warp)[lane][0] = m_h;
    mw(warp)[lane][1] = l_h;
  }
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    ow(warp)[h][16 * g + t0] = (acc[g][0] + acc[g][1]) * (1.f / 16384.f);
    ow(warp)[h][16 * g + t0 + 8] = (acc[g][2] + acc[g][3]) * (1.f / 16384.f);
  }
  __syncthreads();
  for (int hh = 0; hh < H; ++hh) {
    float M = dninf();
    for (int w = 0; w < DN_WARPS; ++w) M = fmaxf(M, mw(w)[hh][0]);
    float L = 0.f, O = 0.f;
    if (M != dninf()) {
      for (int w = 0; w < DN_WARPS; ++w) {
        if (mw(w)[hh][0] == dninf()) continue;
        const float sc = expf(mw(w)[hh][0] - M);
        L += mw(w)[hh][1] * sc;
        O += ow(w)[hh][tid] * sc;
      }
    }
    if (tid == 0) {
      outp[hh * 132 + 0] = M;
      outp[hh * 132 + 1] = L;
    }
    outp[hh * 132 + 4 + tid] = O;
  }
  dense_split_done(a, item, mscratch);
  }  // task loop
}


// The step's bound report straight into the caller's pinned host buffer
// (ckv_step.host_report): the last kernel of the step, launched behind the dense
// pass as a programmatic dependent; griddepcontrol.wait orders it after every
// earlier kernel of the step and makes their writes visible.
struct PublishArgs {
  const uint32_t* cert;
  const int32_t* status;
  const int32_t* ps;
  const int32_t* en;
  uint8_t* dst;
  int32_t n_cert, n_ps, n_en;  // 4-byte words
  int64_t off_status, off_ps, off_en;
};

__global__ void __launch_bounds__(256) k_publish(PublishArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t* d = reinterpret_cast<uint32_t*>(a.dst);
  const int n = a.n_cert + 8 + a.n_ps + a.n_en;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < a.n_cert) {
      d[i] = __ldcg(a.cert + i);
    } else if (i < a.n_cert + 8) {
      const int j = i - a.n_cert;
      reinterpret_cast<int32_t*>(a.dst + a.off_status)[j] = __ldcg(a.status + j);
    } else if (i < a.n_cert + 8 + a.n_ps) {
      const int j = i - a.n_cert - 8;
      reinterpret_cast<int32_t*>(a.dst + a.off_ps)[j] = __ldcg(a.ps + j);
    } else {
      const int j = i - a.n_cert - 8 - a.n_ps;
      reinterpret_cast<int32_t*>(a.dst + a.off_en)[j] = __ldcg(a.en + j);
    }
  }
}

cudaError_t launch_publish(const ckv_cache* c, const ckv_step* st, cudaStream_t s) {
  int64_t lay[4];
  report_layout(c->n_units, st->n_heads, lay);
  PublishArgs a;
  a.cert = reinterpret_cast<const uint32_t*>(st->cert);
  a.status = c->status;
  a.ps = st->page_stats;
  a.en = st->explore_n;
  a.dst = static_cast<uint8_t*>(st->host_report);
  a.n_cert = (int32_t)((int64_t)c->n_units * st->n_heads * (int64_t)sizeof(ckv_cert) / 4);
  a.n_ps = st->page_stats ? c->n_units * 4 : 0;
  a.n_en = st->explore_n ? c->n_units * st->n_heads : 0;
  a.off_status = lay[1];
  a.off_ps = lay[2];
  a.off_en = lay[3];
  const int n = a.n_cert + 8 + a.n_ps + a.n_en;
  const int grid = (n + 255) / 256 < dev_state().sms ? (n + 255) / 256 : dev_state().sms;
  cudaError_t e = launch_k(true, k_publish, dim3(grid), dim3(256), 0, s, a);
  g_launches += 1;
  return e;
}

cudaError_t launch_group_flags(const ckv_cache* c, const ckv_step* st, cudaStream_t s) {
  DenseArgs a{*c, *st, 0, 0, 0, PageView{}};
  cudaMemsetAsync(st->group_flags, 0, sizeof(int32_t) * st->n_groups, s);
  const int n = c->n_units * st->n_heads;
  k_group_flags<<<(n + 255) / 256, 256, 0, s>>>(a);
  g_launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_dense(const ckv_cache* c, const ckv_step* st, const ckv_scratch* sc,
                         int host_max_tokens, bool resolved, cudaStream_t s) {
  (void)host_max_tokens;
  DenseArgs a{*c, *st, resolved ? 1 : 0, 1, 0, PageView{}};
  if (a.st.dense_splits <= 0 && knobs().dn_splits > 0) a.st.dense_splits = knobs().dn_splits;
  if (sc && (sc->key_slots || sc->value_slots)) {
    a.pv.kslots = sc->key_capacity > 0 ? sc->key_slots : nullptr;
    a.pv.vslots = sc->value_capacity > 0 ? sc->value_slots : nullptr;
    a.pv.kcap = sc->key_capacity;
    a.pv.vcap = sc->value_capacity;
    a.pv.kstride = lru_words(c->max_blocks, sc->key_capacity);
    a.pv.vstride = lru_words(c->max_blocks, sc->value_capacity);
    a.pv.kslot_of = sc->key_lru + lru_slot_offset(c->max_blocks, sc->key_capacity);
    a.pv.vslot_of = sc->value_lru + lru_slot_offset(c->max_blocks, sc->value_capacity);
  }
  set_max_dyn_smem(k_dense, (int)sizeof(DenseSmem));
  DevState& ds = dev_state();
  if (!ds.dense_slots) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dense, DN_WARPS * 32, sizeof(DenseSmem));
    ds.dense_slots = max(1, ds.sms * max(1, per));
  }
  const int slots = ds.dense_slots;
  if (resolved) {  // right behind the combine that resolved the step (PDL)
    cudaError_t e = launch_k(true, k_dense, dim3(slots), dim3(DN_WARPS * 32), sizeof(DenseSmem), s, a);
    g_launches += 1;
    return e;
  }
  cudaMemsetAsync(st->dense_list, 0, sizeof(int32_t) * (1 + c->n_units), s);  // count + done counters
  k_resolve<<<(c->n_units + 255) / 256, 256, 0, s>>>(a);
  k_dense<<<slots, DN_WARPS * 32, sizeof(DenseSmem), s>>>(a);
  g_launches += 2;
  // the dataflow path (resolved) expects the step-wide requests cleared
  cudaMemsetAsync(st->group_flags, 0, sizeof(int32_t) * st->n_groups, s);
  return cudaGetLastError();
}

}  // namespace ckv
