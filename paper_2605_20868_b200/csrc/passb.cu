// Pass B and combine.
//
//   k_union    per unit: the union over its q-heads of promoted (F_h) and
//              value-promoted (V_h) blocks, ascending, with 4-bit head masks.
//   k_pass_b   per unit over that union only: the block's quantized scores
//              for all 4 heads (phase1_block, bit-identical to pass A), the
//              original-key scores on the tensor cores (orig_block over the
//              fragment-ordered FP16 Tier-2 keys), and per head the additive
//              correction that turns pass A's speculative attend into the
//              mask-gated Phase 2 of attention.py:251-282: for b in F_h
//              add e^{s-m} v_new - e^{s'-m} v_hat, for b in V_h \ F_h add
//              e^{s'-m} (v - v_hat).  Also the phase-2 log-mass of every
//              promoted block (attention.py:283-296), the canary gap
//              (fallback.py:190-199) and the F part of E_val.
//   k_combine  per (unit, head): merge, output, ranking / boundary / canary
//              monitors (harness.py:231-260), E_key / E_val (certifier.py:135-212).
#include "step.cuh"

namespace ckv {

constexpr int UN_THREADS = 256;

__global__ void __launch_bounds__(UN_THREADS) k_union(StepArgs a) {
  extern __shared__ __align__(16) uint32_t ub[];
  __shared__ int ws[32];
  build_union(a.c, a.st, a.u0 + blockIdx.x, ub, ws);
}

// -----------------------------------------------------------------------------
constexpr int PB_WARPS = 4;

struct PassBSmem {
  uint8_t rec[PB_WARPS][2][REC];
  uint8_t kt[PB_WARPS][2][B * D * 2];  // FP16 Tier-2 key tile (fragment order) of promoted blocks
  uint64_t bar[PB_WARPS][2];
  float sst[PB_WARPS][2][H * B];  // stashed phase-1 scores of the item (pass A), [head][token]
  float qh[H * D];
  float cq[PB_WARPS][H][B];  // coefficient of v_hat per (head, token), tokens permuted
  float ca[PB_WARPS][H][B];  // coefficient of the original v
};

// One chunk (IPC consecutive items of unit u's union list, 4 warps interleaved).
// Page one missed FP16 tile (4 KB) from Tier-2 into its HBM slot, 16 B per lane per
// group; the caller's lane re-reads exactly the words it wrote.  Out of line: it
// runs for the few missed items only and keeps pass B's hot loop free of spills.
__device__ __noinline__ void page_in_tile(const uint16_t* slot, const uint16_t* tier2, int lane) {
  const uint4* src = reinterpret_cast<const uint4*>(tier2);
  uint4* dst = reinterpret_cast<uint4*>(const_cast<uint16_t*>(slot));
  uint4 t[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) t[g] = src[g * 32 + lane];
#pragma unroll
  for (int g = 0; g < NG; ++g) dst[g * 32 + lane] = t[g];
}

// kb = items this warp has pushed through its 2-stage ring so far (stage and
// mbarrier parity continue across the chunks a persistent CTA processes).
// SLOTS: the scratch has HBM slots (Tier-2 in host RAM); without them no slot code is compiled in.
template <bool SLOTS>
__device__ __forceinline__ void pass_b_chunk(const StepArgs& a, PassBSmem& S, const int u,
                                             const int ck, const int C, int& kb) {
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  const int IPC = st.items_per_chunk;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nh = st.n_heads;
  const int nwork = st.n_work[u];
  float* cs = st.chunk_state + ((size_t)u * C + ck) * H * CKV_CHUNK_FLOATS;
  // balanced partition (a.nchunk CTAs per unit, one chunk each) or IPC-sized chunks
  const bool bal = a.nchunk > 0;
  const int lo = bal ? (int)((long long)ck * nwork / a.nchunk) : ck * IPC;
  const int hi = bal ? (int)((long long)(ck + 1) * nwork / a.nchunk) : min(nwork, lo + IPC);
  if (lo >= hi) {
    if (tid < H) cs[tid * CKV_CHUNK_FLOATS] = ninf();
    return;
  }

  const int h = lane & 3;  // the head this lane's scores belong to
  const int hq = (h < nh) ? h : 0;
  const HeadState& hsq =
      *reinterpret_cast<const HeadState*>(st.head_state + ((size_t)u * nh + hq) * CKV_HEAD_FLOATS);
  const double lse = hsq.lse;
  float m_h = hsq.mA;
  if (m_h == ninf()) m_h = -1e30f;
  float dden = 0.f, canary = 0.f;
  double eF = 0.0, sF = 0.0;
  float acc[NG][4], accz[4];
#pragma unroll
  for (int g = 0; g < NG; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
  accz[0] = accz[1] = accz[2] = accz[3] = 0.f;
  const int Sx = value_exp(c.v_max[u]);
  const float p2S = pow2f(Sx);

  const size_t ubk = (size_t)u * c.max_blocks;
  const int32_t* work = st.work + (size_t)u * st.wcap;
  const float* eta = c.eta + ubk;
  float* lm2 = st.lm2 + ((size_t)u * nh + hq) * c.max_blocks;
  const int t0 = lane >> 2;
  const int pi0 = 4 * (t0 >> 1) + (t0 & 1), pi1 = pi0 + 2;
  const int hb = lane >> 3;
  const bool lo_lane = (lane >> 2) & 1;

  // this warp's item sequence: chunks ck, ck+C, ...; items base+warp, +4, ...
  auto item_at = [&](int k) -> int {  // k-th item of this warp, or -1
    if (bal) {
      const int idx = lo + warp + k * PB_WARPS;
      return (idx < hi) ? idx : -1;
    }
    const int per_chunk = (IPC + PB_WARPS - 1 - warp) / PB_WARPS;
    const int chunk = k / per_chunk, within = k % per_chunk;
    const int idx = (ck + chunk * C) * IPC + warp + within * PB_WARPS;
    const int cend = min(nwork, (ck + chunk * C) * IPC + IPC);
    return (idx < cend) ? idx : -1;
  };
  const uint8_t* t1base = c.tier1 + ubk * REC;
  // stage = the Tier-1 record (+ the FP16 key tile when some head promotes the block)
  const PageView& pv = a.pv;
  const int32_t* kslot = (SLOTS && pv.kslots) ? pv.kslot_of + (size_t)u * pv.kstride : nullptr;
  const int32_t* vslot = (SLOTS && pv.vslots) ? pv.vslot_of + (size_t)u * pv.vstride : nullptr;
  // Per-item metadata (work entry, slot, key-scale max, eta, Tier-2 valid,
  // stash epoch) is gathered lane-parallel: lane l holds item j = 32 w + l of
  // the warp's sequence in set w & 1; the set of window w + 2 is refilled at
  // the start of window w + 1 (work entries) and 8 items later (the dependent
  // words), so no load latency sits on the item loop.  Items are fetched from
  // their lane with shuffles two iterations before their copies are issued.
  struct Meta {
    int e, sl, valid, st, vsl;
    float smax, eta;
  };
  const float* stash_u = st.stash ? st.stash + (size_t)u * c.max_blocks * 64 : nullptr;
  int le[2], lsl[2], lval[2], lsep[2], lvs[2];
  float lsm[2], let_[2];
  // fused LRU accounting (scratch holding every block): a block's first request
  // ever is a miss, every other a hit -- decided lane-parallel for a window of 32
  // items when its work entries are loaded, off the item loop
  int lk_h = 0, lk_m = 0, lv_h = 0, lv_m = 0, req_k = 0, req_v = 0;
  auto load_e = [&](int s, int kbase) {
    const int it = item_at(kbase + lane);
    const int e2 = (it >= 0) ? work[it] : -1;
    if (s) le[1] = e2; else le[0] = e2;
    if (pv.fused && e2 != -1) {
      const int b2 = e2 & 0xffffff;
      const int nk = __popc(((uint32_t)e2 >> 24) & 0xfu), nv = __popc(((uint32_t)e2 >> 28) & 0xfu);
      if (nk) {
        const int miss = atomicExch(pv.klru + (size_t)u * pv.kstride + 4 + b2, 1) == 0;
        lk_m += miss;
        lk_h += nk - miss;
        req_k += nk;
      }
      if (nv) {
        const int miss = atomicExch(pv.vlru + (size_t)u * pv.vstride + 4 + b2, 1) == 0;
        lv_m += miss;
        lv_h += nv - miss;
        req_v += nv;
      }
    }
  };
  auto load_words = [&](int s) {
    const int e2 = s ? le[1] : le[0];
    const bool ok = e2 != -1;
    const int b2 = e2 & 0xffffff;
    int sl = (ok && kslot && (((uint32_t)e2 >> 24) & 0xfu)) ? kslot[b2] : -1;
    // missed into its slot this step: read Tier-2, fill the slot (bit 30 of sl)
    if (sl >= 0 && kslot[c.max_blocks + b2] == st.epoch) sl |= 0x40000000;
    const float sm = ok ? c.kscale_max[ubk + b2] : 1.f;
    const float et = ok ? eta[b2] : 0.f;
    const int va = ok ? c.tier2_valid[ubk + b2] : 1;
    const int se = (ok && stash_u) ? st.stash_epoch[ubk + b2] : 0;
    // value slot (bit 30: missed this step), SLOTS instance only
    int vs = -1;
    if (SLOTS && vslot && ok && ((uint32_t)e2 >> 28)) {
      vs = vslot[b2];
      if (vs >= 0 && vslot[c.max_blocks + b2] == st.epoch) vs |= 0x40000000;
    }
    if (s) { lsl[1] = sl; lsm[1] = sm; let_[1] = et; lval[1] = va; lsep[1] = se; lvs[1] = vs; }
    else   { lsl[0] = sl; lsm[0] = sm; let_[0] = et; lval[0] = va; lsep[0] = se; lvs[0] = vs; }
  };
  auto fetch = [&](int j) -> Meta {  // warp-uniform j
    const int s = (j >> 5) & 1, src = j & 31;
    Meta m;
    m.e = __shfl_sync(0xffffffffu, s ? le[1] : le[0], src);
    m.sl = __shfl_sync(0xffffffffu, s ? lsl[1] : lsl[0], src);
    m.smax = __shfl_sync(0xffffffffu, s ? lsm[1] : lsm[0], src);
    m.eta = __shfl_sync(0xffffffffu, s ? let_[1] : let_[0], src);
    m.valid = __shfl_sync(0xffffffffu, s ? lval[1] : lval[0], src);
    m.vsl = SLOTS ? __shfl_sync(0xffffffffu, s ? lvs[1] : lvs[0], src) : -1;
    const int se = __shfl_sync(0xffffffffu, s ? lsep[1] : lsep[0], src);
    // usable when this step's pass A stashed every head the item is promoted for
    const uint32_t need = (((uint32_t)m.e >> 24) | ((uint32_t)m.e >> 28)) & 0xfu;
    m.st = stash_u && m.e != -1 && ((se >> 4) == st.epoch) && ((need & ~(uint32_t)se) == 0u);
    return m;
  };
  auto issue = [&](const Meta& m, int stg) {
    const int b2 = m.e & 0xffffff;
    const bool keys = ((uint32_t)m.e >> 24) & 0xfu;
    if (m.st) {  // scores stashed by pass A: only the value part of the record (+ the stash)
      mbar_expect_tx(&S.bar[warp][stg], (REC - OFF_VCODES) + H * B * 4 + (keys ? B * D * 2 : 0));
      bulk_g2s(S.rec[warp][stg] + OFF_VCODES, t1base + (size_t)b2 * REC + OFF_VCODES, REC - OFF_VCODES,
               &S.bar[warp][stg]);
      bulk_g2s(S.sst[warp][stg], stash_u + (size_t)b2 * 64, H * B * 4, &S.bar[warp][stg]);
    } else {
      mbar_expect_tx(&S.bar[warp][stg], REC + (keys ? B * D * 2 : 0));
      bulk_g2s(S.rec[warp][stg], t1base + (size_t)b2 * REC, REC, &S.bar[warp][stg]);
    }
    // the value tile of a value-promoted item is read with plain loads in its value
    // branch (from its HBM slot, or from Tier-2 -- host RAM when missed this step):
    // start pulling it into L2 an item ahead, off the loop's latency
    if ((uint32_t)m.e >> 28) {
      const bool in_slot = SLOTS && m.vsl >= 0 && !(m.vsl & 0x40000000);
      prefetch_l2(in_slot ? pv.vslots + ((size_t)u * pv.vcap + m.vsl) * B * D : c.tier2_v + (ubk + b2) * B * D,
                  B * D * 2);
    }
    if (keys) {
      const uint16_t* src = (m.sl >= 0 && !(m.sl & 0x40000000))
                                ? pv.kslots + ((size_t)u * pv.kcap + m.sl) * B * D
                                : c.tier2_k + (ubk + b2) * B * D;
      bulk_g2s(S.kt[warp][stg], src, B * D * 2, &S.bar[warp][stg]);
    }
  };
  // the item metadata first: its two dependent load rounds overlap the query setup
  load_e(0, 0);
  load_e(1, 32);
  load_words(0);
  load_words(1);
  __syncthreads();  // the previous chunk's reduction is done with S
  for (int i = tid; i < H * D; i += blockDim.x) {
    const int hh = i / D;
    S.qh[i] = (hh < nh) ? (float)(st.q[((size_t)u * nh + hh) * D + (i % D)] * 0.08838834764831845)
                        : 0.f;
  }
  __syncthreads();
  QFrag f;
  load_qfrag(f, S.qh, lane);
  QFrag16 f16;
  load_qfrag16(f16, S.qh, lane);
  int cur = item_at(0);
  int i1 = item_at(1);
  Meta mc = fetch(0);
  Meta mn = fetch(1);
  if (lane == 0 && cur >= 0) {
    fence_proxy_async();
    issue(mc, kb & 1);
  }
  // the item two ahead, advanced incrementally (no division in the loop)
  const int per_chunk = (IPC + PB_WARPS - 1 - warp) / PB_WARPS;
  int nx_chunk = (per_chunk > 2) ? 0 : 2 / per_chunk, nx_within = (per_chunk > 2) ? 2 : 2 % per_chunk;
  int k = 0;
  for (; cur >= 0; ++k) {
    const int stg = (kb + k) & 1;
    const int nxt = i1;
    if ((k & 31) == 0 && k >= 32) load_e(((k >> 5) + 1) & 1, k + 32);
    if ((k & 31) == 8 && k >= 32) load_words(((k >> 5) + 1) & 1);
    if (lane == 0 && nxt >= 0) {
      if (SLOTS && pv.kslots) bulk_wait_read();  // a slot fill (shared -> global) may still read the stage
      fence_proxy_async();
      issue(mn, stg ^ 1);
    }
    const int e = mc.e;
    const int b = e & 0xffffff;
    const uint32_t fm = ((uint32_t)e >> 24) & 0xfu, vm = ((uint32_t)e >> 28) & 0xfu;
    const bool inF = (fm >> h) & 1u, inV = (vm >> h) & 1u;
    if ((fm | vm) && lane == 0 && !mc.valid) atomicOr(&c.status[CKV_ST_TIER2], 1);
    const float smax = mc.smax;
    const float eta_b = mc.eta;
    mbar_wait(&S.bar[warp][stg], (uint32_t)((kb + k) >> 1) & 1u);
    const uint8_t* rec = S.rec[warp][stg];
    if (SLOTS && fm && mc.sl >= 0 && (mc.sl & 0x40000000) && lane == 0) {  // page-in of a missed key tile
      bulk_s2g(const_cast<uint16_t*>(pv.kslots) + ((size_t)u * pv.kcap + (mc.sl & 0x3fffffff)) * B * D,
               S.kt[warp][stg], B * D * 2);
    }

    BlockScores r;
    if (mc.st) {  // bit-identical to phase1_block in pass A (that is where they come from)
      // heads the item is not promoted for have no stash entry and take no part
      const bool need_h = ((fm | vm) >> h) & 1u;
      r.s0 = need_h ? S.sst[warp][stg][h * B + t0] : ninf();
      r.s1 = need_h ? S.sst[warp][stg][h * B + t0 + 8] : ninf();
      r.delta = 0.f;
    } else {
      r = phase1_block(f, rec, smax, lane);
    }
    float sn0 = r.s0, sn1 = r.s1;
    if (fm) {
      const float2 so = orig_block(f16, reinterpret_cast<const uint4*>(S.kt[warp][stg]), lane);
      if (inF) {
        sn0 = so.x;
        sn1 = so.y;
      }
    }
    // per-head frame, weights, phase-2 block log-mass and canary
    float bmx = fmaxf(sn0, sn1);
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 4));
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 8));
    bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, 16));
    const float m_new = fmaxf(m_h, bmx);
    const float alpha = fast_exp(m_h - m_new);
    m_h = m_new;
    const float wn0 = fast_exp(sn0 - m_h), wn1 = fast_exp(sn1 - m_h);
    const float wq0 = fast_exp(r.s0 - m_h), wq1 = fast_exp(r.s1 - m_h);
    dden = dden * alpha + (inF ? (wn0 - wq0) + (wn1 - wq1) : 0.f);
    if (fm) {
      float es = fast_exp(sn0 - bmx) + fast_exp(sn1 - bmx);
      float gap = fmaxf(fabsf(sn0 - r.s0), fabsf(sn1 - r.s1));
      es += __shfl_xor_sync(0xffffffffu, es, 4);
      es += __shfl_xor_sync(0xffffffffu, es, 8);
      es += __shfl_xor_sync(0xffffffffu, es, 16);
      gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 4));
      gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 8));
      gap = fmaxf(gap, __shfl_xor_sync(0xffffffffu, gap, 16));
      if (inF) {
        const float lb = bmx + __logf(es);
        canary = fmaxf(canary, gap);
        if (lane < H && h < nh) {
          lm2[b] = lb;
          const double rb = (double)__expf(lb - (float)lse);  // phase-2 block mass (fp32 exp: 1e-7 rel.)
          sF += rb;
          if (!inV) eF += rb * (double)eta_b;
        }
      }
    }
    // branch-free correction coefficients: acc_h += ca * v_orig + cq * v_hat
    //   F & V: ca = wn, cq = -wq   F only: ca = 0, cq = wn - wq
    //   V only: ca = wq, cq = -wq  neither: ca = cq = 0
    S.ca[warp][h][pi0] = (inV ? (inF ? wn0 : wq0) : 0.f) * p2S;
    S.ca[warp][h][pi1] = (inV ? (inF ? wn1 : wq1) : 0.f) * p2S;
    S.cq[warp][h][pi0] = (inV ? -wq0 : (inF ? wn0 - wq0 : 0.f)) * p2S;
    S.cq[warp][h][pi1] = (inV ? -wq1 : (inF ? wn1 - wq1 : 0.f)) * p2S;
    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        acc[g][0] *= alpha; acc[g][1] *= alpha; acc[g][2] *= alpha; acc[g][3] *= alpha;
      }
      accz[0] *= alpha; accz[1] *= alpha; accz[2] *= alpha; accz[3] *= alpha;
    }
    __syncwarp();
    {  // v_hat part, as pass A's speculative P.V: the INT4 codes as fp16 subnormals
       // (A operand without conversion), B = cq' * scale (hi/lo); acc in units 2^-24
      PVFrag F;
      pv_frag(F, *reinterpret_cast<const float4*>(&S.cq[warp][hb][4 * (lane & 3)]), lo_lane);
      pv_block_sub(acc, accz, F, rec, lane);
    }
    if (vm) {  // warp-uniform: some head of this block is value-promoted: B = ca' (hi/lo)
      uint32_t h01, l01, h23, l23;
      const float4 p4 = *reinterpret_cast<const float4*>(&S.ca[warp][hb][4 * (lane & 3)]);
      split_h2(p4.x, p4.y, h01, l01);
      split_h2(p4.z, p4.w, h23, l23);
      const uint32_t b0 = lo_lane ? l01 : h01, b1 = lo_lane ? l23 : h23;
      int vsl = SLOTS ? mc.vsl : -1;
      if (vsl >= 0 && (vsl & 0x40000000)) {  // missed into its slot this step
        vsl &= 0x3fffffff;
        page_in_tile(pv.vslots + ((size_t)u * pv.vcap + vsl) * B * D, c.tier2_v + (ubk + b) * B * D, lane);
      }
      const uint4* vf = reinterpret_cast<const uint4*>(
          (vsl >= 0) ? pv.vslots + ((size_t)u * pv.vcap + vsl) * B * D : c.tier2_v + (ubk + b) * B * D);
      uint4 av[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) av[g] = vf[g * 32 + lane];
#pragma unroll
      for (int g = 0; g < NG; ++g) {  // original values in units 1, acc in 2^-24: exact rescale
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        mma_f16r(t, av[g].x, av[g].y, av[g].z, av[g].w, b0, b1);
        acc[g][0] = fmaf(t[0], 5.9604644775390625e-8f, acc[g][0]);
        acc[g][1] = fmaf(t[1], 5.9604644775390625e-8f, acc[g][1]);
        acc[g][2] = fmaf(t[2], 5.9604644775390625e-8f, acc[g][2]);
        acc[g][3] = fmaf(t[3], 5.9604644775390625e-8f, acc[g][3]);
      }
    }
    __syncwarp();
    cur = nxt;
    if (bal) {  // item k + 2
      const int idx = lo + warp + (k + 2) * PB_WARPS;
      i1 = (idx < hi) ? idx : -1;
    } else {
      const int idx = (ck + nx_chunk * C) * IPC + warp + nx_within * PB_WARPS;
      const int cend = min(nwork, (ck + nx_chunk * C) * IPC + IPC);
      i1 = (idx < cend) ? idx : -1;
      if (++nx_within == per_chunk) {
        nx_within = 0;
        ++nx_chunk;
      }
    }
    mc = mn;
    mn = fetch(k + 2);
  }
  kb += k;
  if (SLOTS && lane == 0 && pv.kslots) bulk_wait_all();  // slot fills done before the stages are reused / exit
  if (pv.fused) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lk_h += __shfl_xor_sync(0xffffffffu, lk_h, o);
      lk_m += __shfl_xor_sync(0xffffffffu, lk_m, o);
      lv_h += __shfl_xor_sync(0xffffffffu, lv_h, o);
      lv_m += __shfl_xor_sync(0xffffffffu, lv_m, o);
      req_k += __shfl_xor_sync(0xffffffffu, req_k, o);
      req_v += __shfl_xor_sync(0xffffffffu, req_v, o);
    }
  }
  if (pv.fused && lane == 0) {
    if (lk_h | lk_m | lv_h | lv_m) {
      atomicAdd(pv.page_stats + u * 4 + 0, lk_h);
      atomicAdd(pv.page_stats + u * 4 + 1, lk_m);
      atomicAdd(pv.page_stats + u * 4 + 2, lv_h);
      atomicAdd(pv.page_stats + u * 4 + 3, lv_m);
      unsigned long long* ctr = reinterpret_cast<unsigned long long*>(pv.counters + (size_t)u * 6);
      atomicAdd(ctr + 0, (unsigned long long)lk_h);
      atomicAdd(ctr + 1, (unsigned long long)lk_m);
      atomicAdd(ctr + 2, (unsigned long long)lk_m * (B * D * 2));
      atomicAdd(ctr + 3, (unsigned long long)lv_h);
      atomicAdd(ctr + 4, (unsigned long long)lv_m);
      atomicAdd(ctr + 5, (unsigned long long)lv_m * (B * D * 2));
      atomicAdd(pv.klru + (size_t)u * pv.kstride + 0, req_k);  // clock T
      atomicAdd(pv.klru + (size_t)u * pv.kstride + 2, lk_m);   // resident count
      atomicAdd(pv.vlru + (size_t)u * pv.vstride + 0, req_v);
      atomicAdd(pv.vlru + (size_t)u * pv.vstride + 2, lv_m);
    }
  }

  // ---- reduce within the warp (per head), then across the 4 warps ----------
  dden += __shfl_xor_sync(0xffffffffu, dden, 4);
  dden += __shfl_xor_sync(0xffffffffu, dden, 8);
  dden += __shfl_xor_sync(0xffffffffu, dden, 16);
  canary = fmaxf(canary, __shfl_xor_sync(0xffffffffu, canary, 4));
  canary = fmaxf(canary, __shfl_xor_sync(0xffffffffu, canary, 8));
  canary = fmaxf(canary, __shfl_xor_sync(0xffffffffu, canary, 16));
  const float oz = accz[0] + accz[1];
  const float inv = pow2f(-Sx);
  __syncthreads();
  float* accs = reinterpret_cast<float*>(S.rec);             // [warp][H][D]
  float* mw = accs + PB_WARPS * H * D;                        // [warp][H][4]
  double* dw = reinterpret_cast<double*>(mw + PB_WARPS * H * 4);  // [warp][H][2]
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const float zg = __shfl_sync(0xffffffffu, oz, 4 * g + h);
    const int c0 = 16 * g + t0;
    accs[(warp * H + h) * D + c0] = fmaf(acc[g][0] + acc[g][1], 16777216.f, zg) * inv;
    accs[(warp * H + h) * D + c0 + 8] = fmaf(acc[g][2] + acc[g][3], 16777216.f, zg) * inv;
  }
  if (lane < H) {
    mw[(warp * H + lane) * 4 + 0] = m_h;
    mw[(warp * H + lane) * 4 + 1] = dden;
    mw[(warp * H + lane) * 4 + 2] = canary;
    dw[(warp * H + lane) * 2 + 0] = eF;
    dw[(warp * H + lane) * 2 + 1] = sF;
  }
  __syncthreads();
  for (int hh = 0; hh < H; ++hh) {
    float M = ninf();
    for (int w = 0; w < PB_WARPS; ++w) M = fmaxf(M, mw[(w * H + hh) * 4]);
    float O = 0.f, DD = 0.f, CN = 0.f;
    double E2 = 0.0, S2 = 0.0;
    for (int w = 0; w < PB_WARPS; ++w) {
      const float sc = expf(mw[(w * H + hh) * 4] - M);
      O += accs[(w * H + hh) * D + tid] * sc;
      DD += mw[(w * H + hh) * 4 + 1] * sc;
      CN = fmaxf(CN, mw[(w * H + hh) * 4 + 2]);
      E2 += dw[(w * H + hh) * 2];
      S2 += dw[(w * H + hh) * 2 + 1];
    }
    float* o = cs + hh * CKV_CHUNK_FLOATS;
    o[8 + tid] = O;
    if (tid == 0) {
      o[0] = M;
      o[1] = DD;
      o[2] = CN;
      o[3] = 0.f;
      reinterpret_cast<double*>(o + 4)[0] = E2;
      reinterpret_cast<double*>(o + 4)[1] = S2;
    }
  }
}

// Persistent over (unit, chunk) items pulled from a device queue (balanced
// tail); without st.queue one CTA per (chunk, unit).
template <bool SLOTS>
__global__ void __launch_bounds__(PB_WARPS * 32, 3) k_pass_b(StepArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PassBSmem& S = *reinterpret_cast<PassBSmem*>(smem_raw);
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_PASS_B);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int w = 0; w < PB_WARPS; ++w) {
      mbar_init(&S.bar[w][0], 1);
      mbar_init(&S.bar[w][1], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int C = st.n_chunks;
  int kb = 0;
  if (!st.queue) {
    const int u = a.u0 + blockIdx.y;
    const int U = a.c.n_units;
    if (st.flow) {
      pdl_trigger();
      flow_wait(st.flow + FLOW_SEL_DONE * U + u, st.epoch);  // this unit's selection + union
    }
    pass_b_chunk<SLOTS>(a, S, u, blockIdx.x, C, kb);
    if (st.flow) flow_arrive(st.flow + FLOW_PB_CNT * U + u, st.flow + FLOW_PB_DONE * U + u, gridDim.x, st.epoch);
    return;
  }
  __shared__ int s_item;
  const int total = a.nu * C;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(&st.queue[0], 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= total) break;
    pass_b_chunk<SLOTS>(a, S, a.u0 + item / C, item % C, C, kb);
  }
  if (tid == 0) {  // the last CTA out resets the queue for the next launch
    __threadfence();
    if (atomicAdd(&st.queue[1], 1) == (int)gridDim.x - 1) {
      st.queue[0] = 0;
      st.queue[1] = 0;
      __threadfence();
    }
  }
}

// -----------------------------------------------------------------------------
// Step-wide Rung 4 and the dense work list (k_group_flags + k_resolve in the
// dataflow): every unit's last combine CTA lists the unit if one of its own heads
// returns dense; the last combine CTA of the step only has work when some head
// requested Rung 4 -- then every head of the requesting units' groups turns
// dense (harness.py:362-372) and the list is rebuilt over all units.
__device__ void unit_dense_item(const ckv_cache& c, const ckv_step& st, int u) {
  const int nh = st.n_heads;
  int mask = 0;
  for (int h = 0; h < nh; ++h)
    if (__ldcg(&st.cert[(size_t)u * nh + h].returned_kind) != 0) mask |= 1 << h;
  if (mask) {
    const int slot = atomicAdd(flow_step(st.flow, c.n_units, FLOW_DENSE_N), 1);
    st.dense_list[1 + c.n_units + slot] = u | (mask << 24);
  }
}

__device__ void resolve_step(const ckv_cache& c, const ckv_step& st) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nh = st.n_heads, U = c.n_units;
  int32_t* nlist = flow_step(st.flow, U, FLOW_DENSE_N);
  int32_t* any4 = flow_step(st.flow, U, FLOW_ANY4);
  __shared__ int count, rung4;
  if (tid == 0) {
    rung4 = __ldcg(any4);
    count = rung4 ? 0 : __ldcg(nlist);
  }
  __syncthreads();
  if (rung4) {
    for (int u = tid; u < U; u += nt) {
      const int g = rung4_group_of(st, u);
      const bool gf = (g >= 0 && g < st.n_groups) && __ldcg(&st.group_flags[g]) != 0;
      int mask = 0;
      for (int h = 0; h < nh; ++h) {
        ckv_cert& ct = st.cert[(size_t)u * nh + h];
        if (gf) ct.returned_kind = 2;
        if (__ldcg(&ct.returned_kind) != 0) mask |= 1 << h;
      }
      if (mask) {
        const int slot = atomicAdd(&count, 1);
        st.dense_list[1 + U + slot] = u | (mask << 24);
      }
    }
    __syncthreads();
    for (int g = tid; g < st.n_groups; g += nt) st.group_flags[g] = 0;  // for the next step
  }
  __syncthreads();
  if (tid == 0) {
    st.dense_list[0] = count;
    *nlist = 0;
    *any4 = 0;
  }
}

__global__ void __launch_bounds__(128) k_combine(StepArgs a) {
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_COMBINE);
  const ckv_policy& pol = a.pol;
  const int h = blockIdx.x, u = a.u0 + blockIdx.y, tid = threadIdx.x;
  if (st.flow && !st.queue) flow_wait(st.flow + FLOW_PB_DONE * c.n_units + u, st.epoch);  // its pass B
  const int nh = st.n_heads;
  const size_t hu = (size_t)u * nh + h;
  const HeadState& hs = *reinterpret_cast<const HeadState*>(st.head_state + hu * CKV_HEAD_FLOATS);
  const int C = st.n_chunks;                          // chunk-state stride
  const int Cu = a.nchunk > 0 ? a.nchunk : C;         // chunks written this step
  const int pl = c.partial_len[u];
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  auto chunk = [&](int k) -> const float* {
    return st.chunk_state + (((size_t)u * C + k) * H + h) * CKV_CHUNK_FLOATS;
  };
  __shared__ float cm[256], csc[256];
  __shared__ float red[8];
  // chunk frames: headers in parallel, one max, then independent loads per channel
  float ml = ninf();
  for (int k = tid; k < Cu; k += blockDim.x) {
    cm[k] = chunk(k)[0];
    ml = fmaxf(ml, cm[k]);
  }
  ml = warp_max(ml);
  if ((tid & 31) == 0) red[tid >> 5] = ml;
  __syncthreads();
  float M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  if (hs.lA > 0.f) M = fmaxf(M, hs.mA);
  if (pl > 0) M = fmaxf(M, hs.mp);
  for (int k = tid; k < Cu; k += blockDim.x) csc[k] = (cm[k] == ninf()) ? 0.f : expf(cm[k] - M);
  __syncthreads();
  float den = 0.f, num = 0.f;
  if (hs.lA > 0.f) {
    const float sc = expf(hs.mA - M);
    den += hs.lA * sc;
    num += hs.oA[tid] * sc;
  }
  float canary = 0.f;
  double eF = 0.0, sF = 0.0;
#pragma unroll 8
  for (int k = 0; k < Cu; ++k) {
    const float* cs = chunk(k);
    const float sc = csc[k];
    den += cs[1] * sc;
    num += cs[8 + tid] * sc;
  }
  {  // canary max and the F parts of E_val: chunks spread over the threads
    __shared__ float cw[4];
    __shared__ double ew[4], sw[4];
    for (int k = tid; k < Cu; k += blockDim.x) {
      if (cm[k] == ninf()) continue;
      const float* cs = chunk(k);
      canary = fmaxf(canary, cs[2]);
      eF += reinterpret_cast<const double*>(cs + 4)[0];
      sF += reinterpret_cast<const double*>(cs + 4)[1];
    }
    canary = warp_max(canary);
    eF = warp_sum_d(eF);
    sF = warp_sum_d(sF);
    if ((tid & 31) == 0) {
      cw[tid >> 5] = canary;
      ew[tid >> 5] = eF;
      sw[tid >> 5] = sF;
    }
    __syncthreads();
    canary = fmaxf(fmaxf(cw[0], cw[1]), fmaxf(cw[2], cw[3]));
    eF = (ew[0] + ew[1]) + (ew[2] + ew[3]);
    sF = (sw[0] + sw[1]) + (sw[2] + sw[3]);
  }
  if (pl > 0) {
    const float sc = expf(hs.mp - M);
    den += hs.lp * sc;
    num += hs.np_[tid] * sc;
  }
  const float out = num / den;
  if (!isfinite(out) || !(den > 0.f)) atomicOr(&bad, 1);
  st.out[hu * D + tid] = out;
  __syncthreads();

  // ---- ranking: top-r of the phase-2 log-masses over F (ties -> lower block
  // index) against the phase-1 order prefix (fallback.py:164-187,
  // harness.py:231-250); one block-wide argmax per rank, all threads
  const int kp = hs.kprime;
  const int r = pol.ranking_depth;
  const int32_t* order = st.order + hu * st.kcap;
  const float* lm2 = st.lm2 + hu * c.max_blocks;
  __shared__ int picked[64];
  __shared__ float rvw[4];
  __shared__ int rbw[4];
  __shared__ int same_s;
  __shared__ float rth_s;
  const bool do_rank = pol.ranking_checks_enabled && kp > 0 && kp >= r;
  if (do_rank) {
    const int rr = min(r, 64);
    if (tid == 0) same_s = 1;
    for (int j = 0; j < rr; ++j) {
      float bv = ninf();
      int bb = 0x7fffffff;
      for (int i = tid; i < kp; i += blockDim.x) {
        const int bi = order[i];
        bool used = false;
        for (int q = 0; q < j; ++q) used |= (picked[q] == bi);
        if (used) continue;
        const float v = lm2[bi];
        if (bb == 0x7fffffff || v > bv || (v == bv && bi < bb)) {
          bv = v;
          bb = bi;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
        if (ob != 0x7fffffff && (bb == 0x7fffffff || ov > bv || (ov == bv && ob < bb))) {
          bv = ov;
          bb = ob;
        }
      }
      if ((tid & 31) == 0) {
        rvw[tid >> 5] = bv;
        rbw[tid >> 5] = bb;
      }
      __syncthreads();
      if (tid == 0) {
        float v0 = rvw[0];
        int b0 = rbw[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
          if (rbw[w] != 0x7fffffff && (b0 == 0x7fffffff || rvw[w] > v0 || (rvw[w] == v0 && rbw[w] < b0))) {
            v0 = rvw[w];
            b0 = rbw[w];
          }
        }
        picked[j] = b0;
        rth_s = v0;
        if (order[j] != b0) same_s = 0;
      }
      __syncthreads();
    }
  }

  // E_val's terms are taken relative to the Phase-1 lse.  When Phase 2 moves every
  // mass more than ~700 nats below it (corrupted key metadata: the canary trips by
  // orders of magnitude) they underflow in fp64; then E_val is recomputed from the
  // block log-masses against the Phase-2 maximum (certifier.py:153-160) -- one
  // pass over the unit's blocks, on this rare path only
  __shared__ double ev_fix;
  if (!(hs.alpha_hat + hs.partial_mass + sF > 1e-250)) {
    __shared__ uint32_t fb[(CKV_MAX_BLOCKS + 31) / 32], vb[(CKV_MAX_BLOCKS + 31) / 32];
    __shared__ float mw[4];
    __shared__ double nw[4], dw[4];
    const int nb = c.n_blocks[u];
    const int nw32 = (nb + 31) / 32;
    for (int i = tid; i < nw32; i += blockDim.x) fb[i] = vb[i] = 0u;
    __syncthreads();
    const int32_t* vl = st.vlist + hu * c.max_blocks;
    for (int i = tid; i < kp; i += blockDim.x) atomicOr(&fb[order[i] >> 5], 1u << (order[i] & 31));
    for (int i = tid; i < hs.n_v; i += blockDim.x) atomicOr(&vb[vl[i] >> 5], 1u << (vl[i] & 31));
    __syncthreads();
    const float* lm1 = st.lm1 + hu * c.max_blocks;
    auto ell = [&](int b) -> float { return ((fb[b >> 5] >> (b & 31)) & 1u) ? lm2[b] : lm1[b]; };
    const float lpart = (pl > 0) ? hs.mp + logf(hs.lp) : ninf();
    float mx = lpart;
    for (int b = tid; b < nb; b += blockDim.x) mx = fmaxf(mx, ell(b));
    mx = warp_max(mx);
    if ((tid & 31) == 0) mw[tid >> 5] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(mw[0], mw[1]), fmaxf(mw[2], mw[3]));
    double num = 0.0, den = 0.0;
    const float* eta = c.eta + (size_t)u * c.max_blocks;
    for (int b = tid; b < nb; b += blockDim.x) {
      const double w = exp((double)ell(b) - (double)mx);
      den += w;
      if (!((vb[b >> 5] >> (b & 31)) & 1u)) num += w * (double)eta[b];
    }
    num = warp_sum_d(num);
    den = warp_sum_d(den);
    if ((tid & 31) == 0) {
      nw[tid >> 5] = num;
      dw[tid >> 5] = den;
    }
    __syncthreads();
    if (tid == 0) {
      num = (nw[0] + nw[1]) + (nw[2] + nw[3]);
      den = (dw[0] + dw[1]) + (dw[2] + dw[3]);
      if (pl > 0) den += exp((double)lpart - (double)mx);
      ev_fix = (den > 0.0) ? num / den : 0.0;
    }
    __syncthreads();
  } else if (tid == 0) {
    ev_fix = -1.0;
  }

  if (tid == 0) {
    ckv_cert& ct = st.cert[hu];
    uint32_t fl = ct.flags;
    const double delta = (double)hs.delta;
    if (pol.ranking_checks_enabled && kp > 0) {
      if (kp < r) {
        fl |= CKV_F_RANKING;
      } else {
        if (!same_s) fl |= CKV_F_RANKING;
        if (hs.tailmax != ninf() && !((double)hs.tailmax + delta <= (double)rth_s)) fl |= CKV_F_BOUNDARY;
      }
    }
    if (pol.canary_enabled && kp > 0) {
      if (!((double)canary <= delta + pol.epsilon_guard)) fl |= CKV_F_CANARY;
    }
    if (bad) fl |= CKV_F_NUMERIC;
    const double vmax = (double)c.v_max[u];
    const double at = hs.alpha_hat;
    const double denomE = at + hs.partial_mass + sF;
    ct.delta_h = delta;
    ct.est_tail_mass = at;
    ct.v_max = vmax;
    // certifier.py:191-212 records both exponent modes; returned_e_key uses mode 3
    ct.e_key_tight = 2.0 * vmax * exp(2.0 * delta) * at * (exp(2.0 * delta) - 1.0);
    ct.e_key_impl = 2.0 * vmax * exp(3.0 * delta) * at * (exp(2.0 * delta) - 1.0);
    ct.e_val = (ev_fix >= 0.0) ? ev_fix : (hs.e_tail + eF) / denomE;
    ct.canary_gap = (double)canary;
    ct.flags = fl;
    int kind = 0;
    if (fl & (CKV_F_CANARY | CKV_F_NUMERIC)) kind = 2;
    else if (fl & (CKV_F_RANKING | CKV_F_BOUNDARY)) kind = 1;
    ct.returned_kind = kind;
    if (a.finish && kind == 2) {  // a step-wide Rung-4 request for the unit's group
      const int g = rung4_group_of(st, u);
      if (g >= 0 && g < st.n_groups) atomicOr(&st.group_flags[g], 1);
      atomicOr(flow_step(st.flow, c.n_units, FLOW_ANY4), 1);
    }
  }
  if (a.finish) {  // the unit's last head lists it, the step's last CTA resolves
    __shared__ int last_u, last;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      int32_t* cu = st.flow + FLOW_CB_UNIT * c.n_units + u;
      last_u = atomicAdd(cu, 1) == nh - 1;
      if (last_u) {
        *cu = 0;
        __threadfence();
        unit_dense_item(c, st, u);
      }
      int32_t* cnt = flow_step(st.flow, c.n_units, FLOW_CB_CNT);
      __threadfence();
      last = atomicAdd(cnt, 1) == (int)(gridDim.x * gridDim.y) - 1;
      if (last) *cnt = 0;
      __threadfence();
    }
    __syncthreads();
    if (last) {
      resolve_step(c, st);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release_gpu(flow_step(st.flow, c.n_units, FLOW_RESOLVED), st.epoch);
    }
  }
}


static void passb_attrs(const ckv_cache* c) {
  set_max_dyn_smem(k_pass_b<false>, (int)sizeof(PassBSmem));
  set_max_dyn_smem(k_pass_b<true>, (int)sizeof(PassBSmem));
  set_max_dyn_smem(k_union, 2 * H * ((c->max_blocks + 31) / 32) * 4);
}

cudaError_t launch_union(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st, int u0, int nu,
                         cudaStream_t s) {
  passb_attrs(c);
  StepArgs a{*c, *st, *pol, PageView{}, u0};
  const int W = (c->max_blocks + 31) / 32;
  k_union<<<nu, UN_THREADS, 2 * H * W * 4, s>>>(a);
  g_launches += 1;
  return cudaGetLastError();
}

// Pass-B chunks per unit: the union list is split evenly over them, and their
// count makes units x chunks fill the SMs' pass-B slots (3 CTAs each) in whole
// waves -- chunks of 64..256 items of the expected union (<= 4 K' blocks).
static int pb_chunks(long long units, int kcap, int cap, int sms) {
  if (knobs().pb_chunks > 0) return min(cap, knobs().pb_chunks);
  const long long slots = (long long)sms * 3;
  const int items = (4 * kcap * 15) / 16;
  const int lo = max(1, (items + 255) / 256), hi = max(lo, min(cap, (items + 63) / 64));
  int best = min(lo, cap);
  double best_eff = -1.0;
  for (int c = lo; c <= hi && c <= cap; ++c) {
    const long long ctas = units * c;
    const long long waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = c;
    }
  }
  return best;
}

cudaError_t launch_passb(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st,
                         const PageView& pv, int u0, int nu, bool pdl, bool finish, cudaStream_t s) {
  passb_attrs(c);
  StepArgs a{*c, *st, *pol, pv, u0, nu, 0, finish && st->flow && !st->queue ? 1 : 0};
  a.nchunk = st->queue ? 0 : pb_chunks(st->plan_units > 0 ? st->plan_units : nu, st->kcap, st->n_chunks,
                                       dev_state().sms);
  // the dataflow chain (st->flow): pass B right behind the selection, combine
  // right behind pass B, each waiting per unit (no persistent queue in that mode)
  const bool flow = st->flow != nullptr && !st->queue;
  const bool slots_ = pv.kslots || pv.vslots;
  if (st->queue) {
    DevState& ds = dev_state();
    if (!ds.passb_slots) {
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pass_b<false>, PB_WARPS * 32, sizeof(PassBSmem));
      ds.passb_slots = max(1, ds.sms * max(1, per));
    }
    const int slots = ds.passb_slots;
    const int grid = min(slots, nu * st->n_chunks);
    if (slots_) k_pass_b<true><<<grid, PB_WARPS * 32, sizeof(PassBSmem), s>>>(a);
    else k_pass_b<false><<<grid, PB_WARPS * 32, sizeof(PassBSmem), s>>>(a);
  } else {
    const dim3 g(a.nchunk, nu);
    cudaError_t e = slots_ ? launch_k(pdl && flow, k_pass_b<true>, g, dim3(PB_WARPS * 32), sizeof(PassBSmem), s, a)
                           : launch_k(pdl && flow, k_pass_b<false>, g, dim3(PB_WARPS * 32), sizeof(PassBSmem), s, a);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_k(flow, k_combine, dim3(st->n_heads, nu), dim3(128), 0, s, a);
  g_launches += 2;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace ckv
