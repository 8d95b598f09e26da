// Device-side state shared by the decode-step kernels.
#pragma once
#include <cstddef>
#include "phase1.cuh"

namespace ckv {

struct HeadState {
  double lse;          // phase-1 log-sum-exp over full blocks + partial
  double alpha_hat;    // estimated tail mass (non-promoted full blocks)
  double e_tail;       // sum over b not in F u V of p_b eta_b
  double partial_mass;
  float mA, lA;        // merged pass-A softmax state
  float delta;         // Delta_h
  float tailmax;       // max phase-1 log-mass over the tail (-inf if empty)
  float mp, lp;        // partial block state
  int32_t kprime;      // |F| after rung 1
  int32_t kstar0;      // K* before rung 1
  int32_t n_v;
  int32_t k_cov;
  int32_t pad[2];
  float oA[D];
  float np_[D];
};
static_assert(sizeof(HeadState) <= CKV_HEAD_FLOATS * 4, "head state too large");


// Where pass B reads promoted originals from: HBM scratch slots (Tier-2 in host
// RAM, blocks resident after this step's LRU) or Tier-2 itself.
struct PageView {
  const uint16_t* kslots;
  const uint16_t* vslots;
  const int32_t* kslot_of;  // per unit: + u * kstride
  const int32_t* vslot_of;
  int32_t kstride, vstride, kcap, vcap;
  // fused LRU accounting (no-eviction scratch without HBM slots): pass B stamps
  // the requested blocks and counts hits / misses itself
  int32_t* klru;
  int32_t* vlru;
  int64_t* counters;
  int32_t* page_stats;
  int32_t fused;
};

struct StepArgs {
  ckv_cache c;
  ckv_step st;
  ckv_policy pol;
  PageView pv;
  int32_t u0;  // first unit of this launch (units u0 + blockIdx)
  int32_t nu;  // units in this launch (persistent kernels)
  int32_t nsplit;  // pass-A splits per unit of this step (<= st.n_splits, pa_splits())
  int32_t finish;  // the last combine CTA resolves the step (group flags, dense list)
  int32_t nchunk;  // pass-B chunks per unit of this step, balanced over the union (0: IPC-sized)
};

__device__ __forceinline__ int rung4_group_of(const ckv_step& st, int u) {
  return st.unit_group ? st.unit_group[u] : u / st.rung4_group;
}

// Exponent S of the unit's value scaling: every fp16 product p' * scale with
// p' = p * 2^S <= 2^S stays below 2^15 (scale <= max(2 v_max / 15, 1), since
// |v| <= nu <= v_max and a constant group has scale 1).
__device__ __forceinline__ int value_exp(float vmax) {
  const float sb = fmaxf(2.f * vmax * (1.f / 15.f), 1.f);
  return 14 - (ilogbf(sb) + 1);
}

__device__ __forceinline__ float ninf() { return __int_as_float(0xff800000); }

__device__ __forceinline__ uint32_t okey(float x) {  // order-preserving float -> u32
  uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float ukey(uint32_t k) {  // inverse of okey
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// The union work list of unit u: every block some q-head promotes (F_h) or
// value-promotes (V_h), ascending, as block | F-mask << 24 | V-mask << 28.
// Word-parallel over the per-head bitmaps; ub = 2 * H * ceil(nb / 32) words of
// shared memory, ws = 32 ints; blockDim.x a multiple of 32.
__device__ inline void build_union(const ckv_cache& c, const ckv_step& st, int u, uint32_t* ub,
                                   int* ws) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int nh = st.n_heads;
  const int nb = c.n_blocks[u];
  const int W = (nb + 31) / 32;
  uint32_t* fb = ub;           // [H][W]
  uint32_t* vb = ub + H * W;   // [H][W]
  for (int i = tid; i < 2 * H * W; i += nt) ub[i] = 0u;
  __syncthreads();
  for (int h = 0; h < nh; ++h) {
    const size_t hu = (size_t)u * nh + h;
    const int kp = __ldcg(&st.cert[hu].k_star);
    const int nv = __ldcg(&st.cert[hu].n_value_promoted);
    const int32_t* ord = st.order + hu * st.kcap;
    const int32_t* vl = st.vlist + hu * c.max_blocks;
    for (int i = tid; i < kp; i += nt) {
      const int b = __ldcg(ord + i);
      atomicOr(&fb[h * W + (b >> 5)], 1u << (b & 31));
    }
    for (int i = tid; i < nv; i += nt) {
      const int b = __ldcg(vl + i);
      atomicOr(&vb[h * W + (b >> 5)], 1u << (b & 31));
    }
  }
  __syncthreads();
  int32_t* work = st.work + (size_t)u * st.wcap;
  int base = 0;
  for (int w0 = 0; w0 < W; w0 += nt) {
    const int w = w0 + tid;
    uint32_t any = 0;
    if (w < W)
      for (int h = 0; h < nh; ++h) any |= fb[h * W + w] | vb[h * W + w];
    const int cnt = __popc(any);
    int x = cnt;  // block-wide exclusive scan of the per-word counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < nw; ++k) {
      const int v = ws[k];
      before += (k < warp) ? v : 0;
      total += v;
    }
    int pos = base + before + x - cnt;
    while (any) {
      const int bit = __ffs(any) - 1;
      any &= any - 1;
      const int b = w * 32 + bit;
      uint32_t fm = 0, vm = 0;
      for (int h = 0; h < nh; ++h) {
        fm |= ((fb[h * W + w] >> bit) & 1u) << h;
        vm |= ((vb[h * W + w] >> bit) & 1u) << h;
      }
      work[pos++] = b | (int)(fm << 24) | (int)(vm << 28);
    }
    base += total;
    __syncthreads();
  }
  if (tid == 0) st.n_work[u] = base;
}

// The speculative Phase-2 P.V of one block on the tensor cores.  The INT4
// codes are fed as fp16 *subnormals* (the bit pattern of the code u is the
// half u * 2^-24, so one AND per two codes builds the A operand, no bias);
// B = p' * scale per (token, group) as an fp16 hi/lo pair (column 2h + part),
// so each product is exact and the sum is fp32.  Tokens 8..15 enter as 16u
// (nibble at bits 4..7) with their B divided by 16.  The offsets add
// sum_t p'_t offset_t,g through one more MMA (rows = groups).
//   acc[g]: rows = channels 16g + l/4 (+8), cols = (head l%4, hi|lo), in
//           units of 2^(S-24);  accz: rows = groups, same cols, units 2^S.
struct PVFrag {
  uint32_t phi0, phi1;   // p' hi of tokens (2j, 2j+1), (2j+8, 2j+9)/16   [column head]
  uint32_t nph0, nph1;   // -phi on lo-part lanes, 0 on hi lanes
  uint32_t plo0, plo1;   // p' lo (/16 for the second) on lo lanes, 0 on hi lanes
  uint32_t z0, z1;       // offset-MMA B: p' hi (hi lanes) or lo (lo lanes), unscaled
};

__device__ __forceinline__ void pv_frag(PVFrag& F, const float4 p, bool lo_lane) {
  uint32_t h01, l01, h23, l23;
  split_h2(p.x, p.y, h01, l01);
  split_h2(p.z, p.w, h23, l23);
  F.z0 = lo_lane ? l01 : h01;
  F.z1 = lo_lane ? l23 : h23;
  const uint32_t s16 = 0x2c002c00u;  // half2(1/16, 1/16)
  const uint32_t h23s = h2_mul(h23, s16), l23s = h2_mul(l23, s16);
  F.phi0 = h01;
  F.phi1 = h23s;
  F.nph0 = lo_lane ? (h01 ^ 0x80008000u) : 0u;
  F.nph1 = lo_lane ? (h23s ^ 0x80008000u) : 0u;
  F.plo0 = lo_lane ? l01 : 0u;
  F.plo1 = lo_lane ? l23s : 0u;
}

__device__ __forceinline__ void pv_block_sub(float (&acc)[NG][4], float (&accz)[4], const PVFrag& F,
                                            const uint8_t* rec, int lane) {
  const uint4 w0 = *reinterpret_cast<const uint4*>(rec + OFF_VCODES + lane * 16);
  const uint4 w1 = *reinterpret_cast<const uint4*>(rec + OFF_VCODES + 512 + lane * 16);
  const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
  const uint4* sc = reinterpret_cast<const uint4*>(rec + OFF_VSCALE + (lane & 3) * 64);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 s4 = sc[q];  // groups 2q, 2q+1: (s_2j, s_2j+1), (s_2j+8, s_2j+9)
    const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 2 * q + e;
      const uint32_t s01 = sv[2 * e], s23 = sv[2 * e + 1];
      const uint32_t b0 = h2_fma(F.plo0, s01, h2_fma(F.phi0, s01, h2_mul(F.nph0, s01)));
      const uint32_t b1 = h2_fma(F.plo1, s23, h2_fma(F.phi1, s23, h2_mul(F.nph1, s23)));
      const uint32_t w = wv[(g >> 2) * 4 + (g & 3)];
      const uint32_t w8 = w >> 8;
      mma_f16r(acc[g], w & 0x000f000fu, w8 & 0x000f000fu, w & 0x00f000f0u, w8 & 0x00f000f0u, b0, b1);
    }
  }
  const uint2 oz = *reinterpret_cast<const uint2*>(rec + OFF_VOFF + ((lane & 3) * 8 + (lane >> 2)) * 8);
  mma_f16r(accz, oz.x, 0u, oz.y, 0u, F.z0, F.z1);
}


}  // namespace ckv
