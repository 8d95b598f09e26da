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
};

struct StepArgs {
  ckv_cache c;
  ckv_step st;
  ckv_policy pol;
  PageView pv;
  int32_t u0;  // first unit of this launch (units u0 + blockIdx)
};

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

}  // namespace ckv
