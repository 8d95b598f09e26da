// Phase-1 block scoring on the tensor cores, shared by pass A and pass B so
// both see bit-identical quantized scores.
//
// s'_t,h = sum_c q'_hc (code_tc * sigma_c + z_c),  q' = q / sqrt(d)
//        = 2^(eQ_h + eS_b - 21) * sum_c code_tc * X_hc + constz_h
// with X_hc = rint(q'_hc 2^(21-eQ_h) * sigma_c 2^(-eS_b)), |X| < 2^21.
// The INT8 codes are the A operand of mma.m16n8k32.s8.u8 straight from the
// record (no conversion); X is fed as three unsigned bytes of U = X + 2^22
// (taken directly from the fp32 bit pattern of fma(x, 1, 1.5*2^23)), and a
// column of ones recovers sum_c code_tc to remove the 2^22 bias.
//
// B-operand column map (n = lane/4 for the fragment that a lane supplies):
//   tile 0: n = 2h + {0,1}  -> head h, byte 0 / byte 1 of U
//   tile 1: n = 2h          -> head h, byte 2 of U;  n = 2h + 1 -> ones
// so accumulator lane l ends up owning head h = l % 4 for tokens l/4, l/4+8.
#pragma once
#include "common.cuh"

namespace ckv {

struct QFrag {
  float qsc[16];   // q'_{h,c} * 2^(21-eQ_h) for h = lane/8, the lane's half (4 per k-tile)
  int eq_l;        // exponent of head lane%4: max|q'_h| < 2^eq_l
};

// channel of the lane's j-th B element in k-tile kt
__device__ __forceinline__ int bchan(int lane, int kt, int j) {
  return kt * 32 + (lane & 3) * 4 + (j & 3) + ((j >> 2) << 4);
}

__device__ __forceinline__ float pow2f(int e) {  // exact 2^e, e clamped to the normal range
  e = max(-126, min(127, e));
  return __uint_as_float((uint32_t)(e + 127) << 23);
}

// qh: q'[4][128] float in shared memory.
__device__ inline void load_qfrag(QFrag& f, const float* qh, int lane) {
  const int hb = lane >> 3;
  int eq_b = 0;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    float m = 0.f;
    for (int c = lane; c < D; c += 32) m = fmaxf(m, fabsf(qh[h * D + c]));
    m = warp_max(m);
    const int e = (m > 0.f) ? (ilogbf(m) + 1) : 0;
    if (h == (lane & 3)) f.eq_l = e;
    if (h == hb) eq_b = e;
  }
  const float sc = pow2f(21 - eq_b);
  const int half = (lane >> 2) & 1;
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
#pragma unroll
    for (int i = 0; i < 4; ++i) f.qsc[kt * 4 + i] = qh[hb * D + bchan(lane, kt, 4 * half + i)] * sc;
  }
}

struct BlockScores {
  float s0, s1;    // scores of tokens lane/4 and lane/4+8 for head lane%4
  float delta;     // Delta_b for head lane%4 (already / 2 / sqrt(d) folded)
};

// rec: Tier-1 record in shared (or global) memory; smax: the block's max key scale.
__device__ __forceinline__ BlockScores phase1_block(const QFrag& f, const uint8_t* rec, float smax,
                                                    int lane) {
  const float* sig = reinterpret_cast<const float*>(rec + OFF_KSCALE);
  const float* zz = reinterpret_cast<const float*>(rec + OFF_KOFF);
  const int es = ilogbf(smax) + 1;    // smax < 2^es
  // fma(qsc, sigma, 1.5*2^(23+es)) has the same mantissa bits as
  // fma(qsc, sigma*2^-es, 1.5*2^23) (exact power-of-two scaling): the bytes of
  // U = X + 2^22 come out unchanged, except that byte 2 carries the exponent
  // LSB (es & 1) in its top bit, removed below with the sum-of-codes column.
  const float magic_b = __uint_as_float(((uint32_t)(150 + es) << 23) | 0x400000u);
  // Lanes l and l^4 (byte parity of the same head) share their y values: each
  // computes 4 of the 8 channels of a k-tile (one 16-byte sigma / z load each
  // instead of two) and they swap halves with a shuffle.  The shared-memory
  // data pipe is pass A's bottleneck.  Delta and sum q z partials are taken
  // over the lane's own 4 channels and reduced over the 8 lanes of the head.
  const int half = (lane >> 2) & 1;
  int d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
  float dacc = 0.f, zacc = 0.f;
#pragma unroll
  for (int kt = 0; kt < 4; ++kt) {
    const int cm = kt * 32 + (lane & 3) * 4 + 16 * half;  // my 4 channels
    const float4 s4 = *reinterpret_cast<const float4*>(sig + cm);
    const float4 z4 = *reinterpret_cast<const float4*>(zz + cm);
    const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
    const float zv[4] = {z4.x, z4.y, z4.z, z4.w};
    uint32_t ym[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float q = f.qsc[kt * 4 + i];
      ym[i] = __float_as_uint(fmaf(q, sv[i], magic_b));
      dacc = fmaf(fabsf(q), sv[i], dacc);
      zacc = fmaf(q, zv[i], zacc);
    }
    // all three byte planes of my 4 y values (7 PRMT), then one shuffle of the
    // plane the partner needs for tile 0 (its byte parity) and one of byte 2
    const uint32_t a01 = __byte_perm(ym[0], ym[1], 0x5140u), a23 = __byte_perm(ym[2], ym[3], 0x5140u);
    const uint32_t c01 = __byte_perm(ym[0], ym[1], 0x6262u), c23 = __byte_perm(ym[2], ym[3], 0x6262u);
    const uint32_t pl0 = __byte_perm(a01, a23, 0x5410u);  // byte 0 of y0..y3
    const uint32_t pl1 = __byte_perm(a01, a23, 0x7632u);  // byte 1
    const uint32_t pl2 = __byte_perm(c01, c23, 0x5410u);  // byte 2
    const uint32_t r1 = __shfl_xor_sync(0xffffffffu, half ? pl0 : pl1, 4);  // partner's byte p
    const uint32_t r2 = __shfl_xor_sync(0xffffffffu, pl2, 4);               // partner's byte 2
    // tile 0: byte p of channels cb..cb+3 (b00) and cb+16..cb+19 (b01);
    // tile 1: byte 2 (even lane/4) or the ones column (odd lane/4)
    const uint32_t b00 = half ? r1 : pl0, b01 = half ? pl1 : r1;
    const uint32_t b10 = half ? 0x01010101u : pl2, b11 = half ? 0x01010101u : r2;
    const uint4 a = *reinterpret_cast<const uint4*>(rec + OFF_KCODES + kt * 512 + lane * 16);
    mma_s8u8(d0, a, b00, b01);
    mma_s8u8(d1, a, b10, b11);
  }
  // reduce over the 8 lanes of head lane/8, then fetch head lane%4's sums
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    zacc += __shfl_xor_sync(0xffffffffu, zacc, o);
  }
  const int h = lane & 3;
  const float dsum = __shfl_sync(0xffffffffu, dacc, h * 8);  // sum |qsc| sigma (head h)
  const float zsum = __shfl_sync(0xffffffffu, zacc, h * 8);  // sum qsc z (head h)
  const float inv_q = pow2f(f.eq_l - 21);
  const float scl = pow2f(f.eq_l + es - 21);
  const float constz = zsum * inv_q;
  const int bias = 64 + ((es & 1) << 7);
  BlockScores r;
  {
    int lo = d0[0] + 256 * d0[1];
    int hi = d1[0] - bias * d1[1];
    r.s0 = fmaf(fmaf((float)hi, 65536.f, (float)lo), scl, constz);
  }
  {
    int lo = d0[2] + 256 * d0[3];
    int hi = d1[2] - bias * d1[3];
    r.s1 = fmaf(fmaf((float)hi, 65536.f, (float)lo), scl, constz);
  }
  r.delta = 0.5f * dsum * inv_q;
  return r;
}

// ---------------------------------------------------------------------------
// Original-key scores of a 16-token block for the four q-heads on the tensor
// cores: A = the block's FP16 keys (fragment order, exact), B = q' split into
// fp16 hi + lo (scaled by 2^(14-eQ) into fp16 range), fp32 accumulation.
// Column n = 2h + part, so accumulator lane l owns head l%4 for tokens l/4,
// l/4+8 -- the same layout as phase1_block.
struct QFrag16 {
  uint32_t b[8][2];
  float unscale;  // 2^(eQ - 14) for head lane%4
};

__device__ inline void load_qfrag16(QFrag16& f, const float* qh, int lane) {
  const int hb = lane >> 3, part = (lane >> 2) & 1;
  int eq_b = 0, eq_l = 0;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    float m = 0.f;
    for (int c = lane; c < D; c += 32) m = fmaxf(m, fabsf(qh[h * D + c]));
    m = warp_max(m);
    const int e = (m > 0.f) ? (ilogbf(m) + 1) : 0;
    if (h == (lane & 3)) eq_l = e;
    if (h == hb) eq_b = e;
  }
  const float sc = pow2f(14 - eq_b);
  f.unscale = pow2f(eq_l - 14);
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int c = kt * 16 + (lane & 3) * 2 + 8 * p;
      const float x0 = qh[hb * D + c] * sc, x1 = qh[hb * D + c + 1] * sc;
      __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
      if (part) {
        h0 = __float2half_rn(x0 - __half2float(h0));
        h1 = __float2half_rn(x1 - __half2float(h1));
      }
      __half2 v = __halves2half2(h0, h1);
      f.b[kt][p] = *reinterpret_cast<uint32_t*>(&v);
    }
  }
}

// kf: the block's Tier-2 keys (4 KB, fragment order) in global memory.
__device__ __forceinline__ float2 orig_block(const QFrag16& f, const uint4* kf, int lane) {
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  uint4 a[8];
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) a[kt] = kf[kt * 32 + lane];
#pragma unroll
  for (int kt = 0; kt < 8; ++kt) mma_f16(d, a[kt], f.b[kt][0], f.b[kt][1]);
  return make_float2((d[0] + d[1]) * f.unscale, (d[2] + d[3]) * f.unscale);
}

}  // namespace ckv
