// Rung 3 / Rung 4 terminal fallback on device (fallback.py:230-255,
// harness.py:271-281, 362-372):
//
//   k_resolve      step-wide (per rung4 group of units) Rung 4: a canary or
//                  numeric flag anywhere makes every head of the group dense;
//                  builds the compact list of units that need a dense pass.
//   k_dense        exact softmax attention over the FP16 originals (full
//                  blocks from Tier-2 + the partial block), fp32, split over
//                  the sequence; the four q-heads of a unit share each K/V read.
//   k_dense_merge  merges the splits and overwrites the fast-path output of
//                  every dense head.
#include "common.cuh"

namespace ckv {

constexpr int DN_TOK = 2048;  // tokens per dense split
constexpr int DN_WARPS = 4;

struct DenseArgs {
  ckv_cache c;
  ckv_step st;
  int32_t group;     // units per rung-4 group
  int32_t n_dsplit;  // splits per unit
};

__device__ __forceinline__ float dninf() { return __int_as_float(0xff800000); }

__global__ void k_resolve(DenseArgs a) {
  // one CTA per rung-4 group
  const ckv_step& st = a.st;
  const int g0 = blockIdx.x * a.group;
  const int g1 = min(a.c.n_units, g0 + a.group);
  const int nh = st.n_heads;
  __shared__ int any4;
  if (threadIdx.x == 0) any4 = 0;
  __syncthreads();
  for (int i = g0 * nh + threadIdx.x; i < g1 * nh; i += blockDim.x) {
    if (st.cert[i].flags & (CKV_F_CANARY | CKV_F_NUMERIC)) any4 = 1;
  }
  __syncthreads();
  for (int u = g0 + threadIdx.x; u < g1; u += blockDim.x) {
    int mask = 0;
    for (int h = 0; h < nh; ++h) {
      ckv_cert& ct = st.cert[(size_t)u * nh + h];
      if (any4) ct.returned_kind = 2;
      if (ct.returned_kind != 0) mask |= 1 << h;
    }
    if (mask) {
      const int slot = atomicAdd(&st.dense_list[0], 1);
      st.dense_list[1 + slot] = u | (mask << 24);
    }
  }
}

struct DenseSmem {
  float qh[H][D];
  float s[DN_WARPS][B][H];
  float mrg[DN_WARPS][H][2];
};

__global__ void __launch_bounds__(DN_WARPS * 32) k_dense(DenseArgs a) {
  __shared__ DenseSmem S;
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  const int item = blockIdx.y, sp = blockIdx.x;
  if (item >= st.dense_list[0]) return;
  const int e = st.dense_list[1 + item];
  const int u = e & 0xffffff;
  const int nh = st.n_heads;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = c.n_blocks[u];
  const int pl = c.partial_len[u];
  const int ntok = nb * B + pl;
  const int t0 = sp * DN_TOK, t1 = min(ntok, t0 + DN_TOK);
  float* outp = st.dense_part + (((size_t)item * a.n_dsplit + sp) * H) * 132;
  for (int i = tid; i < H * D; i += blockDim.x) {
    const int h = i / D;
    S.qh[h][i % D] = (h < nh) ? (float)(st.q[((size_t)u * nh + h) * D + (i % D)] * 0.08838834764831845)
                              : 0.f;
  }
  __syncthreads();
  if (t0 >= t1) {
    for (int i = tid; i < H * 132; i += blockDim.x) outp[i] = (i % 132 == 0) ? dninf() : 0.f;
    return;
  }
  // Tier-2 must hold every full block we read (cache.py:138-142)
  for (int b = t0 / B + tid; b < min(nb, (t1 + B - 1) / B); b += blockDim.x)
    if (!c.tier2_valid[(size_t)u * c.max_blocks + b]) atomicOr(&c.status[CKV_ST_TIER2], 1);

  const size_t t2 = (size_t)u * c.max_blocks * B * D;
  float m[H], l[H], o[H][4];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    m[h] = dninf();
    l[h] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[h][j] = 0.f;
  }
  const int tok = lane >> 1, hf = lane & 1;
  for (int base = t0 + warp * B; base < t1; base += DN_WARPS * B) {
    // scores: two lanes per token, 64 channels each, 4 heads
    const int t = base + tok;
    float s4[H] = {0.f, 0.f, 0.f, 0.f};
    if (t < t1) {
      const uint16_t* kp = (t < nb * B) ? c.tier2_k + t2 + (size_t)t * D
                                        : c.partial_k + ((size_t)u * B + (t - nb * B)) * D;
      const uint4* k4 = reinterpret_cast<const uint4*>(kp + hf * 64);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 w = k4[k];
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 kf = __half22float2(*reinterpret_cast<const __half2*>(&ww[j]));
          const int ch = hf * 64 + k * 8 + 2 * j;
#pragma unroll
          for (int h = 0; h < H; ++h) s4[h] = fmaf(kf.x, S.qh[h][ch], fmaf(kf.y, S.qh[h][ch + 1], s4[h]));
        }
      }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) s4[h] += __shfl_xor_sync(0xffffffffu, s4[h], 1);
    if (hf == 0) {
#pragma unroll
      for (int h = 0; h < H; ++h) S.s[warp][tok][h] = (t < t1) ? s4[h] : dninf();
    }
    __syncwarp();
    const int nvalid = min(B, t1 - base);
    float sc[B][H];
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int h = 0; h < H; ++h) sc[i][h] = S.s[warp][i][h];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      float mx = m[h];
#pragma unroll
      for (int i = 0; i < B; ++i) mx = fmaxf(mx, sc[i][h]);
      const float al = (m[h] == dninf()) ? 0.f : expf(m[h] - mx);
      l[h] *= al;
#pragma unroll
      for (int j = 0; j < 4; ++j) o[h][j] *= al;
      m[h] = mx;
    }
    // values: lane owns channels 4*lane .. 4*lane+3
    for (int i = 0; i < nvalid; ++i) {
      const int tt = base + i;
      const uint16_t* vp = (tt < nb * B) ? c.tier2_v + t2 + (size_t)tt * D
                                         : c.partial_v + ((size_t)u * B + (tt - nb * B)) * D;
      const uint2 raw = *reinterpret_cast<const uint2*>(vp + lane * 4);
      const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
      const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float p = expf(sc[i][h] - m[h]);
        l[h] += p;
        o[h][0] = fmaf(p, a0.x, o[h][0]);
        o[h][1] = fmaf(p, a0.y, o[h][1]);
        o[h][2] = fmaf(p, a1.x, o[h][2]);
        o[h][3] = fmaf(p, a1.y, o[h][3]);
      }
    }
    __syncwarp();
  }
  // merge warps through shared memory (reuse S.s as scratch for o)
  __shared__ float ow[DN_WARPS][H][D];
  if (lane == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h) {
      S.mrg[warp][h][0] = m[h];
      S.mrg[warp][h][1] = l[h];
    }
  }
#pragma unroll
  for (int h = 0; h < H; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j) ow[warp][h][lane * 4 + j] = o[h][j];
  __syncthreads();
  for (int h = 0; h < H; ++h) {
    float M = dninf();
    for (int w = 0; w < DN_WARPS; ++w) M = fmaxf(M, S.mrg[w][h][0]);
    float L = 0.f, O = 0.f;
    if (M != dninf()) {
      for (int w = 0; w < DN_WARPS; ++w) {
        if (S.mrg[w][h][0] == dninf()) continue;
        const float sc2 = expf(S.mrg[w][h][0] - M);
        L += S.mrg[w][h][1] * sc2;
        O += ow[w][h][tid] * sc2;
      }
    }
    if (tid == 0) {
      outp[h * 132 + 0] = M;
      outp[h * 132 + 1] = L;
    }
    outp[h * 132 + 4 + tid] = O;
  }
}

__global__ void k_dense_merge(DenseArgs a) {
  const ckv_step& st = a.st;
  const int item = blockIdx.x;
  if (item >= st.dense_list[0]) return;
  const int e = st.dense_list[1 + item];
  const int u = e & 0xffffff, mask = (e >> 24) & 0xf;
  const int nh = st.n_heads;
  const int tid = threadIdx.x;
  for (int h = 0; h < nh; ++h) {
    if (!((mask >> h) & 1)) continue;
    const float* p0 = st.dense_part + ((size_t)item * a.n_dsplit * H) * 132;
    float M = dninf();
    for (int s = 0; s < a.n_dsplit; ++s) M = fmaxf(M, p0[(s * H + h) * 132]);
    float L = 0.f, O = 0.f;
    for (int s = 0; s < a.n_dsplit; ++s) {
      const float* p = p0 + (s * H + h) * 132;
      if (p[0] == dninf()) continue;
      const float sc = expf(p[0] - M);
      L += p[1] * sc;
      O += p[4 + tid] * sc;
    }
    st.out[((size_t)u * nh + h) * D + tid] = O / L;
  }
}

extern int g_launches;

cudaError_t launch_dense(const ckv_cache* c, const ckv_step* st, int host_max_tokens, cudaStream_t s) {
  DenseArgs a{*c, *st, st->rung4_group > 0 ? st->rung4_group : c->n_units, 0};
  a.n_dsplit = (host_max_tokens + DN_TOK - 1) / DN_TOK;
  if (a.n_dsplit < 1) a.n_dsplit = 1;
  if (a.n_dsplit > st->n_dsplit_cap) a.n_dsplit = st->n_dsplit_cap;
  cudaMemsetAsync(st->dense_list, 0, sizeof(int32_t), s);
  const int ngroups = (c->n_units + a.group - 1) / a.group;
  k_resolve<<<ngroups, 256, 0, s>>>(a);
  k_dense<<<dim3(a.n_dsplit, c->n_units), DN_WARPS * 32, 0, s>>>(a);
  k_dense_merge<<<c->n_units, 128, 0, s>>>(a);
  g_launches += 3;
  return cudaGetLastError();
}

}  // namespace ckv
