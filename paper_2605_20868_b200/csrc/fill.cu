// K1: quantize-on-append.  Tokens accumulate in an fp16 partial block per
// unit; every time 16 tokens are present the block is fitted atomically
// (keys: per-channel INT8, values: per-(token, group) INT4, fp64 arithmetic
// with explicit _rn intrinsics so nothing is contracted into an FMA), the
// Tier-1 record, annotations and Tier-2 originals are written, and v_max is
// raised.  Restates cache.py:76-120 and quantizer.py:105-236.
#include "common.cuh"

namespace ckv {

// quantizer.py:118-130 -- rint, clip, then a strict -1 / +1 refinement pass.
__device__ __forceinline__ double refine_code(double x, double step, double base, double lo,
                                              double hi) {
  double c = rint(__ddiv_rn(__dsub_rn(x, base), step));
  c = fmin(fmax(c, lo), hi);
  double err = fabs(__dsub_rn(x, __dadd_rn(__dmul_rn(c, step), base)));
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    double cand = fmin(fmax(c + (s == 0 ? -1.0 : 1.0), lo), hi);
    double e2 = fabs(__dsub_rn(x, __dadd_rn(__dmul_rn(cand, step), base)));
    if (e2 < err) {
      c = cand;
      err = e2;
    }
  }
  return c;
}

// numpy's 8-accumulator pairwise sum over 128 contiguous float64 values.
__device__ __forceinline__ double pairwise128(const double* a) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  for (int i = 8; i < 128; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

__global__ void k_check_finite(const uint4* k, const uint4* v, size_t n16, int32_t* status) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (; i < n16; i += stride) {
    uint4 a = k[i], b = v[i];
    uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bad |= ((w[j] & 0x7c00u) == 0x7c00u) | ((w[j] & 0x7c000000u) == 0x7c000000u);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status[CKV_ST_APPEND_BAD], 1);
}

struct FillArgs {
  ckv_cache c;
  const uint16_t* k_new;
  const uint16_t* v_new;
  int32_t n_tok;
};

// Fit block j of this append for unit u (the 16 tokens at [partial | new]
// positions 16 j ..) and write its record, Tier-2 originals and annotations at
// block index n_blocks[u] + j -- invisible to readers until n_blocks moves.
// v_max is raised here unless the caller commits it later (vmax_now = false).
__device__ __forceinline__ void fill_block(const FillArgs& a, int u, int j, bool vmax_now) {
  const ckv_cache& c = a.c;
  const int tid = threadIdx.x;
  const int p = c.partial_len[u];
  const int nf = (p + a.n_tok) / B;
  if (j >= nf) return;
  const int b = c.n_blocks[u] + j;
  if (b >= c.max_blocks) {
    if (tid == 0) atomicOr(&c.status[CKV_ST_CAPACITY], 1);
    return;
  }
  __shared__ __align__(16) uint8_t rec[REC];
  __shared__ uint16_t sv[B][D];
  __shared__ double sq[B][D];   // squared reconstruction error, then reused
  __shared__ double sn[B][D];   // squared value
  __shared__ uint8_t vcs[B][D]; // value codes, unpacked
  __shared__ float red[4];

  // ---- gather the 16 tokens of this block from [partial | new] -------------
  const size_t ubase_new = (size_t)u * a.n_tok * D;
  const size_t ubase_par = (size_t)u * B * D;
  const size_t t2base = ((size_t)u * c.max_blocks + b) * B * D;
  double kx[B];
#pragma unroll
  for (int t = 0; t < B; ++t) {
    int gi = j * B + t;
    uint16_t kb, vb;
    if (gi < p) {
      kb = c.partial_k[ubase_par + gi * D + tid];
      vb = c.partial_v[ubase_par + gi * D + tid];
    } else {
      kb = a.k_new[ubase_new + (size_t)(gi - p) * D + tid];
      vb = a.v_new[ubase_new + (size_t)(gi - p) * D + tid];
    }
    kx[t] = half_bits_to_double(kb);
    sv[t][tid] = vb;
    c.tier2_k[t2base + k2_offset(t, tid)] = kb;
    c.tier2_v[t2base + v2_offset(t, tid)] = vb;
  }

  // ---- keys: thread = channel (quantizer.py:133-150) ----------------------
  double lo = kx[0], hi = kx[0];
#pragma unroll
  for (int t = 1; t < B; ++t) {
    lo = fmin(lo, kx[t]);
    hi = fmax(hi, kx[t]);
  }
  const bool flat = (hi == lo);
  const double scale = flat ? 1.0 : __ddiv_rn(__dsub_rn(hi, lo), 255.0);
  const double offset = flat ? lo : __dadd_rn(lo, __dmul_rn(128.0, scale));
#pragma unroll
  for (int t = 0; t < B; ++t) {
    double code = refine_code(kx[t], scale, offset, -128.0, 127.0);
    rec[kcode_offset(t, tid)] = (uint8_t)(int8_t)(int)code;
  }
  const float s32 = __double2float_rn(scale);
  reinterpret_cast<float*>(rec + OFF_KSCALE)[tid] = s32;
  reinterpret_cast<float*>(rec + OFF_KOFF)[tid] = __double2float_rn(offset);
  float smax = warp_max(s32);
  if ((tid & 31) == 0) red[tid >> 5] = smax;
  __syncthreads();

  // ---- values: thread = (token t, group g) (quantizer.py:178-230) ----------
  {
    const int t = tid >> 3, g = tid & 7;
    double v[G];
#pragma unroll
    for (int i = 0; i < G; ++i) v[i] = half_bits_to_double(sv[t][g * G + i]);
    double vlo = v[0], vhi = v[0];
#pragma unroll
    for (int i = 1; i < G; ++i) {
      vlo = fmin(vlo, v[i]);
      vhi = fmax(vhi, v[i]);
    }
    const double vs = (vhi == vlo) ? 1.0 : __ddiv_rn(__dsub_rn(vhi, vlo), 15.0);
    const uint16_t s16 = double_to_half_rn(vs);
    const uint16_t o16 = double_to_half_rn(vlo);
    const double ns = half_bits_to_double(s16), no = half_bits_to_double(o16);
    uint32_t nib[G];
#pragma unroll
    for (int i = 0; i < G; ++i) {
      double code = refine_code(v[i], vs, vlo, 0.0, 15.0);
      nib[i] = (uint32_t)code;
      // eta uses the narrowed (stored) metadata: recon = code*scale + offset
      double recon = __dadd_rn(__dmul_rn(code, ns), no);
      double diff = __dsub_rn(recon, v[i]);
      sq[t][g * G + i] = __dmul_rn(diff, diff);
      sn[t][g * G + i] = __dmul_rn(v[i], v[i]);
    }
#pragma unroll
    for (int i = 0; i < G; ++i) vcs[t][g * G + i] = (uint8_t)nib[i];
    reinterpret_cast<uint16_t*>(rec + OFF_VSCALE)[vmeta_index(t, g)] = s16;
    reinterpret_cast<uint16_t*>(rec + OFF_VOFF)[vmeta_index(t, g)] = o16;
  }
  __syncthreads();
  // pack the nibbles in fragment order (common.cuh): 256 words, two per thread
  for (int wi = tid; wi < 256; wi += 128) {
    const int g = (wi >> 7) * 4 + (wi & 3), l = (wi >> 2) & 31;
    const int r = l >> 2, j = l & 3;
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = 2 * j + (k & 1) + 8 * (k >> 1);
#pragma unroll
      for (int up = 0; up < 2; ++up) {
        const int ch = 16 * g + r + 8 * up;
        w |= (uint32_t)vcs[t][ch] << vcode_bit(t, ch);
      }
    }
    *reinterpret_cast<uint32_t*>(rec + OFF_VCODES + wi * 4) = w;
  }
  __syncthreads();

  // ---- annotations: eta = max_t ||recon - v||, nu = max_t ||v|| -------------
  if (tid < 32) {
    double e = 0.0, n = 0.0;
    if (tid < B) {
      e = sqrt(pairwise128(sq[tid]));
      n = sqrt(pairwise128(sn[tid]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
      n = fmax(n, __shfl_xor_sync(0xffffffffu, n, o));
    }
    if (tid == 0) {
      size_t ib = (size_t)u * c.max_blocks + b;
      // rounded up to fp32: E_val / E_key built from the stored annotations stay
      // upper bounds of the fp64 ones (certifier.py:135-160)
      c.eta[ib] = __double2float_ru(e);
      c.nu[ib] = __double2float_ru(n);
      c.kscale_max[ib] = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
      c.tier2_valid[ib] = 1;
      if (vmax_now) atomicMax(reinterpret_cast<int*>(&c.v_max[u]), __float_as_int(__double2float_ru(n)));
    }
  }
  // ---- write the record -------------------------------------------------------
  uint4* dst = reinterpret_cast<uint4*>(c.tier1 + ((size_t)u * c.max_blocks + b) * REC);
  const uint4* srcv = reinterpret_cast<const uint4*>(rec);
  for (int i = tid; i < REC / 16; i += 128) dst[i] = srcv[i];
}

__global__ void __launch_bounds__(128) k_fill(FillArgs a) {
  if (a.c.status[CKV_ST_APPEND_BAD]) return;  // the whole append is rejected
  fill_block(a, blockIdx.y, blockIdx.x, true);
}

// One-token append (the decode step's) in one launch: every unit checks its token,
// writes it into its partial block -- or, when that completes the block, fits the
// block -- at positions nobody reads yet; the last CTA commits every unit's
// lengths and v_max, or, if any token was non-finite, counts the rejection and
// commits nothing (same effect as k_check_finite + k_fill + k_tail).
__global__ void __launch_bounds__(128) k_append1(FillArgs a) {
  // a programmatic dependent of whatever ran before it on the stream (the step's
  // report kernel): its launch is staged early, its work waits for that to finish
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const ckv_cache& c = a.c;
  const int u = blockIdx.x, tid = threadIdx.x;
  const uint16_t kb = a.k_new[(size_t)u * D + tid], vb = a.v_new[(size_t)u * D + tid];
  const bool bad = ((kb & 0x7c00u) == 0x7c00u) | ((vb & 0x7c00u) == 0x7c00u);
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&c.status[CKV_ST_APPEND_BAD], 1);
  const int p = c.partial_len[u];
  if (p + 1 < B) {
    c.partial_k[((size_t)u * B + p) * D + tid] = kb;
    c.partial_v[((size_t)u * B + p) * D + tid] = vb;
  } else {
    fill_block(a, u, 0, false);
  }
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    last = atomicAdd(&c.status[CKV_ST_APPEND_CNT], 1) == (int)gridDim.x - 1;
    __threadfence();
  }
  __syncthreads();
  if (!last) return;
  const bool rejected = __ldcg(&c.status[CKV_ST_APPEND_BAD]) != 0;
  if (!rejected) {
    for (int v = tid; v < c.n_units; v += blockDim.x) {
      const int pv = __ldcg(&c.partial_len[v]);
      if (pv + 1 < B) {
        c.partial_len[v] = pv + 1;
      } else {
        const int nb = __ldcg(&c.n_blocks[v]);
        if (nb < c.max_blocks) {
          c.v_max[v] = fmaxf(__ldcg(&c.v_max[v]), __ldcg(&c.nu[(size_t)v * c.max_blocks + nb]));
          c.n_blocks[v] = nb + 1;
        }
        c.partial_len[v] = 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (rejected) c.status[CKV_ST_NONFINITE] += 1;
    c.status[CKV_ST_APPEND_BAD] = 0;
    c.status[CKV_ST_APPEND_CNT] = 0;
  }
}

__global__ void k_tail(FillArgs a) {
  const ckv_cache& c = a.c;
  const int u = blockIdx.x, tid = threadIdx.x;
  if (c.status[CKV_ST_APPEND_BAD]) {  // rejected: count it once, mutate nothing
    if (u == 0 && tid == 0) atomicAdd(&c.status[CKV_ST_NONFINITE], 1);
    return;
  }
  const int p = c.partial_len[u];
  const int total = p + a.n_tok;
  const int nf = total / B;
  const int rem = total - nf * B;
  const size_t ubase_new = (size_t)u * a.n_tok * D;
  const size_t ubase_par = (size_t)u * B * D;
  // leftover stream positions [nf*B, total): from new unless nf == 0
  for (int i = (nf == 0 ? p : 0); i < rem; ++i) {
    int gi = nf * B + i;  // position in the [partial | new] stream
    c.partial_k[ubase_par + i * D + tid] = a.k_new[ubase_new + (size_t)(gi - p) * D + tid];
    c.partial_v[ubase_par + i * D + tid] = a.v_new[ubase_new + (size_t)(gi - p) * D + tid];
  }
  __syncthreads();
  if (tid == 0) {
    int nb = c.n_blocks[u] + nf;
    c.n_blocks[u] = nb > c.max_blocks ? c.max_blocks : nb;
    c.partial_len[u] = rem;
  }
}

__global__ void k_read_tier1(ckv_cache c, int u, int b0, int8_t* kc, float* ks, float* ko,
                             uint8_t* vc, uint16_t* vs, uint16_t* vo) {
  const int i = blockIdx.x, tid = threadIdx.x;  // block b0+i, thread = channel
  const uint8_t* rec = c.tier1 + ((size_t)u * c.max_blocks + b0 + i) * REC;
  for (int t = 0; t < B; ++t) {
    kc[((size_t)i * B + t) * D + tid] = (int8_t)rec[kcode_offset(t, tid)];
    const uint32_t w = *reinterpret_cast<const uint32_t*>(rec + vcode_word(t, tid));
    vc[((size_t)i * B + t) * D + tid] = (uint8_t)((w >> vcode_bit(t, tid)) & 0xFu);
  }
  ks[(size_t)i * D + tid] = reinterpret_cast<const float*>(rec + OFF_KSCALE)[tid];
  ko[(size_t)i * D + tid] = reinterpret_cast<const float*>(rec + OFF_KOFF)[tid];
  {
    int t = tid >> 3, g = tid & 7;
    vs[((size_t)i * B + t) * NG + g] = reinterpret_cast<const uint16_t*>(rec + OFF_VSCALE)[vmeta_index(t, g)];
    vo[((size_t)i * B + t) * NG + g] = reinterpret_cast<const uint16_t*>(rec + OFF_VOFF)[vmeta_index(t, g)];
  }
}

// binary16 ingest of float64 inputs, rounded once (numpy astype(float16));
// casting through float32 first would double-round (cache.py:82-84).
__global__ void k_f64_to_f16(const double* x, uint16_t* y, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) y[i] = double_to_half_rn(x[i]);
}

__global__ void k_fault_offset(ckv_cache c, int u, int b, int ch, float shift) {
  float* off = reinterpret_cast<float*>(c.tier1 + ((size_t)u * c.max_blocks + b) * REC + OFF_KOFF);
  off[ch] = off[ch] + shift;
}

__global__ void k_tier2_drop(ckv_cache c, int u, int b) {
  c.tier2_valid[(size_t)u * c.max_blocks + b] = 0;
}

__global__ void k_reset(ckv_cache c) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < c.n_units) {
    c.n_blocks[i] = 0;
    c.partial_len[i] = 0;
    c.v_max[i] = 0.0f;
  }
  if (i < 8) c.status[i] = 0;
}

}  // namespace ckv

// ---------------------------------------------------------------------------
// launch wrappers used by capi.cu
namespace ckv {
thread_local int g_launches = 0;

cudaError_t launch_append(const ckv_cache* c, const uint16_t* k_new, const uint16_t* v_new,
                          int32_t n_tok, cudaStream_t s) {
  g_launches = 0;
  if (n_tok == 1) {  // the decode step's append: one launch
    FillArgs a{*c, k_new, v_new, 1};
    cudaError_t e = launch_k(true, k_append1, dim3(c->n_units), dim3(128), 0, s, a);
    ++g_launches;
    return e;
  }
  size_t n16 = (size_t)c->n_units * n_tok * D / 8;
  int grid = (int)((n16 + 255) / 256);
  if (grid > 4 * 148 * 8) grid = 4 * 148 * 8;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(c->status + CKV_ST_APPEND_BAD, 0, sizeof(int32_t), s);
  k_check_finite<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(k_new),
                                      reinterpret_cast<const uint4*>(v_new), n16, c->status);
  ++g_launches;
  FillArgs a{*c, k_new, v_new, n_tok};
  int nfill = (n_tok + B - 1) / B + 1;
  if (nfill > 0) {
    k_fill<<<dim3(nfill, c->n_units), 128, 0, s>>>(a);
    ++g_launches;
  }
  k_tail<<<c->n_units, 128, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_read_tier1(const ckv_cache* c, int u, int b0, int nb, int8_t* kc, float* ks,
                              float* ko, uint8_t* vc, uint16_t* vs, uint16_t* vo, cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  k_read_tier1<<<nb, 128, 0, s>>>(*c, u, b0, kc, ks, ko, vc, vs, vo);
  return cudaGetLastError();
}
cudaError_t launch_f64_to_f16(const double* x, uint16_t* y, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  size_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_f64_to_f16<<<(unsigned)g, 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}
cudaError_t launch_fault_offset(const ckv_cache* c, int u, int b, int ch, float shift,
                                cudaStream_t s) {
  k_fault_offset<<<1, 1, 0, s>>>(*c, u, b, ch, shift);
  return cudaGetLastError();
}
cudaError_t launch_tier2_drop(const ckv_cache* c, int u, int b, cudaStream_t s) {
  k_tier2_drop<<<1, 1, 0, s>>>(*c, u, b);
  return cudaGetLastError();
}
cudaError_t launch_reset(const ckv_cache* c, cudaStream_t s) {
  int n = c->n_units > 8 ? c->n_units : 8;
  k_reset<<<(n + 255) / 256, 256, 0, s>>>(*c);
  return cudaGetLastError();
}
}  // namespace ckv
