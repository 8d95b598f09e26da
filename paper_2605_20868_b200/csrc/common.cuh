// Shared device helpers and the Tier-1 block record layout.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "certkv_b200.h"

namespace ckv {

constexpr int D = CKV_HEAD_DIM;     // 128
constexpr int B = CKV_BLOCK;        // 16
constexpr int G = CKV_GROUP;        // 16
constexpr int NG = D / G;           // 8 value groups
constexpr int H = CKV_MAX_QHEADS;   // 4
constexpr int REC = CKV_BLOCK_BYTES;

// Tier-1 block record (4608 B, one contiguous bulk copy):
//   [   0, 2048) key codes int8, mma.m16n8k32 A-fragment order:
//                for k-tile kt (32 channels) and lane l: 16 bytes =
//                {row l/4 cols 4(l%4)+0..3, row l/4+8 same cols,
//                 row l/4 cols 16+4(l%4)+0..3, row l/4+8 same cols}
//   [2048, 2560) key scale  f32[128]
//   [2560, 3072) key offset f32[128]
//   [3072, 4096) value codes, mma.m16n8k16 A-fragment order of V^T per value
//                group g (rows = the group's 16 channels, k = the 16 tokens):
//                word [g/4][lane l][g%4] (u32) holds the 8 nibbles lane l
//                feeds for group g: channel 16g + l/4 (+8 for bits 8-15 /
//                24-31), tokens 2(l%4) (+1 in the upper half-word, +8 for
//                bits 4-7 / 20-23).  (w & 0x000f000f) is then a half2 of two
//                codes, (w & 0x00f000f0) one of codes x 16, shifted by 8 the
//                same for the upper channel.
//   [4096, 4352) value scale  fp16 [j][g][i]  (j = (t%8)/2, i = t%2 + 2(t/8))
//   [4352, 4608) value offset fp16 [j][g][i]  so lane l reads the (t, t+1),
//                (t+8, t+9) pairs of its k-columns with one 8-byte load
constexpr int OFF_KCODES = 0;
constexpr int OFF_KSCALE = 2048;
constexpr int OFF_KOFF = 2560;
constexpr int OFF_VCODES = 3072;
constexpr int OFF_VSCALE = 4096;
constexpr int OFF_VOFF = 4352;

__host__ __device__ inline int kcode_offset(int t, int c) {
  int kt = c >> 5, cc = c & 31;
  int lane = (t & 7) * 4 + ((cc & 15) >> 2);
  int reg = (t >> 3) + 2 * (cc >> 4);
  return OFF_KCODES + kt * 512 + lane * 16 + reg * 4 + (cc & 3);
}
// byte offset of the u32 word holding the nibble of value code (t, c), and its bit
__host__ __device__ inline int vcode_word(int t, int c) {
  int g = c >> 4, r = c & 15;
  int lane = (r & 7) * 4 + ((t & 7) >> 1);
  return OFF_VCODES + (g >> 2) * 512 + lane * 16 + (g & 3) * 4;
}
__host__ __device__ inline int vcode_bit(int t, int c) {
  return 16 * (t & 1) + 4 * (t >> 3) + 8 * ((c & 15) >> 3);
}
__host__ __device__ inline int vmeta_index(int t, int g) {  // half index within scale / offset
  return ((((t & 7) >> 1) * 8 + g) * 4) + (t & 1) + 2 * (t >> 3);
}

// Tier-2 keys are stored per 16-token block in mma.m16n8k16 (fp16) A-fragment
// order, so the original-key scores of a block are 8 tensor-core MMAs fed by
// one coalesced 16-byte load per lane per k-tile: element (t, c) of a block
// sits at half index  kt*256 + lane*8 + reg*2 + (cc&1)  with kt = c/16,
// cc = c%16, lane = (t%8)*4 + (cc%8)/2, reg = t/8 + 2*(cc/8).
__host__ __device__ inline int k2_offset(int t, int c) {
  int kt = c >> 4, cc = c & 15;
  int lane = (t & 7) * 4 + ((cc & 7) >> 1);
  int reg = (t >> 3) + 2 * (cc >> 3);
  return kt * 256 + lane * 8 + reg * 2 + (cc & 1);
}
// Tier-2 values likewise, as the A operand of V^T (rows = channels of group
// g = c/16, k = tokens): P.V of a block is 8 MMAs with one 16-byte load per
// lane per group.  Half index g*256 + lane*8 + reg*2 + (t&1), lane =
// (r%8)*4 + (t%8)/2, reg = r/8 + 2*(t/8), r = c%16.
__host__ __device__ inline int v2_offset(int t, int c) {
  int g = c >> 4, r = c & 15;
  int lane = (r & 7) * 4 + ((t & 7) >> 1);
  int reg = (r >> 3) + 2 * (t >> 3);
  return g * 256 + lane * 8 + reg * 2 + (t & 1);
}

// ---- host-side runtime state (capi.cu) ----------------------------------------
// Function attributes, occupancy-derived grid sizes and auxiliary streams are
// per device (one process may drive several GPUs); the A/B environment knobs are
// read once per process.
struct Knobs {
  bool separate_lru;     // CKV_SEPARATE_LRU: k_lru_fast instead of the LRU fused into pass B
  bool separate_pagein;  // CKV_SEPARATE_PAGEIN: gather kernel on a side stream before pass B
  int chunks;            // CKV_CHUNKS: unit-chunked overlap of the tail with pass A
  int sel_kpt, sel_nt;   // CKV_SEL=kpt:nt forces a k_select variant (A/B runs)
  int pb_chunks;         // CKV_PB_CHUNKS forces the pass-B chunks per unit (A/B runs)
  int dn_splits;         // CKV_DN_SPLITS forces the dense splits per unit (A/B runs)
};
const Knobs& knobs();
// host_report layout (ckv_report_layout): cert | status[8] | page_stats | explore_n
inline void report_layout(int n_units, int n_heads, int64_t* out) {
  auto up = [](int64_t x) { return (x + 15) & ~(int64_t)15; };
  const int64_t cert = up((int64_t)n_units * n_heads * (int64_t)sizeof(ckv_cert));
  const int64_t status = cert, ps = up(status + 8 * 4), en = up(ps + (int64_t)n_units * 16);
  out[0] = up(en + (int64_t)n_units * n_heads * 4);
  out[1] = status;
  out[2] = ps;
  out[3] = en;
}
struct DevState {
  int sms = 0;
  int dense_slots = 0;
  int passb_slots = 0;
  cudaStream_t tail = nullptr;  // high priority
  cudaStream_t side = nullptr;  // page-in
  int n_attr = 0;
  const void* attr_fn[32] = {};
  int attr_bytes[32] = {};
};
DevState& dev_state();  // of the current device
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the current device
// (set once per device and size)
cudaError_t set_max_dyn_smem_fn(const void* fn, int bytes);
template <class F>
inline cudaError_t set_max_dyn_smem(F* fn, int bytes) {
  return set_max_dyn_smem_fn(reinterpret_cast<const void*>(fn), bytes);
}
constexpr size_t kLruSmemMax = 227 * 1024;
// kernel launch, optionally as a programmatic dependent launch of the previous
// kernel in the stream (see the dataflow helpers below)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

extern thread_local int g_launches;  // kernels launched by the last C-ABI call of this thread

// LRU ring size for a scratch of `cap` blocks (0 = no eviction possible); see scratch.cu
__host__ __device__ inline int lru_ring(int max_blocks, int cap) {
  if (cap >= max_blocks) return 0;
  int need = 2 * cap + max_blocks + 1024;
  int R = 1;
  while (R < need) R <<= 1;
  return R;
}
// words of an evicting k_lru's work arrays (request list, compaction buffer,
// bitmap) kept behind the state for units too large for shared memory
__host__ __device__ inline int lru_work_words(int max_blocks) {
  return 2 * max_blocks + 1024 + (max_blocks + 31) / 32 + 4;
}
__host__ __device__ inline int lru_words(int max_blocks, int cap) {
  const int R = lru_ring(max_blocks, cap);
  return 4 + 3 * max_blocks + R + (R ? lru_work_words(max_blocks) : 0);
}
// per-block epoch of the step that missed it into its slot (the slot is filled by
// that step's pass B, or by k_pagein); = slot table + max_blocks
__host__ __device__ inline int lru_fresh_offset(int max_blocks, int cap) {
  return 4 + 2 * max_blocks + lru_ring(max_blocks, cap);
}
// slot table (HBM slot of each resident block, -1 otherwise) inside an LRU state
__host__ __device__ inline int lru_slot_offset(int max_blocks, int cap) {
  return 4 + max_blocks + lru_ring(max_blocks, cap);
}

// ---- bit helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// Correctly rounded float64 -> binary16 (round to nearest even), matching
// numpy's astype(float16) from float64 (no double rounding through fp32).
__device__ inline uint16_t double_to_half_rn(double x) {
  uint16_t sign = signbit(x) ? 0x8000 : 0;
  double a = fabs(x);
  if (isnan(a)) return 0x7e00;
  if (a >= 65520.0) return sign | 0x7c00;  // rounds to inf
  if (a < 6.103515625e-05) {                // subnormal range: units of 2^-24
    double q = rint(a * 16777216.0);        // exact scaling by a power of two
    return sign | (uint16_t)q;              // q <= 1024 -> 1024 is the min normal
  }
  int e;
  double m = frexp(a, &e);                  // a = m * 2^e, m in [0.5, 1)
  double q = rint(ldexp(m, 11));            // 11 significant bits
  if (q >= 2048.0) { q *= 0.5; e += 1; }
  if (e - 1 + 15 >= 31) return sign | 0x7c00;
  uint16_t exp_bits = (uint16_t)(e - 1 + 15);
  uint16_t man = (uint16_t)((int)q - 1024);
  return sign | (uint16_t)(exp_bits << 10) | man;
}

__device__ __forceinline__ double half_bits_to_double(uint16_t h) {
  return (double)__half2float(__ushort_as_half(h));
}

// ---- warp reductions ----------------------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- mbarrier + bulk async copy (TMA 1-D) -------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// shared -> global bulk copy (bulk async-group); wait_read: the source may be refilled
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, "
      "p;\n}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---- kernel dataflow within a step (programmatic dependent launch) ----------
// pass A -> selection -> pass B -> combine run as a chain of PDL launches: each
// kernel lets its dependent launch as its own last CTAs start, and a consumer
// CTA waits for its unit's producer epoch instead of the whole producer grid,
// so the next kernel's work on finished units overlaps the producer's last wave.
// ckv_step.flow: [6][n_units] = pass-A count, pass-A done, selection done,
// pass-B count, pass-B done, combine count (epochs; counts reset themselves),
// then FLOW_STEP_WORDS step-wide words.
enum { FLOW_PA_CNT = 0, FLOW_PA_DONE = 1, FLOW_SEL_DONE = 2, FLOW_PB_CNT = 3, FLOW_PB_DONE = 4,
       FLOW_CB_UNIT = 5, FLOW_UNIT_WORDS = 6 };
// step-wide words behind the per-unit ones: combine CTAs done, step resolved,
// dense units listed so far, some head requested Rung 4
enum { FLOW_CB_CNT = 0, FLOW_RESOLVED = 1, FLOW_DENSE_N = 2, FLOW_ANY4 = 3, FLOW_STEP_WORDS = 4 };
__host__ __device__ inline int32_t* flow_step(int32_t* flow, int n_units, int k) {
  return flow + FLOW_UNIT_WORDS * n_units + k;
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
// every thread of the CTA returns once *flag == epoch, with acquire semantics; a
// producer that never publishes (a launch-shape bug) traps after 2 s instead of
// hanging the GPU
__device__ __forceinline__ void flow_wait(const int32_t* flag, int epoch) {
  if (threadIdx.x == 0) {
    int ns = 64;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_gpu(flag) != epoch) {
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
      if (globaltimer_ns() - t0 > 2000000000ull) __trap();
    }
  }
  __syncthreads();
  (void)ld_acquire_gpu(flag);
}
// the CTA's writes are done: count it; the last of `total` CTAs publishes epoch
__device__ __forceinline__ void flow_arrive(int32_t* cnt, int32_t* done, int total, int epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(cnt, 1) == total - 1) {
      *cnt = 0;
      __threadfence();
      st_release_gpu(done, epoch);
    }
  }
}

// per-kernel first-start / last-end stamps (ckv_step.trace, profiling only)
struct TraceScope {
  unsigned long long* slot;
  __device__ __forceinline__ TraceScope(unsigned long long* tr, int id)
      : slot(tr ? tr + 2 * id : nullptr) {
    if (slot && threadIdx.x == 0) atomicMin(slot, globaltimer_ns());
  }
  __device__ __forceinline__ ~TraceScope() {
    if (slot && threadIdx.x == 0) atomicMax(slot + 1, globaltimer_ns());
  }
};

// L2 prefetch of a global range by the TMA unit (no registers, no shared memory)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const char* c = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15);
  const char* e = reinterpret_cast<const char*>(p) + bytes;
  while (c < e) {
    const uint32_t n = (uint32_t)min((long long)(e - c + 15) & ~15ll, 16384ll);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(n) : "memory");
    c += n;
  }
}

// ---- cp.async (LDGSTS) ------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- integer MMA: D(16x8,s32) += A(16x32,s8) * B(32x8,u8) ---------------------
__device__ __forceinline__ void mma_s8u8(int (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// fp16 MMA: D(16x8,f32) += A(16x16,f16) * B(16x8,f16)
__device__ __forceinline__ void mma_f16(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_f16r(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ---- half2 arithmetic on raw 32-bit registers ------------------------------------
__device__ __forceinline__ uint32_t h2_mul(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t h2_fma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t h2_sub(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// pack two floats (lo -> low half) to fp16x2, round to nearest even
__device__ __forceinline__ uint32_t f2_to_h2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// hi/lo fp16 split of a float pair: x ~= hi + lo to ~22 significant bits
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = f2_to_h2(x0, x1);
  const __half2 h = *reinterpret_cast<const __half2*>(&hi);
  lo = f2_to_h2(x0 - __low2float(h), x1 - __high2float(h));
}

// exp via the MUFU ex2 unit (flush-to-zero, rel. error ~2^-22) with a pre-scaled argument
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_exp(float x) { return ex2_approx(x * 1.4426950408889634f); }

}  // namespace ckv
