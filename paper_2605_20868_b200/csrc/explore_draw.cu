// Exploration draws on the device, exact to the reference's host generator.
//
// The reference samples, per q-head in head order, count = min(|tail|,
// round(rate * N_B)) positions of the ascending tail list with
// rng.choice(|tail|, count, replace=False) on the workload's numpy Philox
// generator (fallback.py:202-218, harness.py:262-269, 348).  |tail| = N_B - K'
// is only known after the selection, so drawing on the host costs a mid-step
// sync; here the device draws them from the generator's state, in the same
// stream order, and advances the state.
//
// numpy pieces restated (numpy 2.x, random/_generator.pyx choice() and
// src/distributions): Philox4x64-10 (Random123 constants), 64-bit outputs
// served from a 4-word buffer, uint32 draws taken low half first with the high
// half buffered (has_uint32), random_bounded_uint64(0, n) through Lemire's
// 32-bit multiply-shift with rejection, and choice(..., replace=False):
//   pop > 10000 and size > pop // 50: tail shuffle -- Fisher-Yates from pop-1
//       down to max(pop - size, 1) over arange(pop), the last `size` entries;
//   otherwise Floyd's algorithm over j in [pop - size, pop) (a repeat inserts
//       j), then a shuffle of the result (draws for i = size-1 .. 1).
// oracle/explore_rng.py is the Python model these are checked against.
//
// Parallel scheme: every bounded draw consumes one uint32 unless its bound is
// 0 (no draw) or Lemire rejects (one more per rejection, probability
// < bound / 2^32).  Heads get provisional offsets from the no-rejection counts;
// each warp resolves its heads' draws 32 at a time (a rejecting lane makes the
// rest of its chunk shift by one), records the rejections it met, and the
// grid iterates until every head's offset accounts for the rejections of the
// heads before it (cooperative launch, grid-wide syncs; normally one pass).
#include <cooperative_groups.h>

#include "step.cuh"

namespace cg = cooperative_groups;

namespace ckv {

namespace {

constexpr uint64_t PM0 = 0xD2E7470EE14C6C93ull, PM1 = 0xCA5A826395121157ull;
constexpr uint64_t PW0 = 0x9E3779B97F4A7C15ull, PW1 = 0xBB67AE8584CAA73Bull;
constexpr int XD_MAX_WARPS = 8;
constexpr int XD_ITERS = 32;  // iterations before the sequential pass takes over

__device__ __forceinline__ void philox4x64_10(const uint64_t ctr[4], const uint64_t key[2],
                                              uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = PM0 * c0, hi0 = __umul64hi(PM0, c0);
    const uint64_t lo1 = PM1 * c2, hi1 = __umul64hi(PM1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += PW0;
    k1 += PW1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// 256-bit counter + n
__device__ __forceinline__ void ctr_add(const uint64_t a[4], uint64_t n, uint64_t r[4]) {
  uint64_t carry = n;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t s = a[i] + carry;
    carry = (s < a[i]) ? 1ull : 0ull;
    r[i] = s;
  }
}

// generator state as numpy exposes it (bit_generator.state)
struct RngState {
  uint64_t ctr[4], key[2], buf[4];
  int64_t pos;    // buffer_pos
  int64_t has;    // has_uint32
  uint64_t uint;  // uinteger
};

__device__ __forceinline__ RngState load_state(const uint64_t* s) {
  RngState r;
#pragma unroll
  for (int i = 0; i < 4; ++i) r.ctr[i] = s[i];
  r.key[0] = s[4];
  r.key[1] = s[5];
#pragma unroll
  for (int i = 0; i < 4; ++i) r.buf[i] = s[6 + i];
  r.pos = (int64_t)s[10];
  r.has = (int64_t)s[11];
  r.uint = s[12];
  return r;
}

// 64-bit output m (0-based) after the state: the rest of the buffer, then
// Philox blocks of the incremented counter
__device__ __forceinline__ uint64_t out64(const RngState& S, uint64_t m) {
  const uint64_t left = (uint64_t)(4 - S.pos);
  if (m < left) return S.buf[S.pos + m];
  const uint64_t m2 = m - left;
  uint64_t c[4], o[4];
  ctr_add(S.ctr, m2 / 4 + 1, c);
  philox4x64_10(c, S.key, o);
  return o[m2 & 3];
}

// uint32 draw k (0-based) after the state
__device__ __forceinline__ uint32_t u32_at(const RngState& S, uint64_t k) {
  if (S.has) {
    if (k == 0) return (uint32_t)S.uint;
    k -= 1;
  }
  const uint64_t w = out64(S, k >> 1);
  return (k & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
}

// state after T uint32 draws
__device__ void advance(const RngState& S, uint64_t T, uint64_t* out) {
  RngState R = S;
  uint64_t k = T;
  if (S.has && k > 0) {
    R.has = 0;
    k -= 1;
  }
  if (k > 0) {
    const uint64_t F = (k + 1) / 2;  // 64-bit outputs fetched
    const uint64_t left = (uint64_t)(4 - S.pos);
    const uint64_t last = out64(S, F - 1);
    if (F <= left) {
      R.pos = S.pos + (int64_t)F;
    } else {
      const uint64_t m2 = F - left, n = (m2 + 3) / 4;
      ctr_add(S.ctr, n, R.ctr);
      uint64_t o[4];
      philox4x64_10(R.ctr, S.key, o);
#pragma unroll
      for (int i = 0; i < 4; ++i) R.buf[i] = o[i];
      R.pos = (int64_t)(m2 - 4 * (n - 1));
    }
    if (k & 1) {
      R.has = 1;
      R.uint = last >> 32;
    } else {  // numpy keeps the last fetched high half in `uinteger` after using it
      R.has = 0;
      R.uint = last >> 32;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) out[i] = R.ctr[i];
  out[4] = R.key[0];
  out[5] = R.key[1];
#pragma unroll
  for (int i = 0; i < 4; ++i) out[6 + i] = R.buf[i];
  out[10] = (uint64_t)R.pos;
  out[11] = (uint64_t)R.has;
  out[12] = R.uint;
}

struct Head {
  int pop, size, tail;  // tail: the tail-shuffle path
  int calls;            // bounded draws made (incl. bound-0 ones)
  long long base;       // uint32 draws without rejections
};

__device__ __forceinline__ Head head_of(const ckv_cache& c, const ckv_step& st, int item) {
  const int u = item / st.n_heads;
  const int nb = c.n_blocks[u];
  Head H{0, 0, 0, 0, 0};
  if (nb <= 0) return H;
  const int pop = nb - st.cert[item].k_star;
  const int want = (int)rint(st.explore_rate * (double)nb);  // Python round(): half to even
  const int size = min(pop, want);
  if (size <= 0) return H;
  H.pop = pop;
  H.size = size;
  H.tail = (pop > 10000 && size > pop / 50);
  if (H.tail) {
    const int first = max(pop - size, 1);
    H.calls = pop - first;
    H.base = H.calls;
  } else {
    H.calls = size + (size - 1);
    H.base = H.calls - ((pop - size == 0) ? 1 : 0);  // bounded(0) draws nothing
  }
  return H;
}

// the bound of call t of a head
__device__ __forceinline__ uint32_t bound_of(const Head& H, int t) {
  if (H.tail) return (uint32_t)(H.pop - 1 - t);
  if (t < H.size) return (uint32_t)(H.pop - H.size + t);
  return (uint32_t)(H.size - 1 - (t - H.size));  // shuffle: i = size-1 .. 1
}

// open-addressing map in shared memory: key -> value (keys >= 0, empty = -1)
__device__ __forceinline__ int map_find(const int2* tab, int cap, int key) {
  int i = (int)(((uint32_t)key * 2654435761u) & (uint32_t)(cap - 1));
  for (;;) {
    const int2 e = tab[i];
    if (e.x == key || e.x < 0) return i;
    i = (i + 1) & (cap - 1);
  }
}

// Resolve one head's draws from uint32 offset `off`; write its positions and
// return the number of rejections met.  Lane-parallel Lemire draws, lane-serial
// set / swap bookkeeping in the warp's map.
__device__ int draw_head(const RngState& S, const Head& H, long long off, int2* tab, int cap,
                         int32_t* pos_out, int lane) {
  for (int i = lane; i < cap; i += 32) tab[i] = make_int2(-1, -1);
  __syncwarp();
  int rej = 0, t0 = 0, nsel = 0;
  long long k = off;  // next uint32 index
  while (t0 < H.calls) {
    const int t = t0 + lane;
    const bool act = t < H.calls;
    const uint32_t bnd = act ? bound_of(H, t) : 0u;
    // uint32 index of this lane's draw if nothing before it in the chunk rejects;
    // a bound-0 call draws nothing (only call 0 of a Floyd head can have one)
    const bool draws = act && bnd != 0u;
    const unsigned dm = __ballot_sync(0xffffffffu, draws);
    const long long idx = k + __popc(dm & ((1u << lane) - 1u));
    uint32_t val = 0u;
    bool bad = false;
    if (draws) {
      const uint64_t ex = (uint64_t)bnd + 1ull;
      const uint64_t m = (uint64_t)u32_at(S, (uint64_t)idx) * ex;
      const uint32_t leftover = (uint32_t)m;
      if (leftover < ex) {
        const uint32_t thr = (uint32_t)((0xffffffffull - bnd) % ex);
        bad = leftover < thr;
      }
      val = (uint32_t)(m >> 32);
    }
    const unsigned bm = __ballot_sync(0xffffffffu, bad);
    const int L = bm ? __ffs(bm) - 1 : 32;  // lanes < L are resolved
    int nres = min(L, H.calls - t0);
    long long k_after = k + __popc(dm & ((L >= 32) ? 0xffffffffu : ((1u << L) - 1u)));
    uint32_t vL = 0u;
    if (L < 32) {  // lane L's draw rejects: redraw sequentially (every lane agrees)
      const uint32_t b = bound_of(H, t0 + L);
      const uint64_t ex = (uint64_t)b + 1ull;
      const uint32_t thr = (uint32_t)((0xffffffffull - b) % ex);
      long long kk = k_after + 1;  // the rejected draw was consumed
      uint64_t m;
      for (;;) {
        m = (uint64_t)u32_at(S, (uint64_t)kk) * ex;
        ++rej;
        ++kk;
        if ((uint32_t)m >= thr) break;
      }
      vL = (uint32_t)(m >> 32);
      k_after = kk;
      nres = L + 1;
    }
    // bookkeeping in call order (lane-serial; the map is shared by the warp); the
    // Floyd shuffle's draws only advance the stream
    const int nbook = H.tail ? nres : max(0, min(nres, H.size - t0));
    for (int l = 0; l < nbook; ++l) {
      const int tt = t0 + l;
      const uint32_t v = (l == L) ? vL : __shfl_sync(0xffffffffu, val, l);
      if (lane == 0) {
        if (H.tail) {  // swap(data[i], data[v]) with i = pop-1-tt over arange(pop)
          const int i = H.pop - 1 - tt, j = (int)v;
          const int si = map_find(tab, cap, i);
          const int vi = tab[si].x < 0 ? i : tab[si].y;
          const int sj = map_find(tab, cap, j);
          const int vj = tab[sj].x < 0 ? j : tab[sj].y;
          tab[si] = make_int2(i, vj);
          const int sj2 = map_find(tab, cap, j);
          tab[sj2] = make_int2(j, vi);
        } else if (tt < H.size) {  // Floyd: insert v, or j when v is already in
          const int j = H.pop - H.size + tt;
          const int s = map_find(tab, cap, (int)v);
          int ins = (int)v;
          if (tab[s].x >= 0) ins = j;
          const int s2 = map_find(tab, cap, ins);
          tab[s2] = make_int2(ins, 1);
          pos_out[nsel++] = ins;
        }
      }
      __syncwarp();
    }
    k = k_after;
    t0 += nres;
  }
  if (H.tail && lane == 0) {  // the chosen positions: data[pop-size .. pop)
    for (int p = H.pop - H.size; p < H.pop; ++p) {
      const int s = map_find(tab, cap, p);
      pos_out[nsel++] = tab[s].x < 0 ? p : tab[s].y;
    }
  }
  __syncwarp();
  return rej;
}

struct DrawArgs {
  ckv_cache c;
  ckv_step st;
  int32_t items;
  int32_t cap;  // map entries per warp (power of 2)
};

__global__ void __launch_bounds__(XD_MAX_WARPS * 32) k_explore_draw(DrawArgs a) {
  extern __shared__ __align__(16) int2 tabs[];
  cg::grid_group grid = cg::this_grid();
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_XDRAW);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  int2* tab = tabs + (size_t)wib * a.cap;
  const RngState S = load_state(st.explore_rng);
  // work words: rej[items], off_lo/hi[items] (int64 as two words), flags[XD_ITERS + 2]
  int32_t* rej = st.explore_work;
  long long* off = reinterpret_cast<long long*>(st.explore_work + ((a.items + 1) & ~1));
  int32_t* flags = reinterpret_cast<int32_t*>(off + a.items + 1);
  const int n = a.items;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rej[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < XD_ITERS + 2) flags[threadIdx.x] = 0;
  grid.sync();
  bool done = false;
  for (int it = 0; it < XD_ITERS && !done; ++it) {
    if (blockIdx.x == 0) {  // offsets = exclusive scan of base + rejections, head order
      __shared__ long long part[XD_MAX_WARPS * 32];
      const int per = (n + blockDim.x - 1) / blockDim.x;
      const int lo = threadIdx.x * per, hi = min(n, lo + per);
      long long s = 0;
      for (int i = lo; i < hi; ++i) s += head_of(c, st, i).base + __ldcg(rej + i);
      part[threadIdx.x] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        long long run = 0;
        for (int w = 0; w < (int)blockDim.x; ++w) {
          const long long x = part[w];
          part[w] = run;
          run += x;
        }
      }
      __syncthreads();
      long long run = part[threadIdx.x];
      for (int i = lo; i < hi; ++i) {
        off[i] = run;
        run += head_of(c, st, i).base + __ldcg(rej + i);
      }
      if (threadIdx.x == blockDim.x - 1) off[n] = run;  // every draw of the step
    }
    grid.sync();
    for (int i = gw; i < n; i += nwarps) {
      const Head H = head_of(c, st, i);
      if (lane == 0) st.explore_n[i] = H.size;
      if (H.size == 0) continue;
      const int r = draw_head(S, H, __ldcg(off + i), tab, a.cap,
                              st.explore_pos + (size_t)i * st.ecap, lane);
      if (lane == 0 && r != __ldcg(rej + i)) {
        rej[i] = r;
        atomicOr(&flags[it], 1);
      }
    }
    grid.sync();
    done = __ldcg(flags + it) == 0;
  }
  if (!done) {  // pathological rejection chains: one warp walks the heads in order
    if (blockIdx.x == 0 && wib == 0) {
      long long k = 0;
      for (int i = 0; i < n; ++i) {
        const Head H = head_of(c, st, i);
        if (H.size == 0) continue;
        const int r = draw_head(S, H, k, tab, a.cap, st.explore_pos + (size_t)i * st.ecap, lane);
        if (lane == 0) rej[i] = r;
        k += H.base + r;
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the generator's state after every draw
    long long T = __ldcg(off + n);
    if (!done) {  // the sequential pass fixed the rejections: recount
      T = 0;
      for (int i = 0; i < n; ++i) T += head_of(c, st, i).base + __ldcg(rej + i);
    }
    uint64_t o[13];
    advance(S, (uint64_t)T, o);
    for (int i = 0; i < 13; ++i) st.explore_rng[i] = o[i];
  }
}

}  // namespace

cudaError_t launch_explore_draw(const ckv_cache* c, const ckv_step* st, cudaStream_t s) {
  const int items = c->n_units * st->n_heads;
  int cap = 64;
  while (cap < 4 * st->ecap) cap <<= 1;  // Floyd set / tail-shuffle map, load <= 1/2
  // warps per CTA so that their maps fit in 160 KB of shared memory
  const int wpb = max(1, min(XD_MAX_WARPS, (int)((160 * 1024) / ((size_t)cap * sizeof(int2)))));
  const size_t smem = (size_t)wpb * cap * sizeof(int2);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_max_dyn_smem(k_explore_draw, (int)smem);
  if (e != cudaSuccess) return e;
  DevState& ds = dev_state();
  int per = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_explore_draw, wpb * 32, smem);
  if (e != cudaSuccess) return e;
  if (per < 1) return cudaErrorInvalidConfiguration;
  const int grid = max(1, min(ds.sms * per, (items + wpb - 1) / wpb));
  DrawArgs a{*c, *st, items, cap};
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel((void*)k_explore_draw, dim3(grid), dim3(wpb * 32), args, smem, s);
  ++g_launches;
  return e;
}

}  // namespace ckv
