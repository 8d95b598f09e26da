// LRU scratch accounting for promoted originals, exact to ScratchCache.request
// (cache.py:243-312): per unit and per payload kind, the q-heads' requests are
// processed in head order, each request list ascending; a hit moves the block
// to MRU, a miss admits it at MRU and evicts the LRU entry past capacity; a
// zero-capacity scratch serves but keeps nothing.
//
// State per (unit, kind), int32 words:  [0] T clock, [1] P oldest stamp,
// [2] count, [3] R ring size (0 = capacity covers every block, no eviction
// possible), [4 .. 4+max_blocks) stamp[b] (0 = absent), then ring[R] holding
// the block id last stamped with s at ring[s & (R-1)].  Recency order is stamp
// order; a ring slot is live iff stamp[ring[s]] == s, so a hit simply leaves a
// stale slot behind.  Batches that cannot evict run fully parallel; batches
// that must evict walk the ring from P sequentially (one thread, shared
// memory), which is only reached when the scratch is smaller than the working
// set -- the regime where the Tier-2 transfer dominates anyway.
#include "common.cuh"

namespace ckv {

constexpr int LRU_THREADS = 256;

__device__ __forceinline__ int blk_scan_excl(int v, int* ws, int* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < LRU_THREADS / 32) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < LRU_THREADS / 32) ws[lane] = w;
    if (lane == LRU_THREADS / 32 - 1) *tot = w;
  }
  __syncthreads();
  int r = ((warp > 0) ? ws[warp - 1] : 0) + x - v;
  __syncthreads();
  return r;
}

struct LruArgs {
  ckv_cache c;
  ckv_step st;
  int32_t* state;
  int32_t words;
  int32_t cap;
  int32_t kind;  // 0 keys, 1 values
  int64_t* counters;
};

__global__ void __launch_bounds__(LRU_THREADS) k_lru(LruArgs a) {
  extern __shared__ __align__(16) int32_t sm[];
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  const int u = blockIdx.x, tid = threadIdx.x;
  const int maxb = c.max_blocks;
  const int nb = c.n_blocks[u];
  int32_t* L = a.state + (size_t)u * a.words;
  __shared__ int hdr[4];
  __shared__ int ws[32];
  __shared__ int misc[8];
  if (tid < 4) hdr[tid] = L[tid];
  __syncthreads();
  const int R = hdr[3];
  const int M = R - 1;
  int32_t* stamp = sm;               // [maxb]
  int32_t* ring = sm + maxb;         // [R]
  int32_t* req = ring + R;           // [maxb + 1024] request list
  int32_t* tmp = req + maxb + 1024;  // [maxb] compaction buffer
  uint32_t* bits = reinterpret_cast<uint32_t*>(tmp + maxb);  // [maxb/32]
  for (int i = tid; i < maxb; i += LRU_THREADS) stamp[i] = (i < nb) ? L[4 + i] : 0;
  for (int i = tid; i < R; i += LRU_THREADS) ring[i] = L[4 + maxb + i];
  __syncthreads();
  int T = hdr[0], P = hdr[1], count = hdr[2];
  const int cap = a.cap;
  long long hits = 0, misses = 0;

  for (int h = 0; h < st.n_heads; ++h) {
    const size_t hu = (size_t)u * st.n_heads + h;
    int n;
    // ---- build the ascending request list ---------------------------------
    if (a.kind == 1) {
      n = st.cert[hu].n_value_promoted;
      const int32_t* vl = st.vlist + hu * maxb;
      for (int i = tid; i < n; i += LRU_THREADS) req[i] = vl[i];
    } else {
      const int kp = st.cert[hu].k_star;
      for (int i = tid; i < (nb + 31) / 32; i += LRU_THREADS) bits[i] = 0u;
      __syncthreads();
      const int32_t* ord = st.order + hu * st.kcap;
      for (int i = tid; i < kp; i += LRU_THREADS) atomicOr(&bits[ord[i] >> 5], 1u << (ord[i] & 31));
      __syncthreads();
      const int per = (nb + LRU_THREADS - 1) / LRU_THREADS;
      const int lo = tid * per, hi = min(nb, lo + per);
      int cnt = 0;
      for (int b = lo; b < hi; ++b) cnt += (bits[b >> 5] >> (b & 31)) & 1u;
      int off = blk_scan_excl(cnt, ws, &misc[0]);
      for (int b = lo; b < hi; ++b)
        if ((bits[b >> 5] >> (b & 31)) & 1u) req[off++] = b;
      n = kp;
    }
    __syncthreads();
    if (n == 0) continue;
    // ---- keep T - P + n within the ring (compaction) ------------------------
    if (R > 0 && T + n - P > R) {
      const int span = T - P;
      const int per = (span + LRU_THREADS - 1) / LRU_THREADS;
      const int lo = tid * per, hi = min(span, lo + per);
      int cnt = 0;
      for (int k = lo; k < hi; ++k) {
        const int s = P + k, b = ring[s & M];
        cnt += (b >= 0 && stamp[b] == s);
      }
      int off = blk_scan_excl(cnt, ws, &misc[1]);
      for (int k = lo; k < hi; ++k) {
        const int s = P + k, b = ring[s & M];
        if (b >= 0 && stamp[b] == s) tmp[off++] = b;
      }
      __syncthreads();
      const int live = misc[1];
      for (int i = tid; i < R; i += LRU_THREADS) ring[i] = -1;
      __syncthreads();
      for (int i = tid; i < live; i += LRU_THREADS) {
        stamp[tmp[i]] = 1 + i;
        ring[(1 + i) & M] = tmp[i];
      }
      __syncthreads();
      P = 1;
      T = 1 + live;
    }
    // ---- count misses -----------------------------------------------------------
    int m = 0;
    for (int i = tid; i < n; i += LRU_THREADS) m += (stamp[req[i]] == 0);
    int dummy = blk_scan_excl(m, ws, &misc[2]);
    (void)dummy;
    const int nm = misc[2];
    if (cap > 0 && (R == 0 || count + nm <= cap)) {
      for (int i = tid; i < n; i += LRU_THREADS) {
        const int b = req[i];
        stamp[b] = T + i;
        if (R > 0) ring[(T + i) & M] = b;
      }
      T += n;
      count += nm;
      hits += n - nm;
      misses += nm;
    } else if (cap == 0) {
      misses += n;  // served, nothing retained
    } else {
      if (tid == 0) {
        long long hh = 0, mm = 0;
        for (int i = 0; i < n; ++i) {
          const int b = req[i];
          if (stamp[b] > 0) {
            ++hh;
          } else {
            ++mm;
            if (count == cap) {
              for (;;) {
                const int v = ring[P & M];
                if (v >= 0 && stamp[v] == P) {
                  stamp[v] = 0;
                  ++P;
                  break;
                }
                ++P;
              }
              --count;
            }
            ++count;
          }
          stamp[b] = T;
          ring[T & M] = b;
          ++T;
        }
        misc[3] = (int)hh;
        misc[4] = (int)mm;
        misc[5] = T;
        misc[6] = P;
        misc[7] = count;
      }
      __syncthreads();
      hits += misc[3];
      misses += misc[4];
      T = misc[5];
      P = misc[6];
      count = misc[7];
    }
    __syncthreads();
  }
  // ---- write back ---------------------------------------------------------------
  for (int i = tid; i < nb; i += LRU_THREADS) L[4 + i] = stamp[i];
  for (int i = tid; i < R; i += LRU_THREADS) L[4 + maxb + i] = ring[i];
  if (tid == 0) {
    L[0] = T;
    L[1] = P;
    L[2] = count;
    st.page_stats[u * 4 + 2 * a.kind + 0] = (int32_t)hits;
    st.page_stats[u * 4 + 2 * a.kind + 1] = (int32_t)misses;
    int64_t* ctr = a.counters + (size_t)u * 6 + 3 * a.kind;
    ctr[0] += hits;
    ctr[1] += misses;
    ctr[2] += misses * (long long)(B * D * 2);
  }
}

__global__ void k_lru_init(int32_t* state, int words, int maxb, int R, int n_units) {
  const int u = blockIdx.x;
  int32_t* L = state + (size_t)u * words;
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    int v;
    if (i == 0 || i == 1) v = 1;
    else if (i == 2) v = 0;
    else if (i == 3) v = R;
    else if (i < 4 + maxb) v = 0;
    else v = -1;
    L[i] = v;
  }
  (void)n_units;
}

int lru_ring(int max_blocks, int cap) {
  if (cap >= max_blocks) return 0;
  int need = 2 * cap + max_blocks + 1024;
  int R = 1;
  while (R < need) R <<= 1;
  return R;
}

cudaError_t launch_scratch(const ckv_cache* c, const ckv_step* st, const ckv_scratch* sc,
                           cudaStream_t s) {
  extern int g_launches;
  for (int kind = 0; kind < 2; ++kind) {
    const int cap = kind ? sc->value_capacity : sc->key_capacity;
    const int R = lru_ring(c->max_blocks, cap);
    const int words = 4 + c->max_blocks + R;
    LruArgs a{*c, *st, kind ? sc->value_lru : sc->key_lru, words, cap, kind, sc->counters};
    const size_t smem =
        (size_t)(c->max_blocks + R + c->max_blocks + 1024 + c->max_blocks + (c->max_blocks + 31) / 32 + 4) * 4;
    cudaFuncSetAttribute(k_lru, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_lru<<<c->n_units, LRU_THREADS, smem, s>>>(a);
    ++g_launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_lru_init(int32_t* state, int n_units, int max_blocks, int cap, cudaStream_t s) {
  const int R = lru_ring(max_blocks, cap);
  const int words = 4 + max_blocks + R;
  k_lru_init<<<n_units, 256, 0, s>>>(state, words, max_blocks, R, n_units);
  return cudaGetLastError();
}

}  // namespace ckv
