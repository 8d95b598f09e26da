// LRU scratch for promoted originals, exact to ScratchCache.request
// (cache.py:243-312): per unit and per payload kind, the q-heads' requests are
// processed in head order, each request list ascending; a hit moves the block
// to MRU, a miss admits it at MRU and evicts the LRU entry past capacity; a
// zero-capacity scratch serves but keeps nothing.
//
// State per (unit, kind), int32 words:  [0] T clock, [1] P oldest stamp,
// [2] count, [3] R ring size (0 = capacity covers every block, no eviction
// possible), then stamp[max_blocks] (0 = absent), ring[R] (block id last
// stamped with s at ring[s & (R-1)]), slot[max_blocks] (HBM slot of a resident
// block, -1 otherwise).  Recency order is stamp order; a ring slot is live iff
// stamp[ring[s]] == s, so a hit simply leaves a stale entry behind.  Batches
// that cannot evict run fully parallel (misses take slots count, count+1, ...);
// batches that must evict walk the ring from P sequentially (one thread,
// shared memory) and hand the victim's slot to the new block -- only reached
// when the scratch is smaller than the working set, the regime where the
// Tier-2 transfer dominates anyway.
//
// k_pagein then copies every block missed this step that is still resident
// from Tier-2 (pinned host RAM, read zero-copy over PCIe) into its slot; it
// runs on a side stream joined by an event before pass B.
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
  int32_t* miss_list;  // [U][2][miss_cap]
  int32_t* miss_n;     // [U][2]
  int32_t miss_cap;
  int32_t u0;
  int32_t gmem;  // 1: state too large for shared memory, work on it in global memory
};

__global__ void __launch_bounds__(LRU_THREADS) k_lru(LruArgs a) {
  extern __shared__ __align__(16) int32_t sm[];
  const ckv_cache& c = a.c;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_LRU);
  const int u = a.u0 + blockIdx.x, tid = threadIdx.x;
  const int maxb = c.max_blocks;
  const int nb = c.n_blocks[u];
  int32_t* L = a.state + (size_t)u * a.words;
  __shared__ int hdr[4];
  __shared__ int ws[32];
  __shared__ int misc[8];
  __shared__ int nmiss;
  if (tid < 4) hdr[tid] = L[tid];
  if (tid == 0) nmiss = 0;
  __syncthreads();
  const int R = hdr[3];
  const int M = R - 1;
  // the state (stamp, ring, slot) and the work arrays live in shared memory when
  // they fit (a.gmem == 0); otherwise the kernel works on the global state in
  // place, with the work arrays behind it (lru_work_words)
  int32_t *stamp, *ring, *slot, *req, *tmp;
  if (!a.gmem) {
    stamp = sm;               // [maxb]
    ring = sm + maxb;         // [R]
    slot = ring + R;          // [maxb]
    req = slot + maxb;        // [maxb + 1024] request list
  } else {
    stamp = L + 4;
    ring = L + 4 + maxb;
    slot = ring + R;
    req = L + lru_fresh_offset(maxb, a.cap) + maxb;
  }
  tmp = req + maxb + 1024;  // [maxb] compaction buffer
  uint32_t* bits = reinterpret_cast<uint32_t*>(tmp + maxb);  // [maxb/32]
  if (!a.gmem) {
    const int32_t* Lslot = L + 4 + maxb + R;
    for (int i = tid; i < maxb; i += LRU_THREADS) {
      stamp[i] = (i < nb) ? L[4 + i] : 0;
      slot[i] = (i < nb) ? Lslot[i] : -1;
    }
    for (int i = tid; i < R; i += LRU_THREADS) ring[i] = L[4 + maxb + i];
  }
  __syncthreads();
  int T = hdr[0], P = hdr[1], count = hdr[2];
  const int cap = a.cap;
  long long hits = 0, misses = 0;
  int32_t* mlist = a.miss_list ? a.miss_list + ((size_t)u * 2 + a.kind) * a.miss_cap : nullptr;
  int32_t* fresh_g = L + lru_fresh_offset(maxb, cap);

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
    // ---- count misses (contiguous chunks so ranks follow request order) -------
    const int per = (n + LRU_THREADS - 1) / LRU_THREADS;
    const int lo = tid * per, hi = min(n, lo + per);
    int m = 0;
    for (int i = lo; i < hi; ++i) m += (stamp[req[i]] == 0);
    const int mrank = blk_scan_excl(m, ws, &misc[2]);
    const int nm = misc[2];
    if (cap > 0 && (R == 0 || count + nm <= cap)) {
      int r = mrank;
      for (int i = lo; i < hi; ++i) {
        const int b = req[i];
        if (stamp[b] == 0) {
          slot[b] = count + r;
          fresh_g[b] = st.epoch;
          if (mlist) {
            const int k = atomicAdd(&nmiss, 1);
            if (k < a.miss_cap) mlist[k] = b;
          }
          ++r;
        }
        stamp[b] = T + i;
        if (R > 0) ring[(T + i) & M] = b;
      }
      __syncthreads();
      T += n;
      count += nm;
      hits += n - nm;
      misses += nm;
    } else if (cap == 0) {
      misses += n;  // served straight from Tier-2, nothing retained
    } else {
      if (tid == 0) {
        long long hh = 0, mm = 0;
        for (int i = 0; i < n; ++i) {
          const int b = req[i];
          if (stamp[b] > 0) {
            ++hh;
          } else {
            ++mm;
            int s;
            if (count == cap) {
              for (;;) {
                const int v = ring[P & M];
                if (v >= 0 && stamp[v] == P) {
                  stamp[v] = 0;
                  s = slot[v];
                  slot[v] = -1;
                  ++P;
                  break;
                }
                ++P;
              }
            } else {
              s = count++;
            }
            slot[b] = s;
            fresh_g[b] = st.epoch;
            if (mlist && nmiss < a.miss_cap) mlist[nmiss++] = b;
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
  if (!a.gmem) {
    int32_t* Ls = L + 4 + maxb + R;
    for (int i = tid; i < nb; i += LRU_THREADS) {
      L[4 + i] = stamp[i];
      Ls[i] = slot[i];
    }
    for (int i = tid; i < R; i += LRU_THREADS) L[4 + maxb + i] = ring[i];
  }
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
    if (a.miss_n) a.miss_n[u * 2 + a.kind] = min(nmiss, a.miss_cap);
  }
}

// Scratch that holds every block (capacity >= max_blocks, ring size 0): no
// eviction can happen, so ScratchCache.request reduces to "the first request of
// a block that is not resident is a miss, every other request a hit" -- per
// block of the step's union work list (k_union: ascending, with the mask of
// requesting heads), one thread per item; misses get the next free slots in
// block order.  Same counters, page stats, stamps and miss list as k_lru.
__global__ void __launch_bounds__(LRU_THREADS) k_lru_fast(LruArgs ka, LruArgs va) {
  const int kind = blockIdx.y;
  const LruArgs& a = kind ? va : ka;
  const ckv_step& st = a.st;
  TraceScope trace_(st.trace, CKV_TR_LRU);
  const int u = a.u0 + blockIdx.x, tid = threadIdx.x;
  const int maxb = a.c.max_blocks;
  int32_t* L = a.state + (size_t)u * a.words;
  int32_t* stamp = L + 4;
  int32_t* slot = L + 4 + maxb;  // R == 0
  int32_t* fresh = L + 4 + 2 * maxb;  // lru_fresh_offset with R == 0
  const int nwork = st.n_work[u];
  const int32_t* work = st.work + (size_t)u * st.wcap;
  __shared__ int ws[32];
  __shared__ int misc[4];
  const int T0 = L[0], count0 = L[2];
  int32_t* mlist = a.miss_list ? a.miss_list + ((size_t)u * 2 + kind) * a.miss_cap : nullptr;
  long long hits = 0, misses = 0;
  int base_m = 0, base_req = 0;
  for (int i0 = 0; i0 < nwork; i0 += LRU_THREADS) {
    const int i = i0 + tid;
    int nreq = 0, miss = 0, b = 0;
    if (i < nwork) {
      const uint32_t e = (uint32_t)work[i];
      b = (int)(e & 0xffffffu);
      nreq = __popc((e >> (kind ? 28 : 24)) & 0xfu);
      if (nreq) miss = (stamp[b] == 0);
    }
    const int rank = blk_scan_excl(miss, ws, &misc[0]);
    const int nm = misc[0];
    const int roff = blk_scan_excl(nreq, ws, &misc[1]);
    const int nr = misc[1];
    if (nreq) {
      if (a.cap > 0) {
        if (miss) {
          slot[b] = count0 + base_m + rank;
          fresh[b] = st.epoch;
          if (mlist && base_m + rank < a.miss_cap) mlist[base_m + rank] = b;
        }
        stamp[b] = T0 + base_req + roff + nreq - 1;  // stamp of its last request
      }
      misses += (a.cap > 0) ? miss : nreq;
      hits += (a.cap > 0) ? nreq - miss : 0;
    }
    base_m += nm;
    base_req += nr;
  }
  // block totals
  __shared__ long long red[2][LRU_THREADS / 32];
  long long hsum = hits, msum = misses;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
    msum += __shfl_xor_sync(0xffffffffu, msum, o);
  }
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = hsum;
    red[1][tid >> 5] = msum;
  }
  __syncthreads();
  if (tid == 0) {
    long long H2 = 0, M2 = 0;
    for (int w = 0; w < LRU_THREADS / 32; ++w) {
      H2 += red[0][w];
      M2 += red[1][w];
    }
    if (a.cap > 0) {
      L[0] = T0 + base_req;
      L[2] = count0 + base_m;
    }
    st.page_stats[u * 4 + 2 * kind + 0] = (int32_t)H2;
    st.page_stats[u * 4 + 2 * kind + 1] = (int32_t)M2;
    int64_t* ctr = a.counters + (size_t)u * 6 + 3 * kind;
    ctr[0] += H2;
    ctr[1] += M2;
    ctr[2] += M2 * (long long)(B * D * 2);
    if (a.miss_n) a.miss_n[u * 2 + kind] = (a.cap > 0) ? min(base_m, a.miss_cap) : 0;
  }
}

// gather: Tier-2 (pinned host, zero-copy) -> HBM slots for this step's misses
__global__ void __launch_bounds__(256) k_pagein(ckv_cache c, ckv_scratch sc, int32_t kw, int32_t vw, int32_t u0) {
  const int u = u0 + blockIdx.x, kind = blockIdx.y, tid = threadIdx.x;
  const int maxb = c.max_blocks;
  const int cap = kind ? sc.value_capacity : sc.key_capacity;
  uint16_t* slots = kind ? sc.value_slots : sc.key_slots;
  if (!slots || cap <= 0) return;
  const int words = kind ? vw : kw;
  const int32_t* slot_of = (kind ? sc.value_lru : sc.key_lru) + (size_t)u * words + lru_slot_offset(maxb, cap);
  const int n = sc.miss_n[u * 2 + kind];
  const int32_t* ml = sc.miss_list + ((size_t)u * 2 + kind) * sc.miss_cap;
  const uint16_t* src0 = kind ? c.tier2_v : c.tier2_k;
  // PCIe reads of zero-copy host memory are latency-bound: every thread keeps
  // PI_DEPTH 16-byte loads (from PI_DEPTH different blocks) in flight
  constexpr int PI_DEPTH = 8;
  for (int k0 = 0; k0 < n; k0 += PI_DEPTH) {
    uint4 v[PI_DEPTH];
    int sl[PI_DEPTH];
#pragma unroll
    for (int i = 0; i < PI_DEPTH; ++i) {
      sl[i] = -1;
      if (k0 + i < n) {
        const int b = ml[k0 + i];
        sl[i] = slot_of[b];
        if (sl[i] >= 0) {  // evicted again later in the same step: pass B reads Tier-2
          if (tid == 0 && !c.tier2_valid[(size_t)u * maxb + b]) atomicOr(&c.status[CKV_ST_TIER2], 1);
          v[i] = reinterpret_cast<const uint4*>(src0 + ((size_t)u * maxb + b) * B * D)[tid];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < PI_DEPTH; ++i)
      if (sl[i] >= 0)
        reinterpret_cast<uint4*>(slots + ((size_t)u * cap + sl[i]) * B * D)[tid] = v[i];
  }
}

__global__ void k_lru_init(int32_t* state, int words, int maxb, int R) {
  const int u = blockIdx.x;
  int32_t* L = state + (size_t)u * words;
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    int v;
    if (i == 0 || i == 1) v = 1;
    else if (i == 2) v = 0;
    else if (i == 3) v = R;
    else if (i < 4 + maxb) v = 0;
    else v = -1;  // ring entries and slots
    L[i] = v;
  }
}


cudaError_t launch_scratch(const ckv_cache* c, const ckv_step* st, const ckv_scratch* sc, int u0, int nu,
                           cudaStream_t s) {
  int words[2];
  LruArgs la[2];
  bool fast = true;
  for (int kind = 0; kind < 2; ++kind) {
    const int cap = kind ? sc->value_capacity : sc->key_capacity;
    const int R = lru_ring(c->max_blocks, cap);
    words[kind] = lru_words(c->max_blocks, cap);
    (void)R;
    la[kind] = LruArgs{*c, *st, kind ? sc->value_lru : sc->key_lru, words[kind], cap, kind, sc->counters,
                       sc->miss_list, sc->miss_n, sc->miss_cap, u0, 0};
    fast = fast && (R == 0);
  }
  if (fast) {  // no eviction possible for either kind: one light pass over the union list
    k_lru_fast<<<dim3(nu, 2), LRU_THREADS, 0, s>>>(la[0], la[1]);
    ++g_launches;
  } else {
    for (int kind = 0; kind < 2; ++kind) {
      const int R = lru_ring(c->max_blocks, la[kind].cap);
      size_t smem = (size_t)(c->max_blocks + R + c->max_blocks + lru_work_words(c->max_blocks)) * 4;
      if (smem > kLruSmemMax) {
        la[kind].gmem = 1;
        smem = 0;
      } else {
        set_max_dyn_smem(k_lru, (int)smem);
      }
      k_lru<<<nu, LRU_THREADS, smem, s>>>(la[kind]);
      ++g_launches;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // Default: pass B reads this step's misses from Tier-2 and fills their slots itself
  // (the PCIe transfer overlaps pass B); CKV_SEPARATE_PAGEIN=1: gather kernel first.
  const bool separate = knobs().separate_pagein;
  if (separate && (sc->key_slots || sc->value_slots) && sc->miss_list && sc->miss_n) {
    // page-in on a side stream: forked after the LRU, joined before pass B
    cudaStream_t side = dev_state().side;
    cudaEvent_t fork, join;
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    cudaEventRecord(fork, s);
    cudaStreamWaitEvent(side, fork, 0);
    k_pagein<<<dim3(nu, 2), 256, 0, side>>>(*c, *sc, words[0], words[1], u0);
    ++g_launches;
    cudaEventRecord(join, side);
    cudaStreamWaitEvent(s, join, 0);
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
  }
  return cudaGetLastError();
}

cudaError_t launch_lru_init(int32_t* state, int n_units, int max_blocks, int cap, cudaStream_t s) {
  const int R = lru_ring(max_blocks, cap);
  const int words = lru_words(max_blocks, cap);
  k_lru_init<<<n_units, 256, 0, s>>>(state, words, max_blocks, R);
  return cudaGetLastError();
}

}  // namespace ckv
