// extern "C" entry points of libcertkv_b200.so (declared in include/certkv_b200.h).
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include "common.cuh"

namespace ckv {
const Knobs& knobs() {
  static const Knobs k = [] {
    Knobs r;
    r.separate_lru = getenv("CKV_SEPARATE_LRU") != nullptr;
    r.separate_pagein = getenv("CKV_SEPARATE_PAGEIN") != nullptr;
    const char* ch = getenv("CKV_CHUNKS");
    r.chunks = ch ? atoi(ch) : 1;
    r.sel_kpt = r.sel_nt = 0;
    if (const char* sv = getenv("CKV_SEL")) sscanf(sv, "%d:%d", &r.sel_kpt, &r.sel_nt);
    const char* pc = getenv("CKV_PB_CHUNKS");
    r.pb_chunks = pc ? atoi(pc) : 0;
    const char* ds = getenv("CKV_DN_SPLITS");
    r.dn_splits = ds ? atoi(ds) : 0;
    return r;
  }();
  return k;
}

static std::mutex g_dev_mu;
static DevState g_dev[64];

DevState& dev_state() {
  int d = 0;
  cudaGetDevice(&d);
  DevState& ds = g_dev[d & 63];
  if (!ds.sms) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!ds.sms) {
      int lo = 0, hi = 0, sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStreamCreateWithPriority(&ds.tail, cudaStreamNonBlocking, hi);
      cudaStreamCreateWithFlags(&ds.side, cudaStreamNonBlocking);
      ds.sms = sms > 0 ? sms : 148;
    }
  }
  return ds;
}

cudaError_t set_max_dyn_smem_fn(const void* fn, int bytes) {
  DevState& ds = dev_state();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  for (int i = 0; i < ds.n_attr; ++i)
    if (ds.attr_fn[i] == fn) {
      if (ds.attr_bytes[i] >= bytes) return cudaSuccess;
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) ds.attr_bytes[i] = bytes;
      return e;
    }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && ds.n_attr < 32) {
    ds.attr_fn[ds.n_attr] = fn;
    ds.attr_bytes[ds.n_attr] = bytes;
    ++ds.n_attr;
  }
  return e;
}
cudaError_t launch_append(const ckv_cache*, const uint16_t*, const uint16_t*, int32_t, cudaStream_t);
cudaError_t launch_read_tier1(const ckv_cache*, int, int, int, int8_t*, float*, float*, uint8_t*,
                              uint16_t*, uint16_t*, cudaStream_t);
cudaError_t launch_fault_offset(const ckv_cache*, int, int, int, float, cudaStream_t);
cudaError_t launch_tier2_drop(const ckv_cache*, int, int, cudaStream_t);
cudaError_t launch_f64_to_f16(const double*, uint16_t*, size_t, cudaStream_t);
cudaError_t launch_reset(const ckv_cache*, cudaStream_t);
cudaError_t launch_decode(const ckv_cache*, const ckv_policy*, const ckv_step*, const ckv_scratch*, int, bool,
                          cudaStream_t);
cudaError_t launch_dense(const ckv_cache*, const ckv_step*, const ckv_scratch*, int, bool, cudaStream_t);
bool decode_flow(const ckv_cache*, const ckv_step*);
cudaError_t launch_group_flags(const ckv_cache*, const ckv_step*, cudaStream_t);
cudaError_t launch_publish(const ckv_cache*, const ckv_step*, cudaStream_t);
cudaError_t launch_explore(const ckv_cache*, const ckv_policy*, const ckv_step*, int, cudaStream_t);
cudaError_t launch_explore_draw(const ckv_cache*, const ckv_step*, cudaStream_t);
cudaError_t launch_scratch(const ckv_cache*, const ckv_step*, const ckv_scratch*, cudaStream_t);
cudaError_t launch_lru_init(int32_t*, int, int, int, cudaStream_t);
cudaError_t launch_block_logmass(const double*, const int64_t*, int, double*, double*, double*,
                                 cudaStream_t);
cudaError_t launch_fused_attend(const float*, const float*, const int64_t*, int, int, float*, float*,
                                cudaStream_t);
}  // namespace ckv

static thread_local char g_err[256] = "";
static ckv_status st_of(cudaError_t e) {
  if (e == cudaSuccess) return CKV_OK;
  snprintf(g_err, sizeof(g_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return CKV_ECUDA;
}
static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static bool cache_ok(const ckv_cache* c) {
  return c && c->n_units > 0 && c->max_blocks > 0 && c->tier1 && c->eta && c->nu && c->kscale_max &&
         c->v_max && c->n_blocks && c->partial_len && c->partial_k && c->partial_v && c->tier2_k &&
         c->tier2_v && c->tier2_valid && c->status;
}

extern "C" {

int32_t ckv_version(void) { return 100; }

void ckv_struct_sizes(int32_t* out) {
  if (!out) return;
  out[0] = (int32_t)sizeof(ckv_cache);
  out[1] = (int32_t)sizeof(ckv_policy);
  out[2] = (int32_t)sizeof(ckv_cert);
  out[3] = (int32_t)sizeof(ckv_step);
  out[4] = (int32_t)sizeof(ckv_scratch);
}

void ckv_report_layout(int32_t n_units, int32_t n_heads, int64_t* out) {
  if (!out) return;
  ckv::report_layout(n_units, n_heads, out);
}

int32_t ckv_lru_words(int32_t max_blocks, int32_t capacity) {
  return ckv::lru_words(max_blocks, capacity);
}

ckv_status ckv_scratch_init(int32_t n_units, int32_t max_blocks, const ckv_scratch* sc,
                            void* stream) {
  if (!sc || n_units <= 0 || max_blocks <= 0 || sc->key_capacity < 0 || sc->value_capacity < 0 ||
      !sc->key_lru || !sc->value_lru || !sc->counters)
    return CKV_EINVAL;
  cudaError_t e = ckv::launch_lru_init(sc->key_lru, n_units, max_blocks, sc->key_capacity, S(stream));
  if (e == cudaSuccess)
    e = ckv::launch_lru_init(sc->value_lru, n_units, max_blocks, sc->value_capacity, S(stream));
  if (e == cudaSuccess)
    e = cudaMemsetAsync(sc->counters, 0, sizeof(int64_t) * 6 * (size_t)n_units, S(stream));
  return st_of(e);
}

ckv_status ckv_plan(int32_t n_units, int32_t max_blocks, int32_t n_heads, const ckv_policy* pol,
                    ckv_step* st) {
  if (!pol || !st || n_units <= 0 || max_blocks <= 0 || n_heads < 1 || n_heads > CKV_MAX_QHEADS)
    return CKV_EINVAL;
  if (max_blocks > CKV_MAX_BLOCKS) return CKV_EINVAL;  /* selection holds <= 32768 blocks per unit */
  if (pol->k_max < 0 || pol->k_min < 0 || pol->k_max < pol->k_min || pol->k_max > 511 ||
      pol->ranking_depth < 1 || pol->ranking_depth > 64)
    return CKV_EINVAL;
  /* pass-A split capacity: splits of >= 64 blocks; the launch picks how many it
     uses (pa_splits in decode.cu) */
  const int bps = 64;
  st->n_heads = n_heads;
  st->blocks_per_split = bps;
  st->n_splits = (max_blocks + bps - 1) / bps;
  st->kcap = 2 * pol->k_max + 2;
  st->wcap = st->kcap + max_blocks;
  st->items_per_chunk = 192;  /* measured at C3: 192 < 128 < 352 < 256 us */
  /* few units (e.g. 8-way KV-head sharding): smaller chunks so pass B still fills the GPU */
  while (st->items_per_chunk > 32 &&
         (long long)n_units * ((4 * st->kcap + st->items_per_chunk - 1) / st->items_per_chunk) < 888)
    st->items_per_chunk /= 2;
  if (st->items_per_chunk < 32) st->items_per_chunk = 32;
#ifdef CKV_PB_IPC
  st->items_per_chunk = CKV_PB_IPC;
#endif
  st->n_chunks = (4 * st->kcap + st->items_per_chunk - 1) / st->items_per_chunk;
  if (st->n_chunks < 1) st->n_chunks = 1;
  if (st->n_chunks > 256) st->n_chunks = 256;
  st->n_dsplit_cap = max_blocks / 8 < 1 ? 1 : (max_blocks / 8 > 256 ? 256 : max_blocks / 8);  /* dense splits per unit */
  return CKV_OK;
}

ckv_status ckv_append(const ckv_cache* c, const uint16_t* k_new, const uint16_t* v_new,
                      int32_t n_tok, void* stream) {
  if (!cache_ok(c) || n_tok < 0 || (n_tok > 0 && (!k_new || !v_new))) return CKV_EINVAL;
  if (n_tok == 0) return CKV_OK;
  return st_of(ckv::launch_append(c, k_new, v_new, n_tok, S(stream)));
}

ckv_status ckv_reset(const ckv_cache* c, void* stream) {
  if (!cache_ok(c)) return CKV_EINVAL;
  return st_of(ckv::launch_reset(c, S(stream)));
}

static bool step_ok(const ckv_cache* c, const ckv_policy* pol, const ckv_step* st,
                    int32_t host_max_blocks) {
  if (!cache_ok(c) || !pol || !st || !st->q || !st->out || !st->cert || !st->lm1 ||
      !st->split_state || !st->order || !st->work || !st->n_work || !st->vlist || !st->lm2 ||
      !st->head_state || !st->chunk_state || !st->dense_list || !st->dense_part ||
      !st->group_flags || st->n_groups < 1 || (!st->unit_group && st->rung4_group < 1))
    return false;
  return host_max_blocks >= 0 && host_max_blocks <= c->max_blocks;
}

static ckv_status decode_begin(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                               const ckv_scratch* scratch, int32_t host_max_blocks, bool finish,
                               void* stream) {
  if (!step_ok(c, pol, st, host_max_blocks)) return CKV_EINVAL;
  if (scratch && (!st->page_stats || !scratch->key_lru || !scratch->value_lru || !scratch->counters))
    return CKV_EINVAL;
  // (the per-step words -- Tier-2 loss, page stats -- are cleared by k_step_begin)
  return st_of(ckv::launch_decode(c, pol, st, scratch, host_max_blocks, finish, S(stream)));
}

ckv_status ckv_decode_begin(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                            const ckv_scratch* scratch, int32_t host_max_blocks, void* stream) {
  return decode_begin(c, pol, st, scratch, host_max_blocks, false, stream);
}

ckv_status ckv_decode_flags(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                            int32_t host_max_blocks, void* stream) {
  if (!step_ok(c, pol, st, host_max_blocks)) return CKV_EINVAL;
  cudaError_t e = cudaSuccess;
  if (st->explore_rng) {  // exploration samples drawn on the device (explore_draw.cu)
    if (!st->explore_n || !st->explore_pos || !st->explore_work || st->ecap <= 0 ||
        !(st->explore_rate > 0.0))
      return CKV_EINVAL;
    e = ckv::launch_explore_draw(c, st, S(stream));
    if (e != cudaSuccess) return st_of(e);
  }
  if (st->explore_n) {
    if (!st->explore_pos || st->ecap <= 0) return CKV_EINVAL;
    e = ckv::launch_explore(c, pol, st, host_max_blocks, S(stream));
    if (e != cudaSuccess) return st_of(e);
  }
  return st_of(ckv::launch_group_flags(c, st, S(stream)));
}

ckv_status ckv_decode_finish(const ckv_cache* c, ckv_step* st, const ckv_scratch* scratch,
                             int32_t host_max_blocks, void* stream) {
  ckv_policy dummy{};
  dummy.k_max = 1;
  if (!step_ok(c, &dummy, st, host_max_blocks)) return CKV_EINVAL;
  cudaError_t e = ckv::launch_dense(c, st, scratch, (host_max_blocks + 1) * CKV_BLOCK, false, S(stream));
  if (e == cudaSuccess && st->host_report) e = ckv::launch_publish(c, st, S(stream));
  return st_of(e);
}

ckv_status ckv_decode_end(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                          const ckv_scratch* scratch, int32_t host_max_blocks, void* stream) {
  ckv_status r = ckv_decode_flags(c, pol, st, host_max_blocks, stream);
  if (r != CKV_OK) return r;
  return ckv_decode_finish(c, st, scratch, host_max_blocks, stream);
}

ckv_status ckv_decode_step(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                           const ckv_scratch* scratch, int32_t host_max_blocks, void* stream) {
  if (st && c && !st->explore_rng && ckv::decode_flow(c, st)) {
    // the whole step as one dataflow: the last combine CTA resolves the step-wide
    // Rung 4 and the dense list, the dense pass launches right behind it
    ckv_status r = decode_begin(c, pol, st, scratch, host_max_blocks, true, stream);
    if (r != CKV_OK) return r;
    cudaError_t e = ckv::launch_dense(c, st, scratch, (host_max_blocks + 1) * CKV_BLOCK, true, S(stream));
    if (e == cudaSuccess && st->host_report) e = ckv::launch_publish(c, st, S(stream));
    return st_of(e);
  }
  ckv_status r = ckv_decode_begin(c, pol, st, scratch, host_max_blocks, stream);
  if (r != CKV_OK) return r;
  int32_t* en = st->explore_n;
  // host-drawn samples need the begin half's K' first (begin / end); device draws
  // (explore_rng) happen in stream order inside the step
  if (!st->explore_rng) st->explore_n = nullptr;
  r = ckv_decode_end(c, pol, st, scratch, host_max_blocks, stream);
  st->explore_n = en;
  return r;
}

ckv_status ckv_read_tier1(const ckv_cache* c, int32_t unit, int32_t b0, int32_t nb, int8_t* kcodes,
                          float* kscale, float* koffset, uint8_t* vcodes, uint16_t* vscale,
                          uint16_t* voffset, void* stream) {
  if (!cache_ok(c) || unit < 0 || unit >= c->n_units || b0 < 0 || nb < 0 || b0 + nb > c->max_blocks)
    return CKV_EINVAL;
  return st_of(ckv::launch_read_tier1(c, unit, b0, nb, kcodes, kscale, koffset, vcodes, vscale,
                                      voffset, S(stream)));
}

ckv_status ckv_fault_offset(const ckv_cache* c, int32_t unit, int32_t block, int32_t channel,
                            float shift, void* stream) {
  if (!cache_ok(c) || unit < 0 || unit >= c->n_units || block < 0 || block >= c->max_blocks ||
      channel < 0 || channel >= CKV_HEAD_DIM)
    return CKV_EINVAL;
  return st_of(ckv::launch_fault_offset(c, unit, block, channel, shift, S(stream)));
}

ckv_status ckv_tier2_drop(const ckv_cache* c, int32_t unit, int32_t block, void* stream) {
  if (!cache_ok(c) || unit < 0 || unit >= c->n_units || block < 0 || block >= c->max_blocks)
    return CKV_EINVAL;
  return st_of(ckv::launch_tier2_drop(c, unit, block, S(stream)));
}

ckv_status ckv_block_logmass(const double* scores, const int64_t* bounds, int32_t nb,
                             double* block_max, double* block_sum, double* log_mass, void* stream) {
  if (nb < 0 || (nb > 0 && (!scores || !bounds || !block_max || !block_sum || !log_mass)))
    return CKV_EINVAL;
  return st_of(ckv::launch_block_logmass(scores, bounds, nb, block_max, block_sum, log_mass, S(stream)));
}

ckv_status ckv_fused_attend(const float* scores, const float* values, const int64_t* bounds,
                            int32_t nb, int32_t d, float* out, float* ml, void* stream) {
  if (nb < 0 || d <= 0 || d > 1024 || !out || !ml) return CKV_EINVAL;
  return st_of(ckv::launch_fused_attend(scores, values, bounds, nb, d, out, ml, S(stream)));
}

ckv_status ckv_f64_to_f16(const double* x, uint16_t* y, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return CKV_EINVAL;
  return st_of(ckv::launch_f64_to_f16(x, y, (size_t)n, S(stream)));
}

int32_t ckv_last_launches(void) { return ckv::g_launches; }

const char* ckv_last_error(void) { return g_err; }

}  // extern "C"
