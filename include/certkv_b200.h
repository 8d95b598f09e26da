/*
 * certkv_b200.h -- C ABI of the B200-native certified quantized decode-attention
 * path (libcertkv_b200.so).  Plain pointers and sizes only; every buffer is
 * owned by the caller (device memory, or mapped pinned host memory where
 * noted).  No function throws; all return a ckv_status.
 *
 * Each entry point replaces a reference interface (paths relative to
 * /root/reference/pkg/src/certkv):
 *
 *   ckv_append          <- TieredCache.append_token / append_tokens / _fill_block
 *                          (cache.py:76-120) + quantize_key_block /
 *                          quantize_value_block / value_annotations
 *                          (quantizer.py:133-236)
 *   ckv_decode_step     <- harness.run_decode_step for every q-head of every
 *                          unit (harness.py:186-300): phase1_score
 *                          (attention.py:89-113), compute_delta
 *                          (certifier.py:89-104), adaptive_topk + rung1/rung2
 *                          (attention.py:162-203, fallback.py:134-161),
 *                          promote_blocks (cache.py:294-312), phase2_attend
 *                          (attention.py:227-300), ranking/boundary/canary
 *                          (fallback.py:164-199), assemble_certificate
 *                          (certifier.py:191-212)
 *   ckv_block_logmass   <- _kernels backend block_logmass (pure.py:16-36,
 *                          _core.pyx:16-44)
 *   ckv_fused_attend    <- _kernels backend fused_attend (pure.py:39-66,
 *                          _core.pyx:47-83)
 *   ckv_read_tier1      <- CacheBlock payload views (cache.py:42-46, quantizer.py:39-95)
 *   ckv_fault_offset    <- verification.corrupt_block_offset (verification.py:420-428)
 *   ckv_tier2_drop      <- "cache.tier2_keys[i] = None" (cache.py:138-142)
 *
 * Fixed geometry of the device path (Llama-3.1-8B attention): head_dim 128,
 * block_size 16, value group 16, up to 4 query heads per KV head.
 */
#ifndef CERTKV_B200_H
#define CERTKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKV_HEAD_DIM 128
#define CKV_BLOCK 16
#define CKV_GROUP 16
#define CKV_MAX_QHEADS 4
#define CKV_BLOCK_BYTES 4608 /* Tier-1 record: 2048 key codes + 1024 key meta + 1024 value codes + 512 value meta */

typedef enum {
  CKV_OK = 0,
  CKV_EINVAL = 1,          /* bad argument (maps to ValueError) */
  CKV_EMPTY = 2,           /* attention over an empty cache (EmptyCacheError) */
  CKV_ECAPACITY = 3,       /* append beyond the allocated block capacity (ValueError) */
  CKV_EPAGING = 4,         /* PagingError */
  CKV_ETIER2 = 5,          /* Tier2UnavailableError */
  CKV_ENONFINITE = 6,      /* non-finite key/value ingest (ValueError) */
  CKV_ECUDA = 7            /* CUDA launch / runtime error */
} ckv_status;

/* Device-resident tiered cache of n_units KV-head units (units = layers x
 * KV heads x sequences).  All arrays are [n_units][...] row-major. */
typedef struct {
  int32_t n_units;
  int32_t max_blocks;      /* full-block capacity per unit */
  uint8_t* tier1;          /* [n_units][max_blocks][CKV_BLOCK_BYTES] */
  float* eta;              /* [n_units][max_blocks] value error annotation */
  float* nu;               /* [n_units][max_blocks] value norm annotation */
  float* kscale_max;       /* [n_units][max_blocks] max key scale of the block */
  float* v_max;            /* [n_units] running max of nu over full blocks */
  int32_t* n_blocks;       /* [n_units] */
  int32_t* partial_len;    /* [n_units] */
  uint16_t* partial_k;     /* fp16 [n_units][16][128] trailing partial block */
  uint16_t* partial_v;
  uint16_t* tier2_k;       /* fp16 [n_units][max_blocks*16][128]; device or mapped pinned host */
  uint16_t* tier2_v;
  uint8_t* tier2_valid;    /* [n_units][max_blocks] 1 = originals present */
  int32_t* status;         /* [8] device error words (see CKV_ST_*) */
} ckv_cache;

/* status words.  NONFINITE counts the appends rejected for a non-finite entry
 * since the last reset (a host compares it with the count it has reported, so
 * every rejection is reported once, also through deferred checks); CAPACITY is
 * sticky; TIER2 is per decode step (cleared when the step begins, set by any
 * kernel of the step that needed a lost Tier-2 block); APPEND_BAD is the
 * verdict of the append in flight (cleared when it begins). */
#define CKV_MAX_BLOCKS 32768 /* full blocks per unit the selection holds (524288 tokens) */

#define CKV_ST_NONFINITE 0
#define CKV_ST_CAPACITY 1
#define CKV_ST_TIER2 2
#define CKV_ST_APPEND_BAD 3
#define CKV_ST_APPEND_CNT 4  /* internal: CTAs of the one-token append done */

typedef struct {
  double tau_cov;
  double v_tol;
  double epsilon_guard;
  double greedy_value_budget;   /* < 0 means None (threshold mode) */
  int32_t k_min;
  int32_t k_max;
  int32_t ranking_depth;
  int32_t exponent_mode;        /* 2 or 3 */
  int32_t rung1_enabled;
  int32_t rung2_enabled;
  int32_t ranking_checks_enabled;
  int32_t canary_enabled;
} ckv_policy;

/* Per (unit, q-head) certificate + decision summary, written by the device. */
typedef struct {
  double delta_h;
  double e_key_tight;
  double e_key_impl;
  double e_val;
  double est_tail_mass;
  double v_max;
  double canary_gap;        /* max |s_ref - s_quant| over promoted tokens */
  double partial_mass;
  int32_t k_star;           /* after rung 1 */
  int32_t k_star0;          /* before rung 1 */
  int32_t k_coverage;       /* -1 when larger than the sorted prefix */
  int32_t n_value_promoted;
  uint32_t flags;           /* CKV_F_* */
  int32_t returned_kind;    /* 0 quantized, 1 dense_per_head, 2 dense_all_heads */
} ckv_cert;

#define CKV_F_RUNG1 (1u << 0)
#define CKV_F_RUNG2 (1u << 1)
#define CKV_F_RANKING (1u << 2)   /* rung 3, cause ranking_disagree */
#define CKV_F_BOUNDARY (1u << 3)  /* rung 3, cause boundary */
#define CKV_F_CANARY (1u << 4)    /* rung 4, cause canary */
#define CKV_F_CLAMPED (1u << 5)
#define CKV_F_NUMERIC (1u << 6)   /* non-finite fast-path output -> rung 4 (precondition) */
#define CKV_F_ACTIVE (1u << 7)
#define CKV_F_EXPLORE (1u << 8)   /* rung 4, cause canary, from the exploration spot check */

/* Caller-owned per-step buffers (device memory). */
typedef struct {
  int32_t n_heads;          /* active q-heads per unit, 1..4 */
  int32_t n_splits;         /* pass-A split capacity per unit (from ckv_plan); each step
                               partitions a unit's blocks over at most this many */
  int32_t blocks_per_split; /* the smallest split ckv_plan sized the capacity for */
  int32_t kcap;             /* promoted-list capacity per head (>= 2*k_max+1) */
  int32_t wcap;             /* work-list capacity per head (kcap + max_blocks) */
  int32_t n_chunks;         /* pass-B chunks per head */
  int32_t items_per_chunk;
  const double* q;          /* [n_units][n_heads][128] queries */
  float* out;               /* [n_units][n_heads][128] */
  ckv_cert* cert;           /* [n_units][n_heads] */
  float* lm1;               /* [n_units][n_heads][max_blocks] phase-1 block log-mass */
  float* split_state;       /* [n_units][n_splits][4][CKV_SPLIT_FLOATS] */
  int32_t* order;           /* [n_units][n_heads][kcap] promoted blocks in mass order */
  int32_t* work;            /* [n_units][wcap] union work list: block | F-mask<<24 | V-mask<<28 */
  int32_t* n_work;          /* [n_units] */
  int32_t* vlist;           /* [n_units][n_heads][max_blocks] value promotions, ascending */
  float* lm2;               /* [n_units][n_heads][max_blocks] phase-2 log-mass of promoted blocks */
  float* head_state;        /* [n_units][n_heads][CKV_HEAD_FLOATS] */
  float* chunk_state;       /* [n_units][n_chunks][4][CKV_CHUNK_FLOATS] */
  int32_t* page_stats;      /* [n_units][4] key hits, key misses, value hits, value misses */
  void* prof_begin;         /* optional cudaEvent_t recorded before / after pass A */
  void* prof_end;
  int32_t rung4_group;      /* units sharing a step-wide rung 4 (0 = all units) */
  int32_t n_dsplit_cap;     /* dense-fallback splits per unit (from ckv_plan) */
  int32_t* dense_list;      /* [1 + 2 n_units] count, per-item split counters, then
                               unit | head_mask << 24 per dense item */
  float* dense_part;        /* [n_units][n_dsplit_cap][4][132] dense split states */
  int32_t ecap;             /* exploration samples per head (capacity) */
  int32_t* explore_n;       /* [n_units][n_heads] samples drawn by the host, or NULL */
  int32_t* explore_pos;     /* [n_units][n_heads][ecap] ascending tail positions */
  const int32_t* unit_group; /* [n_units] Rung-4 group of each unit (e.g. its (layer, sequence)),
                                or NULL for u / rung4_group */
  int32_t* group_flags;     /* [n_groups] step-wide Rung-4 request per group */
  int32_t n_groups;
  int32_t* unit_done;       /* [n_units] zero-initialised, self-resetting: the last q-head
                               selection of a unit builds its union work list (NULL: a
                               separate launch does) */
  int32_t* queue;           /* [2] zero-initialised, self-resetting work-queue counters of the
                               persistent pass B (NULL: one CTA per (chunk, unit)) */
  float* stash;             /* [n_units][max_blocks][4][16] phase-1 scores of likely-promoted
                               blocks, written by pass A (NULL: off) */
  int32_t* stash_epoch;     /* [n_units][max_blocks] epoch << 4 | mask of stashed heads (init -1) */
  int32_t epoch;            /* this step's epoch, < 2^27 (the caller increments it every step) */
  float stash_margin;       /* a block is stashed when some head's l'_b exceeds that head's
                               largest tail l' of the previous step minus this margin */
  int32_t plan_units;       /* 0: launch-shape heuristics follow the units of the launch;
                               > 0: they follow this many units (pass ckv_plan's n_units of
                               the whole job so a shard computes bit for bit what the
                               unsharded step computes for its units) */
  int32_t dense_splits;     /* 0: dense splits per unit adapt to the number of dense units;
                               > 0: fixed (independent of which other units are dense) */
  uint64_t* explore_rng;    /* [16] numpy Philox4x64 generator state (counter[4], key[2],
                               buffer[4], buffer_pos, has_uint32, uinteger): when set, the
                               exploration samples are drawn on the device from it, in the
                               reference's stream order, and it is advanced in place;
                               NULL: explore_n / explore_pos hold host-drawn samples */
  double explore_rate;      /* exploration_rate of the policy (device draws) */
  int32_t* explore_work;    /* [CKV_EXPLORE_WORK(n_units * n_heads)] device-draw scratch */
  int32_t* flow;            /* [6 * n_units + 4] zero-initialised, self-maintaining: per-unit
                               completion epochs of pass A / selection / pass B (+ counters
                               and step-wide words), so those kernels, and in ckv_decode_step
                               the dense pass, run as programmatic dependent launches that
                               overlap on finished units (NULL: plain stream order) */
  unsigned long long* trace; /* [32][2] optional timeline (profiling): per kernel of the step,
                               the first CTA start / last CTA end (globaltimer ns) by
                               atomicMin / atomicMax; the caller resets it (NULL: off) */
  void* host_report;        /* optional pinned host buffer the device can write (e.g.
                               cudaHostAlloc / pinned torch memory under unified addressing):
                               the step's last kernel writes the step's bound report there,
                               cert[n_units][n_heads] | the cache's 8 status words |
                               page_stats[n_units][4] (when set) | explore_n[n_units][n_heads]
                               (when set), each part 16-byte aligned
                               (ckv_report_bytes), so the caller reads it after the step's
                               completion with no device-to-host copies (NULL: off) */
} ckv_step;

/* trace slots */
#define CKV_TR_PASS_A 0
#define CKV_TR_SELECT 1
#define CKV_TR_PASS_B 2
#define CKV_TR_COMBINE 3
#define CKV_TR_FLAGS 4
#define CKV_TR_RESOLVE 5
#define CKV_TR_DENSE 6
#define CKV_TR_XDRAW 7
#define CKV_TR_EXPLORE 8
#define CKV_TR_LRU 9

#define CKV_EXPLORE_WORK(items) (4 * (items) + 64)

#define CKV_SPLIT_FLOATS 136
#define CKV_HEAD_FLOATS 288
#define CKV_CHUNK_FLOATS 136

/* Scratch (LRU page-in) state per unit; capacity in blocks for keys and values.
 * When key_slots / value_slots are given (Tier-2 in pinned host RAM), every
 * miss is stamped with st->epoch in the LRU state and copied from Tier-2 into
 * its HBM slot by pass B as it reads it (or, with CKV_SEPARATE_PAGEIN=1 in the
 * environment, by a gather kernel on a side stream joined before pass B); pass B
 * and the dense fallback read resident originals from the slots
 * (ScratchCache.request, cache.py:261-286).  The caller must change st->epoch
 * every step.  Without slots (Tier-2 already in HBM) only the reference
 * accounting runs.  LRU state words per unit: ckv_lru_words(). */
typedef struct {
  int32_t key_capacity;
  int32_t value_capacity;
  int32_t* key_lru;         /* [n_units][ckv_lru_words(max_blocks, key_capacity)] */
  int32_t* value_lru;
  int64_t* counters;        /* [n_units][6] hits, misses, bytes for keys then values */
  uint16_t* key_slots;      /* [n_units][key_capacity][16*128] fp16, or NULL */
  uint16_t* value_slots;    /* [n_units][value_capacity][16*128] fp16, or NULL */
  int32_t* miss_list;       /* [n_units][2][miss_cap] block ids paged in this step */
  int32_t* miss_n;          /* [n_units][2] */
  int32_t miss_cap;
} ckv_scratch;

/* Library / device info. */
int32_t ckv_version(void);
/* sizeof of the ABI structs as this library was compiled: out[0..4] = ckv_cache,
 * ckv_policy, ckv_cert, ckv_step, ckv_scratch (lets a binding check its mirrors) */
void ckv_struct_sizes(int32_t* out);
int32_t ckv_lru_words(int32_t max_blocks, int32_t capacity);
/* Byte size and part offsets of the host_report layout: out[0..3] = total bytes,
 * offset of the status words, of page_stats, of explore_n (cert at 0). */
void ckv_report_layout(int32_t n_units, int32_t n_heads, int64_t* out);
/* Initialise both LRU states and zero the cumulative counters. */
ckv_status ckv_scratch_init(int32_t n_units, int32_t max_blocks, const ckv_scratch* s, void* stream);

/* Plan a decode step: fills the sizing fields of *st from the cache size. */
ckv_status ckv_plan(int32_t n_units, int32_t max_blocks, int32_t n_heads, const ckv_policy* pol,
                     ckv_step* st);

/* Quantize-on-append: k_new, v_new fp16 device [n_units][n_tok][128]. */
ckv_status ckv_append(const ckv_cache* c, const uint16_t* k_new, const uint16_t* v_new,
                      int32_t n_tok, void* stream);

/* Binary16 ingest of float64 data (correctly rounded, as numpy's astype(float16)). */
ckv_status ckv_f64_to_f16(const double* x, uint16_t* y, int64_t n, void* stream);

/* Zero a cache's counters (n_blocks, partial_len, v_max, status). */
ckv_status ckv_reset(const ckv_cache* c, void* stream);

/* One certified decode step over every unit; host_max_blocks bounds the
 * grid (the largest n_blocks of any unit).  scratch may be NULL (no LRU
 * accounting, promoted originals read straight from Tier-2). */
ckv_status ckv_decode_step(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                           const ckv_scratch* scratch, int32_t host_max_blocks,
                           void* stream);

/* The step in parts, for callers that must act between them:
 *   ckv_decode_begin:  pass A, selection, LRU scratch + page-in (when scratch),
 *                      pass B, combine (certificates written).  The exploration
 *                      spot check draws its host-side Philox samples from the
 *                      tail size K' reported here.
 *   ckv_decode_flags:  exploration (when st->explore_n), then the step-wide
 *                      Rung-4 request of every group into st->group_flags.
 *                      A KV-head sharded caller all-reduces (MAX) group_flags
 *                      across ranks here (harness.py:362-372 per layer).
 *   ckv_decode_finish: every head of a flagged group returns dense
 *                      (dense_all_heads); exact dense fallback of rung-3/4 heads.
 *                      With a scratch that has HBM slots (Tier-2 in host RAM), blocks
 *                      resident in a slot are read from HBM, the rest from Tier-2
 *                      (same bytes either way; NULL scratch: Tier-2 only).
 *   ckv_decode_end = ckv_decode_flags + ckv_decode_finish. */
ckv_status ckv_decode_begin(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                            const ckv_scratch* scratch, int32_t host_max_blocks, void* stream);
ckv_status ckv_decode_flags(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                            int32_t host_max_blocks, void* stream);
ckv_status ckv_decode_finish(const ckv_cache* c, ckv_step* st, const ckv_scratch* scratch,
                             int32_t host_max_blocks, void* stream);
ckv_status ckv_decode_end(const ckv_cache* c, const ckv_policy* pol, ckv_step* st,
                          const ckv_scratch* scratch, int32_t host_max_blocks, void* stream);

/* Unpack Tier-1 for parity: codes i8 [nb][16][128], kscale/koffset f32 [nb][128],
 * vcodes u8 [nb][16][128], vscale/voffset fp16 [nb][16][8], for blocks
 * [b0, b0+nb) of one unit.  Device output pointers. */
ckv_status ckv_read_tier1(const ckv_cache* c, int32_t unit, int32_t b0, int32_t nb,
                          int8_t* kcodes, float* kscale, float* koffset, uint8_t* vcodes,
                          uint16_t* vscale, uint16_t* voffset, void* stream);

/* Fault injection: add `shift` (fp32) to one stored key offset. */
ckv_status ckv_fault_offset(const ckv_cache* c, int32_t unit, int32_t block, int32_t channel,
                            float shift, void* stream);

/* Mark Tier-2 originals of one block as lost (hard error when needed). */
ckv_status ckv_tier2_drop(const ckv_cache* c, int32_t unit, int32_t block, void* stream);

/* Kernel-backend plugin functions (pure.py:16-66), device pointers:
 * scores f64[T], bounds i64[nb+1] -> block_max, block_sum, log_mass f64[nb]. */
ckv_status ckv_block_logmass(const double* scores, const int64_t* bounds, int32_t nb,
                             double* block_max, double* block_sum, double* log_mass,
                             void* stream);
/* scores f32[T], values f32[T][d], bounds i64[nb+1] -> out f32[d], ml f32[2]. */
ckv_status ckv_fused_attend(const float* scores, const float* values, const int64_t* bounds,
                            int32_t nb, int32_t d, float* out, float* ml, void* stream);

/* Number of kernel launches issued by the last ckv_decode_step / ckv_append
 * on this thread (for the bench's gpu_launches claim). */
int32_t ckv_last_launches(void);

/* Text of the last CUDA error that produced CKV_ECUDA on this thread. */
const char* ckv_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CERTKV_B200_H */
