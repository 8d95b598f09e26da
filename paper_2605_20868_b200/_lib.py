"""ctypes binding of libcertkv_b200.so (include/certkv_b200.h).

The shared library is built in-tree by ``build.py`` (``__graft_entry__.build``).
There is no fallback: if the library is missing or a CUDA device is absent,
every compute entry point raises.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcertkv_b200.so")

HEAD_DIM = 128
BLOCK = 16
GROUP = 16
MAX_QHEADS = 4
BLOCK_BYTES = 4608
SPLIT_FLOATS = 136
HEAD_FLOATS = 288
CHUNK_FLOATS = 136

ST_NONFINITE, ST_CAPACITY, ST_TIER2, ST_APPEND_BAD = 0, 1, 2, 3

F_RUNG1, F_RUNG2, F_RANKING, F_BOUNDARY = 1, 2, 4, 8
F_CANARY, F_CLAMPED, F_NUMERIC, F_ACTIVE = 16, 32, 64, 128
F_EXPLORE = 256

STATUS = {0: "CKV_OK", 1: "CKV_EINVAL", 2: "CKV_EMPTY", 3: "CKV_ECAPACITY",
          4: "CKV_EPAGING", 5: "CKV_ETIER2", 6: "CKV_ENONFINITE", 7: "CKV_ECUDA"}

P = ctypes.c_void_p
I32 = ctypes.c_int32
F64 = ctypes.c_double


class CkvCache(ctypes.Structure):
    _fields_ = [("n_units", I32), ("max_blocks", I32), ("tier1", P), ("eta", P), ("nu", P),
                ("kscale_max", P), ("v_max", P), ("n_blocks", P), ("partial_len", P),
                ("partial_k", P), ("partial_v", P), ("tier2_k", P), ("tier2_v", P),
                ("tier2_valid", P), ("status", P)]


class CkvPolicy(ctypes.Structure):
    _fields_ = [("tau_cov", F64), ("v_tol", F64), ("epsilon_guard", F64),
                ("greedy_value_budget", F64), ("k_min", I32), ("k_max", I32),
                ("ranking_depth", I32), ("exponent_mode", I32), ("rung1_enabled", I32),
                ("rung2_enabled", I32), ("ranking_checks_enabled", I32), ("canary_enabled", I32)]


class CkvCert(ctypes.Structure):
    _fields_ = [("delta_h", F64), ("e_key_tight", F64), ("e_key_impl", F64), ("e_val", F64),
                ("est_tail_mass", F64), ("v_max", F64), ("canary_gap", F64),
                ("partial_mass", F64), ("k_star", I32), ("k_star0", I32), ("k_coverage", I32),
                ("n_value_promoted", I32), ("flags", ctypes.c_uint32), ("returned_kind", I32)]


class CkvStep(ctypes.Structure):
    _fields_ = [("n_heads", I32), ("n_splits", I32), ("blocks_per_split", I32), ("kcap", I32),
                ("wcap", I32), ("n_chunks", I32), ("items_per_chunk", I32), ("q", P),
                ("out", P), ("cert", P), ("lm1", P), ("split_state", P), ("order", P),
                ("work", P), ("n_work", P), ("vlist", P), ("lm2", P), ("head_state", P),
                ("chunk_state", P), ("page_stats", P), ("prof_begin", P), ("prof_end", P),
                ("rung4_group", I32), ("n_dsplit_cap", I32), ("dense_list", P), ("dense_part", P),
                ("ecap", I32), ("explore_n", P), ("explore_pos", P), ("unit_group", P),
                ("group_flags", P), ("n_groups", I32), ("unit_done", P),
                ("queue", P), ("stash", P), ("stash_epoch", P), ("epoch", I32),
                ("stash_margin", ctypes.c_float), ("plan_units", I32), ("dense_splits", I32),
                ("explore_rng", P), ("explore_rate", ctypes.c_double), ("explore_work", P),
                ("flow", P), ("trace", P), ("host_report", P)]


class CkvScratch(ctypes.Structure):
    _fields_ = [("key_capacity", I32), ("value_capacity", I32), ("key_lru", P),
                ("value_lru", P), ("counters", P), ("key_slots", P), ("value_slots", P),
                ("miss_list", P), ("miss_n", P), ("miss_cap", I32)]


CERT_DTYPE_FIELDS = [(n, t) for n, t in CkvCert._fields_]

_lib = None


def load():
    """Load the in-tree library; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the certified decode path)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "ckv_version": (I32, []),
        "ckv_struct_sizes": (None, [P]),
        "ckv_lru_words": (I32, [I32, I32]),
        "ckv_report_layout": (None, [I32, I32, P]),
        "ckv_scratch_init": (I32, [I32, I32, ctypes.POINTER(CkvScratch), P]),
        "ckv_plan": (I32, [I32, I32, I32, ctypes.POINTER(CkvPolicy), ctypes.POINTER(CkvStep)]),
        "ckv_append": (I32, [ctypes.POINTER(CkvCache), P, P, I32, P]),
        "ckv_reset": (I32, [ctypes.POINTER(CkvCache), P]),
        "ckv_decode_step": (I32, [ctypes.POINTER(CkvCache), ctypes.POINTER(CkvPolicy),
                                  ctypes.POINTER(CkvStep), ctypes.POINTER(CkvScratch), I32, P]),
        "ckv_decode_begin": (I32, [ctypes.POINTER(CkvCache), ctypes.POINTER(CkvPolicy),
                                   ctypes.POINTER(CkvStep), ctypes.POINTER(CkvScratch), I32, P]),
        "ckv_decode_end": (I32, [ctypes.POINTER(CkvCache), ctypes.POINTER(CkvPolicy),
                                 ctypes.POINTER(CkvStep), ctypes.POINTER(CkvScratch), I32, P]),
        "ckv_decode_flags": (I32, [ctypes.POINTER(CkvCache), ctypes.POINTER(CkvPolicy),
                                   ctypes.POINTER(CkvStep), I32, P]),
        "ckv_decode_finish": (I32, [ctypes.POINTER(CkvCache), ctypes.POINTER(CkvStep),
                                    ctypes.POINTER(CkvScratch), I32, P]),
        "ckv_read_tier1": (I32, [ctypes.POINTER(CkvCache), I32, I32, I32, P, P, P, P, P, P, P]),
        "ckv_fault_offset": (I32, [ctypes.POINTER(CkvCache), I32, I32, I32, ctypes.c_float, P]),
        "ckv_tier2_drop": (I32, [ctypes.POINTER(CkvCache), I32, I32, P]),
        "ckv_block_logmass": (I32, [P, P, I32, P, P, P, P]),
        "ckv_fused_attend": (I32, [P, P, P, I32, I32, P, P, P]),
        "ckv_last_launches": (I32, []),
        "ckv_f64_to_f16": (I32, [P, P, ctypes.c_int64, P]),
        "ckv_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    """Names every entry point declared in include/certkv_b200.h."""
    return ["ckv_version", "ckv_lru_words", "ckv_scratch_init", "ckv_plan", "ckv_append",
            "ckv_reset", "ckv_decode_step", "ckv_read_tier1", "ckv_fault_offset",
            "ckv_tier2_drop", "ckv_block_logmass", "ckv_fused_attend", "ckv_last_launches",
            "ckv_f64_to_f16", "ckv_last_error", "ckv_decode_begin", "ckv_decode_end",
            "ckv_decode_flags", "ckv_decode_finish", "ckv_struct_sizes", "ckv_report_layout"]


def check(code, what):
    """Map a ckv_status to the reference's exception classes (cache.py:29-39)."""
    if code == 0:
        return
    from .errors import PagingError, Tier2UnavailableError, EmptyCacheError
    name = STATUS.get(code, str(code))
    if code in (1, 3, 6):
        raise ValueError(f"{what}: {name}")
    if code == 2:
        raise EmptyCacheError(f"{what}: {name}")
    if code == 4:
        raise PagingError(f"{what}: {name}")
    if code == 5:
        raise Tier2UnavailableError(f"{what}: {name}")
    detail = ""
    if code == 7 and _lib is not None:
        detail = " (" + (_lib.ckv_last_error() or b"").decode() + ")"
    raise RuntimeError(f"{what}: {name}{detail}")
