"""Certified decode step, fallback ladder and telemetry restated in NumPy.

Restates attention.py, certifier.py, fallback.py and harness.py of the
reference (citations per function).  TEST INFRASTRUCTURE ONLY -- see
``oracle/__init__.py``.
"""

import dataclasses
import math
from dataclasses import dataclass

import numpy as np

from .kv import OracleKV, OracleScratch, PagingFault, promote

QUANTIZED, DENSE_HEAD, DENSE_ALL = "quantized", "dense_per_head", "dense_all_heads"


@dataclass(frozen=True)
class OraclePolicy:
    """Policy fields, defaults and validation of fallback.py:35-111."""
    tau_cov: float = 0.995
    k_min: int = 2
    k_max: int = 128
    v_tol: float = 0.05
    ranking_depth: int = 1
    epsilon_guard: float = 1e-6
    exploration_rate: float = 0.02
    exponent_mode: int = 3
    greedy_value_budget: float | None = None
    rung1_enabled: bool = True
    rung2_enabled: bool = True
    ranking_checks_enabled: bool = True
    canary_enabled: bool = True

    def __post_init__(self):
        if not 0.0 <= self.tau_cov <= 1.0:
            raise ValueError("tau_cov must be in [0, 1]")
        if self.k_min < 0 or self.k_max < self.k_min:
            raise ValueError("need 0 <= k_min <= k_max")
        if self.v_tol <= 0:
            raise ValueError("v_tol must be positive")
        if self.ranking_depth < 1:
            raise ValueError("ranking_depth must be at least 1")
        if self.epsilon_guard < 0:
            raise ValueError("epsilon_guard must be non-negative")
        if self.exploration_rate != 0.0 and not 0.01 <= self.exploration_rate <= 0.05:
            raise ValueError("exploration_rate must be 0 or in [0.01, 0.05]")
        if self.exponent_mode not in (2, 3):
            raise ValueError("exponent_mode must be 2 or 3")
        if self.greedy_value_budget is not None and self.greedy_value_budget < 0:
            raise ValueError("greedy_value_budget must be non-negative")


# -- kernels (_kernels/pure.py) --------------------------------------------

def block_logmass(scores, bounds):
    """(block_max, block_sum, log_mass) in fp64 (pure.py:16-36)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    nb = bounds.shape[0] - 1
    if nb <= 0:
        e = np.empty(0)
        return e, e.copy(), e.copy()
    starts = bounds[:-1]
    bmax = np.maximum.reduceat(scores, starts)
    bsum = np.add.reduceat(np.exp(scores - np.repeat(bmax, np.diff(bounds))), starts)
    return bmax, bsum, bmax + np.log(bsum)


def fused_attend_f32(scores, values, bounds):
    """Blockwise online softmax with float32 (m, l, o) (pure.py:39-66)."""
    s32 = np.ascontiguousarray(scores, dtype=np.float32)
    v32 = np.ascontiguousarray(values, dtype=np.float32)
    m = np.float32(-np.inf)
    l = np.float32(0.0)
    o = np.zeros(v32.shape[1], dtype=np.float32)
    for i in range(len(bounds) - 1):
        lo, hi = bounds[i], bounds[i + 1]
        seg = s32[lo:hi]
        m_new = max(m, np.float32(seg.max()))
        p = np.exp(seg - m_new)
        scale = np.exp(np.float32(m - m_new))
        l = np.float32(l * scale + p.sum(dtype=np.float32))
        o = o * scale + p @ v32[lo:hi]
        m = m_new
    return o / l, m, l


def _lse(x):
    """attention.py:41-45."""
    if x.size == 0:
        return -np.inf
    m = x.max()
    return float(m + np.log(np.sum(np.exp(x - m))))


def _score(rows, q, d):
    """Canonical fp64 scoring rows @ q / sqrt(d) (attention.py:34-38)."""
    if rows.shape[0] == 0:
        return np.empty(0)
    return rows @ q / np.sqrt(d)


def _bounds(nb, bsz, plen=0):
    b = [i * bsz for i in range(nb + 1)]
    if plen:
        b.append(b[-1] + plen)
    return np.asarray(b, dtype=np.int64)


# -- Phase 1 and selection (attention.py:89-203) ---------------------------

def phase1(q, kv):
    """Score every full block on its reconstruction; partial on originals."""
    if kv.num_tokens == 0:
        raise ValueError("cannot score an empty cache")
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    tok = _score(kv.deq_key_rows(), q, kv.head_dim)
    bmax, bsum, lm = block_logmass(tok, _bounds(kv.num_blocks, kv.block_size))
    ps = _score(kv.partial_keys(), q, kv.head_dim)
    plm = None
    if ps.size:
        plm = float(block_logmass(ps, np.asarray([0, ps.size]))[2][0])
    return {"scores": tok, "block_max": bmax, "block_sum": bsum,
            "log_mass": lm, "partial_scores": ps, "partial_log_mass": plm}


def delta_bound(q, kv):
    """Delta_h = max_b sum_c |q_c| scale_bc / (2 sqrt d) (certifier.py:89-104)."""
    if not kv.num_blocks:
        return np.empty(0), 0.0
    aq = np.abs(np.asarray(q, dtype=np.float64).reshape(-1))
    per = np.asarray([float(aq @ s) for s in kv.key_scales_used()])
    per = per / (2.0 * np.sqrt(kv.head_dim))
    return per, float(per.max())


def _cut(k, order, masses):
    promoted = np.sort(order[:k]).astype(np.int64)
    tail = order[k:]
    est_tail = float(masses[tail].sum()) if tail.size else 0.0
    return promoted, est_tail


def select_blocks(p1, tau, kmin, kmax):
    """Adaptive top-K (attention.py:146-189); returns a decision dict."""
    nb = p1["log_mass"].shape[0]
    lm_all = list(p1["log_mass"])
    if p1["partial_log_mass"] is not None:
        lm_all.append(p1["partial_log_mass"])
    lse = _lse(np.asarray(lm_all, dtype=np.float64))
    masses = np.exp(p1["log_mass"] - lse)
    pmass = (float(np.exp(p1["partial_log_mass"] - lse))
             if p1["partial_log_mass"] is not None else 0.0)
    if nb == 0:
        return {"order": np.empty(0, np.int64), "masses": masses,
                "partial_mass": pmass, "k_coverage": 0, "k_star": 0,
                "clamped": False, "promoted": np.empty(0, np.int64),
                "est_tail_mass": 0.0}
    order = np.lexsort((np.arange(nb), -masses))
    cum = pmass + np.cumsum(masses[order])
    hit = np.nonzero(cum >= tau)[0]
    kcov = int(hit[0]) + 1 if hit.size else nb
    k = min(max(kcov, kmin), min(kmax, nb))
    promoted, est_tail = _cut(k, order, masses)
    return {"order": order, "masses": masses, "partial_mass": pmass,
            "k_coverage": kcov, "k_star": k, "clamped": k != kcov,
            "promoted": promoted, "est_tail_mass": est_tail}


def expand(dec, k_new):
    """Rung 1: re-cut at min(k_new, N_B) along the same order (attention.py:192-203)."""
    nb = dec["masses"].shape[0]
    k_new = min(int(k_new), nb)
    out = dict(dec)
    out["k_star"] = k_new
    out["promoted"], out["est_tail_mass"] = _cut(k_new, dec["order"], dec["masses"])
    return out


def value_promotions(masses, etas, policy):
    """Rung 2 (fallback.py:141-161)."""
    c = np.asarray(masses, dtype=np.float64) * np.asarray(etas, dtype=np.float64)
    if policy.greedy_value_budget is None:
        return np.nonzero(c > policy.v_tol)[0].astype(np.int64)
    order = np.lexsort((np.arange(c.shape[0]), -c))
    resid = float(c.sum())
    chosen = []
    for b in order:
        if resid <= policy.greedy_value_budget:
            break
        chosen.append(int(b))
        resid -= float(c[b])
    return np.asarray(sorted(chosen), dtype=np.int64)


# -- Phase 2, dense (attention.py:227-342) ---------------------------------

def phase2(q, kv, promoted, vprom, key_payloads=None, value_payloads=None):
    """Mask-gated single pass: originals for promoted keys / values."""
    if kv.num_tokens == 0:
        raise ValueError("cannot attend over an empty cache")
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    nb, bsz, d = kv.num_blocks, kv.block_size, kv.head_dim
    vset = set(int(b) for b in vprom)

    def paged(pl, b, kind):
        if b not in pl:
            raise PagingFault(f"promoted block {b} ({kind}) was never paged in")
        return pl[b]

    tok = _score(kv.deq_key_rows(), q, d)
    for b in sorted(int(x) for x in promoted):
        rows = (kv.orig_keys32(b) if key_payloads is None
                else paged(key_payloads, b, "keys"))
        tok[b * bsz:(b + 1) * bsz] = _score(rows.astype(np.float64), q, d)
    vrows = []
    for b in range(nb):
        if b in vset:
            vrows.append(kv.orig_values32(b) if value_payloads is None
                         else paged(value_payloads, b, "values"))
        else:
            vrows.append(kv.deq_value_block32(b))
    ps = _score(kv.partial_keys(), q, d)
    if ps.size:
        vrows.append(kv.partial_values().astype(np.float32))
    all_s = np.concatenate([tok, ps])
    vals = (np.concatenate(vrows, axis=0, dtype=np.float32) if vrows
            else np.empty((0, d), dtype=np.float32))
    bnd = _bounds(nb, bsz, ps.size)
    out, m, l = fused_attend_f32(all_s.astype(np.float32), vals, bnd)
    lm_all = block_logmass(all_s, bnd)[2]
    masses_all = np.exp(lm_all - _lse(lm_all))
    if ps.size:
        bm, pm, lm = masses_all[:-1], float(masses_all[-1]), lm_all[:-1]
    else:
        bm, pm, lm = masses_all, 0.0, lm_all
    return {"output": out, "block_masses": bm, "partial_mass": pm,
            "log_mass": lm, "scores": all_s, "m": m, "l": l,
            "promoted_log_mass": {int(b): float(lm[b]) for b in sorted(int(x) for x in promoted)}}


def dense_output(q, kv):
    """Exact two-pass softmax over the originals in fp64 (attention.py:327-342)."""
    if kv.num_tokens == 0:
        raise ValueError("cannot attend over an empty cache")
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    s = np.concatenate([_score(kv.tier2_key_rows(), q, kv.head_dim),
                        _score(kv.partial_keys(), q, kv.head_dim)])
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ np.concatenate([kv.tier2_value_rows(), kv.partial_values()], axis=0)


# -- certificate (certifier.py:135-212) -------------------------------------

def e_key_bound(v_max, delta, tail, mode):
    e = float(mode)
    return 2.0 * float(v_max) * math.exp(e * delta) * float(tail) * (math.exp(2.0 * delta) - 1.0)


def e_val(block_masses, etas, vprom):
    keep = np.ones(block_masses.shape[0], dtype=bool)
    keep[np.asarray(list(vprom), dtype=np.int64)] = False
    return float(block_masses[keep] @ etas[keep])


def _top_r(lmap, r):
    """fallback.py:164-167 / harness.py:181-183: ties toward the lower index."""
    items = sorted(lmap.items(), key=lambda kv: (-kv[1], kv[0]))
    return items[:r]


# -- the step (harness.py:186-300) ------------------------------------------

def decode_step(q, kv, policy, key_scratch=None, value_scratch=None,
                rng=None, head=0, step=0):
    """One q-head through the fixed rung order; returns a flat result dict."""
    p1 = phase1(q, kv)
    _, delta = delta_bound(q, kv)
    events = []
    dec = select_blocks(p1, policy.tau_cov, policy.k_min, policy.k_max)
    k0 = dec["k_star"]
    r1 = False
    if policy.rung1_enabled:
        wide = expand(dec, 2 * dec["k_star"])
        if wide["k_star"] != dec["k_star"]:
            r1 = True
            events.append((1, "coverage_expand"))
        dec = wide
    vprom = np.empty(0, np.int64)
    if policy.rung2_enabled and kv.num_blocks:
        vprom = value_promotions(dec["masses"], kv.etas(), policy)
        if vprom.size:
            events.append((2, "value_tol"))
    pages = {}
    kpl = vpl = None
    if key_scratch is not None:
        rep = promote(key_scratch, kv, dec["promoted"], "keys")
        pages["keys"] = rep
        kpl = rep["payloads"]
    if value_scratch is not None:
        rep = promote(value_scratch, kv, vprom, "values")
        pages["values"] = rep
        vpl = rep["payloads"]
    att = phase2(q, kv, dec["promoted"], vprom, kpl, vpl)

    promoted = dec["promoted"]
    r3 = False
    rank_ok = bound_ok = True
    r = policy.ranking_depth
    if policy.ranking_checks_enabled and promoted.size:
        if promoted.size < r:
            r3 = True
            rank_ok = False
            events.append((3, "ranking_disagree"))
        else:
            quant_lm = {int(b): float(p1["log_mass"][b]) for b in promoted}
            ref_top = [b for b, _ in _top_r(att["promoted_log_mass"], r)]
            q_top = [b for b, _ in _top_r(quant_lm, r)]
            if ref_top != q_top:
                r3 = True
                rank_ok = False
                events.append((3, "ranking_disagree"))
            mask = np.ones(kv.num_blocks, dtype=bool)
            mask[promoted] = False
            tail_lm = p1["log_mass"][mask]
            rth = _top_r(att["promoted_log_mass"], r)[-1][1]
            if tail_lm.size and not (tail_lm.max() + delta <= rth):
                r3 = True
                bound_ok = False
                events.append((3, "boundary"))
    r4 = False
    canary_gap = 0.0
    if policy.canary_enabled and promoted.size:
        bsz = kv.block_size
        idx = np.concatenate([np.arange(b * bsz, (b + 1) * bsz) for b in promoted])
        canary_gap = float(np.abs(att["scores"][idx] - p1["scores"][idx]).max())
        if not canary_gap <= delta + policy.epsilon_guard:
            r4 = True
            events.append((4, "canary"))
    if policy.exploration_rate > 0 and rng is not None and kv.num_blocks:
        mask = np.ones(kv.num_blocks, dtype=bool)
        mask[promoted] = False
        cands = np.nonzero(mask)[0]
        count = min(len(cands), int(round(policy.exploration_rate * kv.num_blocks)))
        passed = True
        nbytes = 0
        if count:
            chosen = rng.choice(len(cands), size=count, replace=False)
            qv = np.asarray(q, dtype=np.float64).reshape(-1)
            for pos in sorted(int(c) for c in chosen):
                b = int(cands[pos])
                ref = _score(kv.orig_keys32(b).astype(np.float64), qv, kv.head_dim)
                qs = p1["scores"][b * kv.block_size:(b + 1) * kv.block_size]
                nbytes += kv.block_size * kv.head_dim * 2
                if not float(np.abs(ref - qs).max()) <= delta + policy.epsilon_guard:
                    passed = False
        pages["exploration"] = {"hits": 0, "misses": count, "bytes": nbytes}
        if not passed:
            r4 = True
            events.append((4, "canary"))

    if r4:
        kind, out = DENSE_ALL, dense_output(q, kv)
    elif r3:
        kind, out = DENSE_HEAD, dense_output(q, kv)
    else:
        kind, out = QUANTIZED, att["output"].astype(np.float64)
    tail = dec["est_tail_mass"]
    return {
        "output": out, "quant_output": att["output"].astype(np.float64),
        "kind": kind, "delta_h": float(delta),
        "e_key_tight": e_key_bound(kv.v_max, delta, tail, 2),
        "e_key_impl": e_key_bound(kv.v_max, delta, tail, 3),
        "e_val": e_val(att["block_masses"], kv.etas(), vprom),
        "est_tail_mass": float(tail), "v_max": float(kv.v_max),
        "k_star": int(dec["k_star"]), "k_star_pre_rung1": int(k0),
        "k_coverage": int(dec["k_coverage"]), "clamped": bool(dec["clamped"]),
        "flags": (r1, bool(vprom.size), r3, r4), "events": events,
        "rank_ok": rank_ok, "boundary_ok": bound_ok, "canary_gap": canary_gap,
        "promoted": promoted, "value_promotions": vprom, "order": dec["order"],
        "masses": dec["masses"], "partial_mass": dec["partial_mass"],
        "log_mass_p1": p1["log_mass"], "log_mass_p2": att["log_mass"],
        "block_masses_p2": att["block_masses"], "etas": kv.etas(), "pages": pages,
        "head": head, "step": step,
    }


# -- workloads and the step loop (harness.py:93-163, 339-394) ---------------

def _philox(seed, purpose):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, purpose))))


def make_workload(kind="gaussian", n_tokens=1024, head_dim=64, block_size=16,
                  group_size=16, query_heads=1, kv_heads=1, steps=8, seed=0,
                  ingest_binary16=False, narrow=False, build_caches=True):
    """Seeded workload identical to generate_workload (harness.py:97-163).

    Returns raw arrays (keys/values f64 [kv, total, d], queries f64
    [steps, hq, d]) plus, when ``build_caches``, one OracleKV per KV head
    prefilled with the first n_tokens.
    """
    if kind not in ("gaussian", "sink", "needle", "near_tie"):
        raise ValueError(f"unknown workload kind {kind!r}")
    d = head_dim
    rng = _philox(seed, 0)
    total = n_tokens + steps
    keys = rng.standard_normal((kv_heads, total, d))
    values = rng.standard_normal((kv_heads, total, d))
    queries = rng.standard_normal((steps, query_heads, d))
    kappa = 3.0
    dirs = np.empty((kv_heads, d))
    for kv in range(kv_heads):
        w = rng.standard_normal(d)
        dirs[kv] = w / np.linalg.norm(w)
    gfac = query_heads // kv_heads
    if kind != "gaussian":
        for h in range(query_heads):
            queries[:, h, :] += kappa * dirs[h // gfac]
    if kind == "sink":
        planted = 2.0 * np.sqrt(d) / kappa
        span = min(block_size, n_tokens)
        for kv in range(kv_heads):
            keys[kv, :span] = planted * dirs[kv] + 0.1 * keys[kv, :span]
    elif kind == "needle":
        planted = 2.5 * np.sqrt(d) / kappa
        for kv in range(kv_heads):
            keys[kv, n_tokens // 2] = planted * dirs[kv]
    elif kind == "near_tie":
        if n_tokens < 2 * block_size:
            raise ValueError("near_tie needs at least two full blocks")
        planted = 2.0 * np.sqrt(d) / kappa
        b = block_size
        for kv in range(kv_heads):
            base = planted * dirs[kv] + 0.5 * keys[kv, :b]
            keys[kv, :b] = base
            keys[kv, b:2 * b] = base + 1e-4 * rng.standard_normal((b, d))
    caches = []
    if build_caches:
        for kv in range(kv_heads):
            c = OracleKV(block_size, d, group_size, ingest_binary16=ingest_binary16,
                         narrow=narrow)
            c.append_tokens(keys[kv, :n_tokens], values[kv, :n_tokens])
            caches.append(c)
    return {"keys": keys, "values": values, "queries": queries,
            "new_keys": np.swapaxes(keys[:, n_tokens:], 0, 1).astype(np.float32),
            "new_values": np.swapaxes(values[:, n_tokens:], 0, 1).astype(np.float32),
            "caches": caches, "group_factor": gfac, "steps": steps,
            "query_heads": query_heads, "kv_heads": kv_heads, "head_dim": d,
            "seed": seed}


def run_workload(wl, policy, key_capacity=2048, value_capacity=2048, layers=1):
    """harness.py:339-394: per step every q-head, step-wide Rung 4, record,
    then append one token per KV head."""
    caches = wl["caches"]
    ks = [OracleScratch(key_capacity) for _ in caches]
    vs = [OracleScratch(value_capacity) for _ in caches]
    rng = _philox(wl["seed"], 1)
    gfac = wl["group_factor"]
    records, results = [], []
    for step in range(wl["steps"]):
        kb = [(s.hits, s.misses, s.bytes_paged_in) for s in ks]
        vb = [(s.hits, s.misses, s.bytes_paged_in) for s in vs]
        res = []
        for h in range(wl["query_heads"]):
            kv = h // gfac
            res.append(decode_step(wl["queries"][step, h], caches[kv], policy,
                                   ks[kv], vs[kv], rng, h, step))
        staging = 0
        if any(r["flags"][3] for r in res):
            staging = int(sum(2 * c.num_tokens * c.head_dim * 2 for c in caches))
            for h, r in enumerate(res):
                r["output"] = dense_output(wl["queries"][step, h], caches[h // gfac])
                r["kind"] = DENSE_ALL
        records.append(step_record(step, res, gfac, caches, _delta(ks, kb),
                                   _delta(vs, vb), staging))
        results.append(res)
        for kv, c in enumerate(caches):
            c.append_token(wl["new_keys"][step, kv], wl["new_values"][step, kv])
    return {"records": records, "results": results,
            "summary": aggregate(records, wl["query_heads"], layers)}


def _delta(scr, before):
    h = sum(s.hits for s in scr) - sum(b[0] for b in before)
    m = sum(s.misses for s in scr) - sum(b[1] for b in before)
    p = sum(s.bytes_paged_in for s in scr) - sum(b[2] for b in before)
    return {"hits": h, "misses": m, "hit_rate": h / (h + m) if h + m else 0.0,
            "bytes_paged_in": p}


def certificate_dict(r):
    """Certificate.to_dict (certifier.py:83-98)."""
    dense = r["kind"] != QUANTIZED
    f = r["flags"]
    return {"head": r["head"], "step": r["step"], "delta_h": r["delta_h"],
            "e_key_tight": r["e_key_tight"], "e_key_impl": r["e_key_impl"],
            "e_val": r["e_val"], "est_tail_mass": r["est_tail_mass"],
            "v_max": r["v_max"], "k_star": r["k_star"],
            "returned_kind": r["kind"],
            "returned_e_key": 0.0 if dense else r["e_key_impl"],
            "returned_e_val": 0.0 if dense else r["e_val"],
            "rung_flags": {"rung1": f[0], "rung2": f[1], "rung3": f[2], "rung4": f[3]}}


def step_record(step, res, gfac, caches, kscr, vscr, staging):
    """harness.py:397-447."""
    certs = [certificate_dict(r) for r in res]
    events = [(rung, cause, r["head"]) for r in res for rung, cause in r["events"]]
    rc = {f"rung{i}": 0 for i in (1, 2, 3, 4)}
    cc = {}
    for rung, cause, _ in events:
        rc[f"rung{rung}"] += 1
        cc[cause] = cc.get(cause, 0) + 1
    union = {}
    for h, r in enumerate(res):
        union.setdefault(h // gfac, set()).update(int(b) for b in r["promoted"])
    fr = [len(union.get(kv, ())) / c.num_blocks for kv, c in enumerate(caches) if c.num_blocks]
    paged = sum(p["bytes"] for r in res for p in r["pages"].values())

    def mean(xs):
        return float(np.mean(xs)) if xs else 0.0

    def mx(xs):
        return float(np.max(xs)) if xs else 0.0

    return {
        "step": step,
        "e_key_step_mean": mean([c["e_key_impl"] for c in certs]),
        "e_key_step_max": mx([c["e_key_impl"] for c in certs]),
        "e_key_step_mean_returned": mean([c["returned_e_key"] for c in certs]),
        "e_key_step_max_returned": mx([c["returned_e_key"] for c in certs]),
        "e_val_step_mean": mean([c["e_val"] for c in certs]),
        "e_val_step_max": mx([c["e_val"] for c in certs]),
        "e_val_step_mean_returned": mean([c["returned_e_val"] for c in certs]),
        "e_val_step_max_returned": mx([c["returned_e_val"] for c in certs]),
        "k_star_mean": mean([c["k_star"] for c in certs]),
        "est_tail_mass_mean": mean([c["est_tail_mass"] for c in certs]),
        "delta_h_max": mx([c["delta_h"] for c in certs]),
        "rung_counts": rc, "cause_counts": cc,
        "events": [{"rung": a, "head": h, "step": step, "cause": b} for a, b, h in events],
        "certificates": certs,
        "key_scratch": kscr, "value_scratch": vscr,
        "bytes_paged_in": paged, "rung4_staging_bytes": staging,
        "union_fraction_mean": mean(fr),
    }


def aggregate(records, query_heads, layers=1):
    """harness.py:450-499."""
    steps = len(records)
    hs = steps * query_heads * layers
    rt = {f"rung{i}": 0 for i in (1, 2, 3, 4)}
    ct = {}
    for rec in records:
        for k, v in rec["rung_counts"].items():
            rt[k] += v
        for k, v in rec["cause_counts"].items():
            ct[k] = ct.get(k, 0) + v
    certs = [c for rec in records for c in rec["certificates"]]

    def stats(key):
        vals = [c[key] for c in certs]
        return {"mean": float(np.mean(vals)) if vals else 0.0,
                "max": float(np.max(vals)) if vals else 0.0}

    dense = sum(1 for c in certs if c["returned_kind"] != QUANTIZED)
    return {
        "steps": steps, "head_steps": hs, "layers": layers,
        "rung_counts": rt, "cause_counts": ct,
        "rates": {"rung3_per_head_step": rt["rung3"] / hs if hs else 0.0,
                  "rung4_per_step": rt["rung4"] / steps if steps else 0.0,
                  "dense_fraction": dense / hs if hs else 0.0},
        "e_key_candidate": stats("e_key_impl"),
        "e_key_tight_candidate": stats("e_key_tight"),
        "e_key_returned": stats("returned_e_key"),
        "e_val": stats("e_val"), "e_val_returned": stats("returned_e_val"),
        "k_star_mean": float(np.mean([c["k_star"] for c in certs])) if certs else 0.0,
        "est_tail_mass_mean": float(np.mean([c["est_tail_mass"] for c in certs])) if certs else 0.0,
        "bytes_paged_in_total": sum(r["bytes_paged_in"] for r in records),
        "rung4_staging_bytes_total": sum(r["rung4_staging_bytes"] for r in records),
        "union_fraction_mean": float(np.mean([r["union_fraction_mean"] for r in records])) if records else 0.0,
    }


def storage_table(head_dim, block_size, group_size):
    """Per-token Tier-1 byte components (cache.py:360-383)."""
    d, b, g = float(head_dim), float(block_size), float(group_size)
    total = d + 8.0 * d / b + d / 2.0 + 4.0 * d / g
    return {"key_codes_bytes": d, "key_metadata_bytes": 8.0 * d / b,
            "value_codes_bytes": d / 2.0, "value_metadata_bytes": 4.0 * d / g,
            "annotation_bytes": 4.0 / b, "tier1_total_bytes": total,
            "tier1_exact_bytes": total + 4.0 / b, "dense_bytes": 4.0 * d,
            "tier1_ratio": total / (4.0 * d)}
