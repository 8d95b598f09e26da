"""Freeze golden vectors from the REAL reference package.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py

It imports ``certkv`` from /root/reference/pkg/src (pure-NumPy kernel
backend, the deterministic one), runs quantizer known-answer inputs, random
and adversarial blocks, and small end-to-end ``run_workload`` runs, and
writes ``tests/golden/*.npz``.  ``tests/test_oracle_golden.py`` pins the
oracle restatement against these files; nothing at GPU-test time reads the
reference itself.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, os.path.dirname(os.path.dirname(HERE)))  # the repo root (oracle.margins)
os.environ["CERTKV_KERNEL"] = "pure"

import certkv  # noqa: E402
from certkv import quantizer  # noqa: E402
from certkv.fallback import PolicyConfig  # noqa: E402
from certkv.harness import WorkloadConfig, generate_workload, run_workload  # noqa: E402


def _blocks(rng):
    """Key/value blocks (16 x 128, fp16-exact) covering the fit edge cases."""
    out = []
    for i in range(40):
        scale = 10.0 ** rng.uniform(-3, 3)
        out.append(rng.standard_normal((16, 128)) * scale)
    b = rng.standard_normal((16, 128))
    b[:, 3] = 0.75                      # constant channel
    b[:, 7] *= 1000.0                   # outlier channel
    b[:, 9] = 1e-4 * b[:, 9] + 12.0     # narrow channel on a large offset
    b[0, 11] = 1e4                      # single spike
    out.append(b)
    b = np.zeros((16, 128))             # all-zero block
    out.append(b)
    b = np.repeat(np.arange(16.0)[:, None], 128, axis=1) * 0.5  # exact grid
    out.append(b)
    b = rng.integers(-3, 4, (16, 128)).astype(np.float64) * 0.125  # ties
    out.append(b)
    return np.stack([x.astype(np.float16).astype(np.float64) for x in out])


def quantizer_golden():
    rng = np.random.default_rng(20260517)
    blocks = _blocks(rng)
    kc, ks, ko, vc, vs, vo, eta, nu = [], [], [], [], [], [], [], []
    for blk in blocks:
        k = quantizer.quantize_key_block(blk)
        v, ann = quantizer.quantize_value_block(blk, 16)
        kc.append(k.codes); ks.append(k.scales); ko.append(k.offsets)
        vc.append(v.codes); vs.append(v.group_scales); vo.append(v.group_offsets)
        eta.append(ann.eta); nu.append(ann.nu)
    # small-shape KATs straight from the reference test file's inputs
    two = quantizer.quantize_key_block(np.array([[-1.0], [1.0]]))
    grp, gann = quantizer.quantize_value_block(np.array([[0.0, 1.5]]), 2)
    np.savez_compressed(
        os.path.join(HERE, "quantizer.npz"),
        blocks=blocks.astype(np.float16),
        kcodes=np.stack(kc), kscale=np.stack(ks), koffset=np.stack(ko),
        vcodes=np.stack(vc), vscale=np.stack(vs), voffset=np.stack(vo),
        eta=np.asarray(eta), nu=np.asarray(nu),
        kat_two_codes=two.codes, kat_two_scale=two.scales, kat_two_offset=two.offsets,
        kat_grp_codes=grp.codes, kat_grp_scale=grp.group_scales,
        kat_grp_offset=grp.group_offsets, kat_grp_eta=np.asarray(gann.eta))


RUNS = [
    # name, workload kwargs, policy kwargs, capacities
    ("gauss", dict(kind="gaussian", n_tokens=520, head_dim=128, query_heads=8,
                   kv_heads=2, steps=3, seed=0), dict(exploration_rate=0.0), (2048, 2048)),
    ("gauss_small_kmax", dict(kind="gaussian", n_tokens=1030, head_dim=128, query_heads=8,
                              kv_heads=2, steps=3, seed=3),
     dict(exploration_rate=0.0, k_max=8), (24, 24)),
    ("sink", dict(kind="sink", n_tokens=600, head_dim=128, query_heads=8,
                  kv_heads=2, steps=3, seed=1), dict(exploration_rate=0.0), (2048, 2048)),
    ("needle", dict(kind="needle", n_tokens=777, head_dim=128, query_heads=8,
                    kv_heads=2, steps=2, seed=2), dict(exploration_rate=0.0, k_max=16), (2048, 2048)),
    ("near_tie", dict(kind="near_tie", n_tokens=640, head_dim=128, query_heads=8,
                      kv_heads=2, steps=2, seed=5), dict(exploration_rate=0.0, k_max=4), (2048, 2048)),
    ("explore", dict(kind="gaussian", n_tokens=900, head_dim=128, query_heads=4,
                     kv_heads=1, steps=2, seed=7), dict(exploration_rate=0.02, k_max=8), (64, 64)),
    ("tight_vtol", dict(kind="sink", n_tokens=700, head_dim=128, query_heads=8,
                        kv_heads=2, steps=2, seed=11), dict(exploration_rate=0.0, v_tol=0.01), (2048, 2048)),
    ("d64", dict(kind="gaussian", n_tokens=333, head_dim=64, query_heads=4,
                 kv_heads=2, steps=2, seed=9), dict(exploration_rate=0.0, k_max=4), (8, 8)),
    # BASELINE.json C1 exactly: the reference's own CPU-runnable case
    ("c1", dict(kind="gaussian", n_tokens=4096, head_dim=128, query_heads=32, kv_heads=8,
                steps=16, seed=0), dict(exploration_rate=0.0), (2048, 2048)),
    # decisions away from "everything promoted": a real K* cut, value promotions
    # with an evicting scratch, greedy Rung 2
    ("gauss16k", dict(kind="gaussian", n_tokens=16384, head_dim=128, query_heads=4,
                      kv_heads=1, steps=3, seed=12), dict(exploration_rate=0.0), (2048, 2048)),
    ("sink8k_vtol", dict(kind="sink", n_tokens=8192, head_dim=128, query_heads=8, kv_heads=2,
                         steps=3, seed=13), dict(exploration_rate=0.0, v_tol=0.002), (512, 256)),
    ("greedy", dict(kind="sink", n_tokens=2000, head_dim=128, query_heads=4, kv_heads=1,
                    steps=2, seed=14), dict(exploration_rate=0.0, greedy_value_budget=0.05),
     (2048, 2048)),
]

# runs whose outputs are frozen as float32 (size; the tests compare at >= 1e-6)
F32_OUTPUTS = {"c1"}


def _margins(r, phase1, cache, policy):
    """Threshold distances of the reference's own decisions (oracle/margins.py),
    computed from the reference objects of this head-step."""
    from oracle.margins import as_row, decision_margins
    dec, att = r.decision, r.attend
    F = sorted(dec.promoted)
    gap = 0.0
    if F:
        bs = cache.block_size
        idx = np.concatenate([np.arange(b * bs, (b + 1) * bs) for b in F])
        gap = float(np.abs(att.token_scores[idx] - phase1.token_scores[idx]).max())
    m = decision_margins(
        dec.normalized_masses, dec.order, dec.k_star, dec.k_coverage, dec.partial_mass,
        cache.etas(), phase1.log_mass, dict(att.promoted_log_masses), r.delta_h, gap,
        tau_cov=policy.tau_cov, k_min=policy.k_min, k_max=policy.k_max, v_tol=policy.v_tol,
        greedy_value_budget=policy.greedy_value_budget, ranking_depth=policy.ranking_depth,
        epsilon_guard=policy.epsilon_guard, rung2_enabled=policy.rung2_enabled,
        ranking_checks_enabled=policy.ranking_checks_enabled,
        canary_enabled=policy.canary_enabled)
    return as_row(m)


def _digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def workload_golden():
    manifest = {}
    for name, wkw, pkw, (kc, vc) in RUNS:
        cfg = WorkloadConfig(ingest_binary16=True, **wkw)
        wl = generate_workload(cfg)
        # digests pin that the oracle regenerates identical inputs
        keys_digest = _digest(np.stack([np.concatenate(c.tier2_keys + [c.partial_key_matrix().astype(np.float32)]) for c in wl.caches]))
        q_digest = _digest(wl.queries)
        policy = PolicyConfig(**pkw)
        res = run_workload(wl, policy, key_capacity=kc, value_capacity=vc)
        arrays = {}
        for rec in res.step_records:
            s = rec["step"]
            for c in rec["certificates"]:
                arrays.setdefault("cert", []).append(
                    [s, c["head"], c["delta_h"], c["e_key_tight"], c["e_key_impl"],
                     c["e_val"], c["est_tail_mass"], c["v_max"], c["k_star"],
                     ["quantized", "dense_per_head", "dense_all_heads"].index(c["returned_kind"]),
                     c["rung_flags"]["rung1"], c["rung_flags"]["rung2"],
                     c["rung_flags"]["rung3"], c["rung_flags"]["rung4"]])
        # per head-step outputs and promoted sets via a replay with hooks
        outs, prom, vprom, margins = [], [], [], []
        wl2 = generate_workload(cfg)
        from certkv.attention import phase1_score
        from certkv.cache import ScratchCache
        from certkv.harness import run_decode_step, _rng
        ks = [ScratchCache(kc) for _ in wl2.caches]
        vs = [ScratchCache(vc) for _ in wl2.caches]
        rng = _rng(cfg.seed, 1)
        for step in range(cfg.steps):
            step_res = []
            for h in range(cfg.query_heads):
                kv = cfg.kv_index(h)
                r = run_decode_step(wl2.queries[step, h], wl2.caches[kv], policy,
                                    ks[kv], vs[kv], rng, h, step)
                step_res.append(r)
                margins.append(_margins(r, phase1_score(wl2.queries[step, h], wl2.caches[kv]),
                                        wl2.caches[kv], policy))
                prom.append(sorted(r.decision.promoted))
                vprom.append(sorted(r.value_promotions))
            if any(r.rung4_requested for r in step_res):
                for h, r in enumerate(step_res):
                    r.output = certkv.dense_attention(wl2.queries[step, h],
                                                      wl2.caches[cfg.kv_index(h)])
            outs.extend(r.output for r in step_res)
            for kv, cache in enumerate(wl2.caches):
                cache.append_token(wl2.new_keys[step, kv], wl2.new_values[step, kv])
        maxp = max(1, max(len(p) for p in prom))
        maxv = max(1, max(len(v) for v in vprom))
        pm = np.full((len(prom), maxp), -1, np.int64)
        vm = np.full((len(vprom), maxv), -1, np.int64)
        for i, p in enumerate(prom):
            pm[i, :len(p)] = p
        for i, v in enumerate(vprom):
            vm[i, :len(v)] = v
        recs = json.dumps(res.step_records, sort_keys=True)
        summ = json.dumps(res.summary, sort_keys=True)
        np.savez_compressed(
            os.path.join(HERE, f"run_{name}.npz"),
            cert=np.asarray(arrays["cert"], dtype=np.float64),
            outputs=np.asarray(outs, dtype=np.float32 if name in F32_OUTPUTS else np.float64),
            margins=np.asarray(margins, dtype=np.float64), promoted=pm, value_promotions=vm,
            records_json=np.asarray(recs), summary_json=np.asarray(summ))
        manifest[name] = {"workload": wkw, "policy": pkw, "capacities": [kc, vc],
                          "keys_digest": keys_digest, "queries_digest": q_digest}
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


def fault_golden():
    """verification.py:405-428 sink cache + offset corruption -> canary Rung 4."""
    from certkv.verification import build_sink_cache, corrupt_block_offset
    from certkv.harness import run_decode_step
    cache, query = build_sink_cache(0)
    pol = PolicyConfig(exploration_rate=0.0)
    honest = run_decode_step(query, cache, pol)
    keys = np.concatenate(cache.tier2_keys)
    vals = np.concatenate(cache.tier2_values)
    corrupt_block_offset(cache, 0, query)
    tripped = run_decode_step(query, cache, pol)
    np.savez_compressed(
        os.path.join(HERE, "fault.npz"), keys=keys, values=vals, query=query,
        honest_output=honest.output, honest_events=np.asarray(
            [[e.rung, ["coverage_expand", "value_tol", "ranking_disagree", "boundary",
                       "canary", "precondition"].index(e.cause)] for e in honest.events] or
            np.zeros((0, 2)), dtype=np.int64),
        tripped_output=tripped.output, tripped_kind=np.asarray(tripped.certificate.returned_kind),
        tripped_rung4=np.asarray(any(e.rung == 4 for e in tripped.events)))


TELEMETRY_MANIFEST = {
    "workload": {"kind": "gaussian", "n_tokens": 2000, "head_dim": 128, "query_heads": 8,
                 "kv_heads": 2, "steps": 3, "ingest_binary16": True},
    "policy": {"exploration_rate": 0.0, "k_max": 24},
    "scratch": {"key_capacity": 64, "value_capacity": 64},
    "seed": 17,
}


def telemetry_golden():
    """The reference CLI's bound report (cli.py:98-117, ``certkv run``) for a fixed
    manifest: tests/golden/telemetry_manifest.json -> telemetry_ref.jsonl."""
    from certkv.cli import RunManifest, cmd_run
    cfg = os.path.join(HERE, "telemetry_manifest.json")
    with open(cfg, "w") as f:
        json.dump(TELEMETRY_MANIFEST, f, indent=1, sort_keys=True)
    # the manifest path is echoed into the header: record it relative to the repo root
    cwd = os.getcwd()
    os.chdir(os.path.dirname(os.path.dirname(HERE)))
    try:
        cmd_run(RunManifest(config_path="tests/golden/telemetry_manifest.json",
                            out_path=os.path.join(HERE, "telemetry_ref.jsonl")))
    finally:
        os.chdir(cwd)


if __name__ == "__main__":
    quantizer_golden()
    workload_golden()
    fault_golden()
    telemetry_golden()
    print("golden vectors written to", HERE)
