"""Host-side logic of the drop-in API (no GPU): policy validation, event
decoding, certificate views, storage accounting and the telemetry schema,
checked against the oracle restatement."""

import numpy as np
import pytest

from paper_2605_20868_b200 import _lib
from paper_2605_20868_b200.harness import aggregate_telemetry, step_record, WorkloadConfig, synth_arrays
from paper_2605_20868_b200.policy import (Certificate, FallbackEvent, PolicyConfig, RungFlags,
                                          events_from_flags)
from paper_2605_20868_b200.cache import storage_table

import oracle
from oracle.step import aggregate as oracle_aggregate, make_workload


def test_policy_validation_matches_reference():
    with pytest.raises(ValueError, match="tau_cov"):
        PolicyConfig(tau_cov=1.5)
    with pytest.raises(ValueError, match="k_min"):
        PolicyConfig(k_min=5, k_max=2)
    with pytest.raises(ValueError, match="exploration_rate"):
        PolicyConfig(exploration_rate=0.5)
    with pytest.raises(ValueError, match="unknown policy fields"):
        PolicyConfig.from_dict({"bogus": 1})
    p = PolicyConfig.naive()
    assert p.k_max == 0 and not p.canary_enabled
    assert PolicyConfig.from_dict(PolicyConfig().to_dict()) == PolicyConfig()
    c = PolicyConfig(greedy_value_budget=0.1).to_c()
    assert c.greedy_value_budget == 0.1 and PolicyConfig().to_c().greedy_value_budget < 0


def test_events_from_flags_order():
    fl = _lib.F_RUNG1 | _lib.F_RUNG2 | _lib.F_RANKING | _lib.F_BOUNDARY | _lib.F_CANARY
    ev = events_from_flags(fl, 3, 7)
    assert [(e.rung, e.cause) for e in ev] == [
        (1, "coverage_expand"), (2, "value_tol"), (3, "ranking_disagree"),
        (3, "boundary"), (4, "canary")]
    with pytest.raises(ValueError):
        FallbackEvent(4, 0, 0, "boundary")


def test_certificate_returned_bounds():
    c = Certificate(0, 0, 0.1, 1.0, 2.0, 0.5, 0.3, 4.0, 8, "dense_per_head", RungFlags(rung3=True))
    assert c.is_dense and c.returned_e_key == 0.0 and c.returned_e_val == 0.0
    q = Certificate(0, 0, 0.1, 1.0, 2.0, 0.5, 0.3, 4.0, 8, "quantized")
    assert q.returned_e_key == 2.0 and q.returned_e_val == 0.5


def test_storage_table_matches_oracle():
    for d, b, g in [(128, 16, 16), (64, 16, 16), (32, 8, 8)]:
        a = storage_table(d, b, g).to_dict()
        o = oracle.storage_table(d, b, g)
        for k, v in o.items():
            assert a[k] == v, k
    assert storage_table(128, 16, 16).tier1_total_bytes == _lib.BLOCK_BYTES / _lib.BLOCK


def test_synth_arrays_match_oracle_generator():
    for kind in ("gaussian", "sink", "needle", "near_tie"):
        cfg = WorkloadConfig(ingest_binary16=True, kind=kind, n_tokens=100, head_dim=128, query_heads=8, kv_heads=2,
                             steps=3, seed=4)
        k, v, q = synth_arrays(cfg)
        o = make_workload(kind=kind, n_tokens=100, head_dim=128, query_heads=8, kv_heads=2,
                          steps=3, seed=4, build_caches=False)
        assert np.array_equal(k, o["keys"]) and np.array_equal(v, o["values"])
        assert np.array_equal(q, o["queries"])


def test_telemetry_schema_matches_oracle():
    """A device-shaped record built from certificates aggregates exactly like
    the oracle's (harness.py:397-499)."""
    cfg = WorkloadConfig(ingest_binary16=True, kind="gaussian", n_tokens=64, head_dim=128, query_heads=4,
                         kv_heads=1, steps=2)
    recs = []
    for s in range(2):
        certs = [Certificate(h, s, 0.1 * h, 0.01, 0.02 * h, 0.3, 0.2, 3.0, 4 + h,
                             "quantized" if h else "dense_per_head",
                             RungFlags(rung3=(h == 0)))
                 for h in range(4)]
        ev = [FallbackEvent(3, 0, s, "ranking_disagree")]
        recs.append(step_record(s, certs, ev, {"hits": 1, "misses": 2, "hit_rate": 1 / 3,
                                               "bytes_paged_in": 8192},
                                {"hits": 0, "misses": 0, "hit_rate": 0.0, "bytes_paged_in": 0},
                                8192, 0, [0.5]))
    a = aggregate_telemetry(recs, cfg)
    b = oracle_aggregate(recs, 4)
    assert a == b
    assert a["rates"]["dense_fraction"] == 0.25


# ---- boundary fidelity: unsupported reference geometry is refused, not coerced ----

def test_workload_config_rejects_unsupported_geometry():
    with pytest.raises(ValueError, match="head_dim=128"):
        WorkloadConfig()  # the reference defaults: head_dim 64, float32 ingest
    with pytest.raises(ValueError, match="ingest_binary16"):
        WorkloadConfig(head_dim=128)
    with pytest.raises(ValueError, match="group_size"):
        WorkloadConfig(head_dim=128, group_size=32, ingest_binary16=True)
    with pytest.raises(ValueError, match="4 query heads"):
        WorkloadConfig(head_dim=128, ingest_binary16=True, query_heads=8, kv_heads=1)
    cfg = WorkloadConfig(head_dim=128, ingest_binary16=True, query_heads=4)
    assert WorkloadConfig.from_dict(cfg.to_dict()) == cfg
    # field names and the remaining defaults are the reference's (harness.py:41-51)
    assert (cfg.kind, cfg.n_tokens, cfg.block_size, cfg.kv_heads, cfg.steps, cfg.seed) == \
        ("gaussian", 1024, 16, 1, 8, 0)


def test_tiered_cache_rejects_float32_ingest_and_other_dims():
    from paper_2605_20868_b200 import TieredCache
    with pytest.raises(ValueError, match="ingest_binary16"):
        TieredCache(16, 128, 16)  # reference default ingest_binary16=False (cache.py:52)
    with pytest.raises(ValueError, match="ingest_binary16"):
        TieredCache(16, 128, 16, ingest_binary16=False)
    with pytest.raises(ValueError, match="head_dim=128"):
        TieredCache(16, 64, 16, ingest_binary16=True)
    with pytest.raises(ValueError, match="does not divide"):
        TieredCache(16, 128, 48, ingest_binary16=True)


def test_scratch_cache_reference_view_and_page_report():
    from paper_2605_20868_b200 import ScratchCache
    from paper_2605_20868_b200.cache import PageInReport
    with pytest.raises(ValueError):
        ScratchCache(-1)
    s = ScratchCache(8)
    assert (s.hits, s.misses, s.bytes_paged_in, s.hit_rate) == (0, 0, 0, 0.0)
    s._account(3, 1, 4096)
    assert (s.hits, s.misses, s.bytes_paged_in, s.hit_rate) == (3, 1, 4096, 0.75)
    r = PageInReport(2, 1, 4096)
    assert r.to_dict() == {"hits": 2, "misses": 1, "bytes": 4096} and r.payloads == {}


def test_resolve_manifest_as_the_reference_cli(tmp_path):
    """Run manifests resolve as cli.py:36-77 resolves them: sections, seed
    override, scratch defaults, and the same refusals."""
    import json
    from paper_2605_20868_b200.harness import resolve_manifest
    p = tmp_path / "m.json"
    p.write_text(json.dumps({"workload": {"kind": "gaussian", "n_tokens": 100, "head_dim": 128,
                                          "ingest_binary16": True}, "seed": 9,
                             "policy": {"k_max": 8}, "scratch": {"key_capacity": 32}}))
    wl, pol, kc, vc, layers = resolve_manifest(str(p))
    assert (wl.seed, pol.k_max, kc, vc, layers) == (9, 8, 32, 2048, 1)
    assert resolve_manifest(str(p), seed=3)[0].seed == 3
    for bad in ({"extra": {}}, {"scratch": {"slots": 1}}, {"workload": {"nope": 1}}, []):
        p.write_text(json.dumps(bad))
        with pytest.raises(ValueError):
            resolve_manifest(str(p))
    p.write_text("{")
    with pytest.raises(ValueError, match="malformed JSON"):
        resolve_manifest(str(p))
