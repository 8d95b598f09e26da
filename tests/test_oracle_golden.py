"""Pin the CPU oracle against golden vectors frozen from the real reference.

The fixtures under tests/golden/ were produced by tests/golden/make_golden.py
from /root/reference (certkv, pure backend).  These tests need no GPU and no
reference checkout.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import quant
from oracle.margins import as_row, margins_from_oracle
from oracle.step import OraclePolicy, make_workload, run_workload

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KINDS = ["quantized", "dense_per_head", "dense_all_heads"]


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


class TestQuantizerGolden:
    def test_blocks_bit_exact(self):
        z = _load("quantizer.npz")
        blocks = z["blocks"].astype(np.float64)
        for i, blk in enumerate(blocks):
            kc, ks, ko = quant.fit_key_block(blk)
            assert np.array_equal(kc, z["kcodes"][i]), i
            assert np.array_equal(ks, z["kscale"][i]), i
            assert np.array_equal(ko, z["koffset"][i]), i
            vc, vs, vo = quant.fit_value_block(blk, 16)
            assert np.array_equal(vc, z["vcodes"][i]), i
            assert np.array_equal(vs, z["vscale"][i]), i
            assert np.array_equal(vo, z["voffset"][i]), i
            eta, nu = quant.value_annotations(blk, quant.dequant_values(vc, vs, vo, 16))
            assert eta == z["eta"][i] and nu == z["nu"][i], i

    def test_kats(self):
        z = _load("quantizer.npz")
        kc, ks, ko = quant.fit_key_block(np.array([[-1.0], [1.0]]))
        assert kc.ravel().tolist() == [-128, 127] == z["kat_two_codes"].ravel().tolist()
        assert ks[0] == 2.0 / 255.0 == z["kat_two_scale"][0]
        assert ko[0] == z["kat_two_offset"][0]
        vc, vs, vo = quant.fit_value_block(np.array([[0.0, 1.5]]), 2)
        assert vc.ravel().tolist() == [0, 15]
        assert vs.ravel()[0] == z["kat_grp_scale"].ravel()[0]
        eta, _ = quant.value_annotations(np.array([[0.0, 1.5]]),
                                         quant.dequant_values(vc, vs, vo, 2))
        assert eta == float(z["kat_grp_eta"]) == 0.0

    def test_constant_and_nonfinite(self):
        kc, ks, ko = quant.fit_key_block(np.full((4, 3), 0.5))
        assert np.all(kc == 0) and np.all(ks == 1.0) and np.all(ko == 0.5)
        x = np.zeros((2, 4))
        x[1, 2] = np.nan
        with pytest.raises(ValueError, match="channel 2"):
            quant.fit_key_block(x)
        with pytest.raises(ValueError, match="does not divide"):
            quant.fit_value_block(np.zeros((2, 6)), 4)

    def test_pairwise_order_matches_numpy(self):
        rng = np.random.default_rng(0)
        for d in (128, 64, 16, 8, 5):
            for _ in range(200):
                row = rng.standard_normal(d) ** 2 * 10 ** rng.uniform(-3, 3)
                assert quant.pairwise_sum128(row) == np.sum(row[None, :], axis=-1)[0]


def _runs():
    with open(os.path.join(GOLD, "runs.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_runs()))
def test_run_workload_golden(name):
    spec = _runs()[name]
    wl = make_workload(ingest_binary16=True, **spec["workload"])
    keys = np.stack([np.concatenate(c.tier2_k + [c.partial_keys().astype(np.float32)])
                     for c in wl["caches"]])
    assert hashlib.sha256(np.ascontiguousarray(keys).tobytes()).hexdigest() == spec["keys_digest"]
    assert hashlib.sha256(wl["queries"].tobytes()).hexdigest() == spec["queries_digest"]
    kc, vc = spec["capacities"]
    pol = OraclePolicy(**spec["policy"])
    res = run_workload(wl, pol, kc, vc)
    z = _load(f"run_{name}.npz")
    recs = json.loads(str(z["records_json"]))
    summ = json.loads(str(z["summary_json"]))
    i = 0
    for step, (rec, gold) in enumerate(zip(res["records"], recs)):
        for r in res["results"][step]:
            row = z["cert"][i]
            assert r["head"] == row[1]
            np.testing.assert_allclose(
                [r["delta_h"], r["e_key_tight"], r["e_key_impl"], r["e_val"],
                 r["est_tail_mass"], r["v_max"]], row[2:8], rtol=1e-10, atol=1e-14)
            assert r["k_star"] == row[8]
            assert KINDS.index(r["kind"]) == row[9]
            assert tuple(bool(x) for x in r["flags"]) == tuple(bool(x) for x in row[10:14])
            np.testing.assert_allclose(r["output"], z["outputs"][i], rtol=1e-6, atol=1e-7)
            p = z["promoted"][i]
            assert r["promoted"].tolist() == p[p >= 0].tolist()
            v = z["value_promotions"][i]
            assert r["value_promotions"].tolist() == v[v >= 0].tolist()
            # threshold distances of every decision, as the reference's own objects give them
            m = np.asarray(as_row(margins_from_oracle(r, pol)))
            g = z["margins"][i]
            assert np.array_equal(np.isinf(m), np.isinf(g)), (i, m, g)
            fin = ~np.isinf(g)
            np.testing.assert_allclose(m[fin], g[fin], rtol=1e-6, atol=1e-12)
            i += 1
        for key in ("rung_counts", "cause_counts", "key_scratch", "value_scratch",
                    "bytes_paged_in", "rung4_staging_bytes", "k_star_mean"):
            assert rec[key] == gold[key], key
        assert rec["events"] == gold["events"]
        np.testing.assert_allclose(rec["union_fraction_mean"], gold["union_fraction_mean"])
    for key in ("steps", "head_steps", "rung_counts", "cause_counts", "rates",
                "bytes_paged_in_total", "rung4_staging_bytes_total"):
        assert res["summary"][key] == summ[key], key


def test_fault_injection_golden():
    z = _load("fault.npz")
    kv = oracle.OracleKV(16, 64, 16)
    kv.append_tokens(z["keys"], z["values"])
    pol = OraclePolicy(exploration_rate=0.0)
    q = z["query"]
    honest = oracle.decode_step(q, kv, pol)
    np.testing.assert_allclose(honest["output"], z["honest_output"], rtol=1e-6, atol=1e-7)
    assert not honest["flags"][3]
    ch = int(np.argmax(np.abs(q)))
    kv.corrupt_offset(0, ch, 10.0 * (1.0 + np.abs(kv.kscale[0]).sum()))
    tripped = oracle.decode_step(q, kv, pol)
    assert tripped["flags"][3] and bool(z["tripped_rung4"])
    assert tripped["kind"] == str(z["tripped_kind"]) == "dense_all_heads"
    np.testing.assert_allclose(tripped["output"], z["tripped_output"], rtol=1e-12, atol=1e-14)


def test_tier2_loss_is_hard_error():
    kv = oracle.OracleKV(16, 32, 16)
    rng = np.random.default_rng(0)
    kv.append_tokens(rng.standard_normal((40, 32)), rng.standard_normal((40, 32)))
    kv.tier2_k[0] = None
    with pytest.raises(oracle.Tier2Lost):
        oracle.decode_step(rng.standard_normal(32), kv, OraclePolicy(exploration_rate=0.0))


def test_storage_table():
    t = oracle.storage_table(128, 16, 16)
    assert t["tier1_total_bytes"] == 288 and t["dense_bytes"] == 512
    assert t["tier1_ratio"] == 0.5625 and t["tier1_exact_bytes"] == 288.25
