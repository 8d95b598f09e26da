"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars: codes bit-exact; key scale/offset == float32(fp64
fit); value scale/offset == float16(fp64 fit); eta/nu == float32(oracle with
the same narrowing); fast-path outputs within 1e-4 of max|O|; Delta, E_key,
E_val, tail mass within 1e-4 relative (+1e-9 absolute); decisions, rung
flags, returned kinds and LRU page accounting identical on these seeded
workloads.
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.step import OraclePolicy, make_workload, run_workload as oracle_run

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ck():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    assert torch.cuda.is_available()
    return ck


def _oracle_blocks(blocks):
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
    kv.append_tokens(blocks.reshape(-1, 128), blocks.reshape(-1, 128)[::-1].copy())
    return kv


# ---- quantize-on-append (K1) -------------------------------------------------

def test_quantize_bit_exact_golden_blocks(ck):
    z = np.load(os.path.join(GOLD, "quantizer.npz"))
    blocks = z["blocks"].astype(np.float64)           # [44, 16, 128] fp16-exact
    keys = blocks.reshape(-1, 128)
    vals = keys[::-1].copy()
    cache = ck.DeviceKVCache(1, keys.shape[0] + 16)
    # append in ragged chunks to exercise the partial-block carry
    pos = 0
    for n in (7, 20, 1, 16, 100, keys.shape[0]):
        n = min(n, keys.shape[0] - pos)
        if n <= 0:
            break
        cache.append(torch.from_numpy(keys[pos:pos + n])[None], torch.from_numpy(vals[pos:pos + n])[None])
        pos += n
    assert cache.num_blocks == blocks.shape[0] and cache.partial_len == 0
    t1 = cache.read_tier1(0)
    kv = _oracle_blocks(blocks)
    for b in range(blocks.shape[0]):
        assert np.array_equal(t1["kcodes"][b], kv.kcodes[b]), b
        assert np.array_equal(t1["kscale"][b], kv.kscale[b].astype(np.float32)), b
        assert np.array_equal(t1["koffset"][b], kv.koffset[b].astype(np.float32)), b
        assert np.array_equal(t1["vcodes"][b], kv.vcodes[b]), b
        assert np.array_equal(t1["vscale"][b], kv.vscale[b].astype(np.float16)), b
        assert np.array_equal(t1["voffset"][b], kv.voffset[b].astype(np.float16)), b
        # golden keys straight from the reference
        assert np.array_equal(t1["kcodes"][b], z["kcodes"][b])
    assert np.array_equal(cache.eta[0, :blocks.shape[0]].cpu().numpy(),
                          np.asarray(kv.eta, dtype=np.float32))
    assert np.array_equal(cache.nu[0, :blocks.shape[0]].cpu().numpy(),
                          np.asarray(kv.nu, dtype=np.float32))
    assert cache.v_max(0) == np.float32(kv.v_max)


def test_quantize_random_multi_unit(ck):
    rng = np.random.default_rng(7)
    U, N = 6, 16 * 37 + 5
    k = (rng.standard_normal((U, N, 128)) * 10 ** rng.uniform(-2, 2, (U, 1, 1))).astype(np.float16)
    v = (rng.standard_normal((U, N, 128)) * 10 ** rng.uniform(-2, 2, (U, 1, 1))).astype(np.float16)
    k[2, :, 5] = 3.0           # constant channel
    v[3, 40:56, 16:32] = -1.5  # constant value group
    cache = ck.DeviceKVCache(U, N)
    cache.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    assert cache.num_blocks == N // 16 and cache.partial_len == 5
    for u in range(U):
        kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
        kv.append_tokens(k[u].astype(np.float64), v[u].astype(np.float64))
        t1 = cache.read_tier1(u)
        assert np.array_equal(t1["kcodes"], np.stack(kv.kcodes))
        assert np.array_equal(t1["vcodes"], np.stack(kv.vcodes))
        assert np.array_equal(t1["kscale"], np.stack(kv.kscale).astype(np.float32))
        assert np.array_equal(t1["voffset"], np.stack(kv.voffset).astype(np.float16))
        assert np.array_equal(cache.eta[u, :cache.num_blocks].cpu().numpy(),
                              np.asarray(kv.eta, dtype=np.float32))
        assert np.array_equal(cache.partial_k[u, :5].cpu().numpy(), k[u, -5:])


def test_nonfinite_append_is_rejected_without_mutation(ck):
    cache = ck.DeviceKVCache(2, 64)
    x = torch.zeros((2, 20, 128), dtype=torch.float16, device="cuda")
    cache.append(x[:, :5], x[:, :5])
    bad = x.clone()
    bad[1, 3, 7] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        cache.append(bad, x)
    assert cache.num_tokens == 5 and int(cache.n_blocks_t.sum()) == 0
    assert cache.partial_len_t.cpu().tolist() == [5, 5]
    with pytest.raises(ValueError, match="capacity"):
        big = torch.zeros((2, cache.max_blocks * 16 + 16, 128), device="cuda")
        cache.append(big, big)


# ---- plugin kernels -----------------------------------------------------------

def test_plugin_kernels_match_oracle(ck):
    rng = np.random.default_rng(1)
    s = rng.standard_normal(16 * 9 + 5) * 3
    bounds = np.asarray([16 * i for i in range(10)] + [16 * 9 + 5], dtype=np.int64)
    a = ck.kernels.block_logmass(s, bounds)
    b = oracle.block_logmass(s, bounds)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-13)
    vals = rng.standard_normal((s.size, 64)).astype(np.float32)
    o1, m1, l1 = ck.kernels.fused_attend(s.astype(np.float32), vals, bounds)
    o2, m2, l2 = oracle.fused_attend_f32(s.astype(np.float32), vals, bounds)
    np.testing.assert_allclose(o1, o2, rtol=2e-5, atol=2e-6)
    assert m1 == m2
    np.testing.assert_allclose(l1, l2, rtol=1e-5)


# ---- the certified decode step --------------------------------------------------

RUNS = [
    ("gauss", dict(kind="gaussian", n_tokens=520, query_heads=8, kv_heads=2, steps=3, seed=0),
     dict(), (2048, 2048)),
    ("gauss_kmax8", dict(kind="gaussian", n_tokens=1030, query_heads=8, kv_heads=2, steps=3,
                         seed=3), dict(k_max=8), (24, 24)),
    ("sink", dict(kind="sink", n_tokens=600, query_heads=8, kv_heads=2, steps=3, seed=1),
     dict(), (2048, 2048)),
    ("needle", dict(kind="needle", n_tokens=777, query_heads=8, kv_heads=2, steps=2, seed=2),
     dict(k_max=16), (2048, 2048)),
    ("near_tie", dict(kind="near_tie", n_tokens=640, query_heads=8, kv_heads=2, steps=2, seed=5),
     dict(k_max=4), (2048, 2048)),
    ("tight_vtol", dict(kind="sink", n_tokens=700, query_heads=8, kv_heads=2, steps=2, seed=11),
     dict(v_tol=0.01), (2048, 2048)),
    ("long_gauss", dict(kind="gaussian", n_tokens=9000, query_heads=8, kv_heads=2, steps=2,
                        seed=21), dict(), (300, 100)),
    ("no_rung1", dict(kind="needle", n_tokens=2000, query_heads=4, kv_heads=1, steps=2, seed=8),
     dict(rung1_enabled=False, k_max=32, ranking_depth=2), (2048, 2048)),
]


def _close(a, b, rtol=1e-4, atol=1e-9):
    return abs(a - b) <= atol + rtol * abs(b)


@pytest.mark.parametrize("name,wkw,pkw,caps", RUNS, ids=[r[0] for r in RUNS])
def test_run_workload_parity(ck, name, wkw, pkw, caps):
    cfg = ck.WorkloadConfig(head_dim=128, ingest_binary16=True, **wkw)
    wl = ck.generate_workload(cfg)
    pol = ck.PolicyConfig(exploration_rate=0.0, **pkw)
    dev = ck.run_workload(wl, pol, key_capacity=caps[0], value_capacity=caps[1], keep_outputs=True)
    ow = make_workload(head_dim=128, ingest_binary16=True, narrow=True, **wkw)
    ref = oracle_run(ow, OraclePolicy(exploration_rate=0.0, **pkw), caps[0], caps[1])
    for s, (drec, orec) in enumerate(zip(dev.step_records, ref["records"])):
        for h, (dc, oc) in enumerate(zip(drec["certificates"], orec["certificates"])):
            ctx = f"{name} step {s} head {h}"
            assert dc["k_star"] == oc["k_star"], ctx
            assert dc["rung_flags"] == oc["rung_flags"], ctx
            assert dc["returned_kind"] == oc["returned_kind"], ctx
            for key in ("delta_h", "e_key_tight", "e_key_impl", "e_val", "est_tail_mass", "v_max"):
                assert _close(dc[key], oc[key]), (ctx, key, dc[key], oc[key])
            r = ref["results"][s][h]
            o_dev = dev.outputs[s][h]
            scale = np.abs(r["output"]).max()
            err = np.abs(o_dev - r["output"]).max() / scale
            assert err < 1e-4, (ctx, err)
        assert drec["events"] == orec["events"], name
        assert drec["key_scratch"] == orec["key_scratch"], name
        assert drec["value_scratch"] == orec["value_scratch"], name
        assert drec["bytes_paged_in"] == orec["bytes_paged_in"]
        assert drec["rung4_staging_bytes"] == orec["rung4_staging_bytes"]
        assert abs(drec["union_fraction_mean"] - orec["union_fraction_mean"]) < 1e-12


def test_promoted_sets_match_golden_reference(ck):
    """Decisions against the frozen reference run (not only the oracle)."""
    spec = json.load(open(os.path.join(GOLD, "runs.json")))["sink"]
    z = np.load(os.path.join(GOLD, "run_sink.npz"))
    cfg = ck.WorkloadConfig(head_dim=128, ingest_binary16=True,
                            **{k: v for k, v in spec["workload"].items() if k != "head_dim"})
    wl = ck.generate_workload(cfg)
    dec = ck.CertifiedDecoder(wl.cache, ck.PolicyConfig(**spec["policy"]), n_heads=4)
    q = torch.from_numpy(wl.queries[0].reshape(2, 4, 128)).cuda()
    res = dec.step(q)
    for h in range(8):
        p = z["promoted"][h]
        assert sorted(res.promoted(h // 4, h % 4).tolist()) == p[p >= 0].tolist()
        v = z["value_promotions"][h]
        assert res.value_promotions(h // 4, h % 4).tolist() == v[v >= 0].tolist()
        out = res.out[h // 4, h % 4].double().cpu().numpy()
        ref = z["outputs"][h]
        assert np.abs(out - ref).max() / np.abs(ref).max() < 2e-3  # includes FP16 value-meta narrowing


def test_per_head_api_matches_oracle(ck):
    rng = np.random.default_rng(3)
    k = rng.standard_normal((500, 128)).astype(np.float16).astype(np.float64)
    v = rng.standard_normal((500, 128)).astype(np.float16).astype(np.float64)
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=1024)
    cache.append_tokens(k, v)
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
    kv.append_tokens(k, v)
    assert cache.num_blocks == kv.num_blocks and cache.partial_len == kv.partial_len
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=6)
    for _ in range(3):
        q = rng.standard_normal(128)
        a = ck.run_decode_step(q, cache, pol)
        b = oracle.decode_step(q, kv, OraclePolicy(exploration_rate=0.0, k_max=6))
        assert sorted(a.decision.promoted) == b["promoted"].tolist()
        assert a.certificate.k_star == b["k_star"]
        assert a.certificate.returned_kind == b["kind"]
        assert np.abs(a.output - b["output"]).max() / np.abs(b["output"]).max() < 1e-4
        assert [(e.rung, e.cause) for e in a.events] == b["events"]


def test_fault_injection_trips_canary(ck):
    z = np.load(os.path.join(GOLD, "fault.npz"))
    # the golden sink cache is d=64; build the d=128 analogue with the same recipe
    rng = np.random.default_rng(0)
    w = rng.standard_normal(128)
    w /= np.linalg.norm(w)
    keys = rng.standard_normal((96, 128))
    keys[:16] = 2.0 * np.sqrt(128) / 3.0 * w + 0.1 * keys[:16]
    vals = rng.standard_normal((96, 128))
    keys = keys.astype(np.float16).astype(np.float64)
    vals = vals.astype(np.float16).astype(np.float64)
    q = 3.0 * w + rng.standard_normal(128)
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=128)
    cache.append_tokens(keys, vals)
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
    kv.append_tokens(keys, vals)
    pol = ck.PolicyConfig(exploration_rate=0.0)
    honest = ck.run_decode_step(q, cache, pol)
    assert not honest.rung4_requested and honest.certificate.returned_kind == "quantized"
    ch = int(np.argmax(np.abs(q)))
    shift = float(10.0 * (1.0 + np.abs(kv.kscale[0]).sum()))
    cache.dev.corrupt_offset(0, 0, ch, shift)
    kv.corrupt_offset(0, ch, shift)
    a = ck.run_decode_step(q, cache, pol)
    b = oracle.decode_step(q, kv, OraclePolicy(exploration_rate=0.0))
    assert a.rung4_requested and b["flags"][3]
    assert a.certificate.returned_kind == "dense_all_heads" == b["kind"]
    assert a.certificate.returned_e_key == 0.0
    np.testing.assert_allclose(a.output, b["output"], rtol=1e-5, atol=1e-6)
    assert bool(z["tripped_rung4"])


def test_tier2_loss_is_hard_error(ck):
    rng = np.random.default_rng(5)
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=256)
    cache.append_tokens(rng.standard_normal((100, 128)), rng.standard_normal((100, 128)))
    cache.dev.drop_tier2(0, 0)
    with pytest.raises(ck.Tier2UnavailableError):
        ck.run_decode_step(rng.standard_normal(128), cache, ck.PolicyConfig(exploration_rate=0.0))


def test_empty_cache_raises(ck):
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=64)
    with pytest.raises(ck.EmptyCacheError):
        ck.run_decode_step(np.zeros(128), cache, ck.PolicyConfig(exploration_rate=0.0))


def test_partial_only_cache(ck):
    rng = np.random.default_rng(6)
    k, v = rng.standard_normal((9, 128)), rng.standard_normal((9, 128))
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=64)
    cache.append_tokens(k, v)
    q = rng.standard_normal(128)
    a = ck.run_decode_step(q, cache, ck.PolicyConfig(exploration_rate=0.0))
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
    kv.append_tokens(k, v)
    b = oracle.decode_step(q, kv, OraclePolicy(exploration_rate=0.0))
    assert a.certificate.k_star == 0 == b["k_star"]
    np.testing.assert_allclose(a.output, b["output"], rtol=1e-5, atol=1e-6)


# ---- full-size properties ------------------------------------------------------------

def test_output_soundness_large(ck):
    """At 32K tokens x 16 units: the fast-path output is within the certified
    E_key(tight) + E_val of the exact dense attention (verification.py:274-319)."""
    U, N = 16, 32768 + 7
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((U, N, 128), generator=g, device="cuda", dtype=torch.float32)
    v = torch.randn((U, N, 128), generator=g, device="cuda", dtype=torch.float32)
    cache = ck.DeviceKVCache(U, N)
    cache.append(k, v)
    pol = ck.PolicyConfig(exploration_rate=0.0)
    dec = ck.CertifiedDecoder(cache, pol, n_heads=4)
    q = torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
    res = dec.step(q)
    assert (res.cert["k_star"] == 256).all()
    for u in range(U):
        kk, vv = cache.tier2_rows(u)
        s = (kk.double() @ q[u].T) / np.sqrt(128)
        ref = torch.softmax(s, 0).T @ vv.double()
        for h in range(4):
            if res.kinds[u, h]:
                continue
            err = float(torch.linalg.norm(res.out[u, h].double() - ref[h]))
            c = res.cert[u, h]
            assert err <= c["e_key_tight"] + c["e_val"] + 1e-5, (u, h, err)


@pytest.mark.parametrize("env", [{}, {"CKV_SEPARATE_PAGEIN": "1"}], ids=["passb_pagein", "gather_pagein"])
def test_host_tier2_matches_device_tier2(ck, monkeypatch, env):
    """Tier-2 in pinned host RAM (misses paged into HBM slots by pass B itself, or
    by the separate gather kernel) gives the same step as Tier-2 in HBM."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    cfg = ck.WorkloadConfig(ingest_binary16=True, kind="sink", n_tokens=3000, head_dim=128, query_heads=8, kv_heads=2,
                            steps=4, seed=4)
    pol = ck.PolicyConfig(exploration_rate=0.0, v_tol=0.01)
    outs = []
    for where in ("device", "host"):
        wl = ck.generate_workload(cfg, tier2=where)
        r = ck.run_workload(wl, pol, 64, 64, keep_outputs=True)
        outs.append((r.outputs, r.step_records))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)
    assert outs[0][1] == outs[1][1]


def test_dense_reads_hbm_slots_bit_identical(ck):
    """Rung-3/4 dense units with Tier-2 in host RAM read their blocks already
    paged into HBM slots from the slots and the rest from host Tier-2: outputs,
    kinds and certificates equal those of the same steps with Tier-2 in HBM."""
    U, N = 4, 4000
    g = torch.Generator(device="cuda").manual_seed(12)
    k = torch.randn((U, N, 128), generator=g, device="cuda", dtype=torch.float32)
    v = torch.randn((U, N, 128), generator=g, device="cuda", dtype=torch.float32)
    qs = [torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
          for _ in range(3)]
    runs = []
    for where in ("device", "host"):
        cache = ck.DeviceKVCache(U, N + 8, tier2=where)
        cache.append(k, v)
        dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0, v_tol=0.01),
                                  n_heads=4, scratch=ck.ScratchCache(cache.max_blocks),
                                  rung4_group=1)
        res = []
        for s, q in enumerate(qs):
            if s == 1:
                cache.corrupt_offset(1, 3, 0, 1e4)  # canary on unit 1 -> its group goes dense
            r = dec.step(q)
            res.append((r.out.clone(), r.kinds.copy(), r.cert.copy()))
        runs.append(res)
    for s, (a, b) in enumerate(zip(*runs)):
        assert torch.equal(a[0], b[0]), s
        assert np.array_equal(a[1], b[1]), s
        assert a[2].tobytes() == b[2].tobytes(), s
    assert runs[1][1][1][1].all() and runs[1][2][1][1].all()
    assert not runs[1][0][1][1].any()


@pytest.mark.parametrize("name", ["explore", "greedy"])
def test_exploration_and_greedy_parity(ck, name, tmp_path):
    """Exploration spot checks (host Philox draws, device rescoring) and the greedy
    Rung-2 budget mode against the oracle; the bound report is written as JSONL."""
    if name == "explore":
        wkw = dict(kind="gaussian", n_tokens=2400, query_heads=8, kv_heads=2, steps=3, seed=7)
        pkw = dict(exploration_rate=0.05, k_max=8)
    else:
        wkw = dict(kind="sink", n_tokens=1500, query_heads=8, kv_heads=2, steps=2, seed=12)
        pkw = dict(exploration_rate=0.0, greedy_value_budget=0.3)
    cfg = ck.WorkloadConfig(head_dim=128, ingest_binary16=True, **wkw)
    wl = ck.generate_workload(cfg)
    dev = ck.run_workload(wl, ck.PolicyConfig(**pkw), 64, 64, keep_outputs=True)
    ow = make_workload(head_dim=128, ingest_binary16=True, narrow=True, **wkw)
    ref = oracle_run(ow, OraclePolicy(**pkw), 64, 64)
    for s, (drec, orec) in enumerate(zip(dev.step_records, ref["records"])):
        assert drec["events"] == orec["events"], (name, s)
        assert drec["rung_counts"] == orec["rung_counts"]
        assert drec["bytes_paged_in"] == orec["bytes_paged_in"]
        assert drec["key_scratch"] == orec["key_scratch"]
        assert drec["value_scratch"] == orec["value_scratch"]
        for dc, oc in zip(drec["certificates"], orec["certificates"]):
            assert dc["returned_kind"] == oc["returned_kind"]
            assert _close(dc["e_val"], oc["e_val"]) and dc["k_star"] == oc["k_star"]
    if name == "greedy":
        assert sum(r["rung_counts"]["rung2"] for r in dev.step_records) > 0
    path = ck.write_telemetry(dev, str(tmp_path / "run.jsonl"))
    lines = open(path).read().splitlines()
    assert len(lines) == cfg.steps + 2 and '"kernel_backend":"b200"' in lines[0]


# ---- adversarial inputs (BASELINE config C5 in miniature) ----------------------------

def test_adversarial_outliers_near_tie_fault(ck):
    """Outlier key channels (x1000 on two channels), near-tie twin blocks and a
    corrupted key offset (verification.py:420-428): the batched decoder agrees
    with the oracle on decisions, kinds and outputs, the fault makes its unit's
    Rung-4 group dense while the other group stays certified."""
    wl = make_workload(kind="near_tie", n_tokens=1500, head_dim=128, query_heads=8, kv_heads=2,
                       steps=3, seed=13, ingest_binary16=True, narrow=True, build_caches=False)
    keys = wl["keys"].copy()
    keys[:, :, 3] *= 1000.0
    keys[:, :, 77] *= 1000.0
    keys = keys.astype(np.float16).astype(np.float64)
    vals = wl["values"].astype(np.float16).astype(np.float64)
    n = 1500
    kvs = []
    for u in range(2):
        kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
        kv.append_tokens(keys[u, :n], vals[u, :n])
        kvs.append(kv)
    cache = ck.DeviceKVCache(2, n + 16)
    cache.append(torch.from_numpy(keys[:, :n]), torch.from_numpy(vals[:, :n]))
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=8)
    opol = OraclePolicy(exploration_rate=0.0, k_max=8)
    # two Rung-4 groups: unit 0 and unit 1 (as two layers would be)
    dec = ck.CertifiedDecoder(cache, pol, n_heads=4, rung4_group=[0, 1])
    for s in range(3):
        if s == 2:  # corrupt one stored key offset of a block head 0 promotes (both sides)
            q0 = wl["queries"][s, 0]
            bf = int(oracle.decode_step(q0, kvs[0], opol)["promoted"][0])
            ch = int(np.argmax(np.abs(q0)))
            # raise the block's phase-1 scores so it stays promoted and is checked
            shift = float(np.sign(q0[ch]) * 50.0 * (1.0 + np.abs(kvs[0].kscale[bf]).sum()))
            cache.corrupt_offset(0, bf, ch, shift)
            kvs[0].corrupt_offset(bf, ch, shift)
        q = torch.from_numpy(wl["queries"][s].reshape(2, 4, 128)).cuda()
        res = dec.step(q)
        out = res.out.double().cpu().numpy()
        refs = [oracle.decode_step(wl["queries"][s, h], kvs[h // 4], opol) for h in range(8)]
        for u in range(2):
            any4 = any(refs[4 * u + j]["flags"][3] for j in range(4))
            for j in range(4):
                r = refs[4 * u + j]
                row = res.cert[u, j]
                ctx = (s, u, j)
                assert int(row["k_star"]) == r["k_star"], ctx
                want = "dense_all_heads" if any4 else r["kind"]
                assert ck.engine.KINDS[int(res.kinds[u, j])] == want, ctx
                if want == "dense_all_heads" and r["kind"] != "dense_all_heads":
                    ref_out = oracle.dense_output(wl["queries"][s, 4 * u + j], kvs[u])
                else:
                    ref_out = r["output"]
                err = np.abs(out[u, j] - ref_out).max() / np.abs(ref_out).max()
                assert err < 1e-4, (ctx, err)
        if s == 2:
            assert (res.kinds[0] == 2).all()      # the corrupted unit's group is dense
            assert not (res.kinds[1] == 2).any()  # the other group is not


# ---- serving-loop API ---------------------------------------------------------------

def test_step_async_matches_step_and_defers_append_check(ck):
    """step_async returns the same certificates as step (one step later on the
    host); a non-finite append with validate="defer" is rejected on the device
    and surfaces as ValueError from the next step's result."""
    rng = np.random.default_rng(21)
    U, n = 3, 700
    k = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    v = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    ca = ck.DeviceKVCache(U, n + 32)
    cb = ck.DeviceKVCache(U, n + 32)
    ca.append(k, v)
    cb.append(k, v)
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=6)
    da = ck.CertifiedDecoder(ca, pol, n_heads=4, rung4_group=[0, 1, 0])
    db = ck.CertifiedDecoder(cb, pol, n_heads=4, rung4_group=[0, 1, 0])
    qs = [torch.from_numpy(rng.standard_normal((U, 4, 128))).cuda() for _ in range(3)]
    pend = []
    for q in qs:
        pend.append(da.step_async(q))
        rb = db.step(q)
        ra = pend[-1].result()
        np.testing.assert_array_equal(ra.cert, rb.cert)
        np.testing.assert_array_equal(da.out.cpu().numpy(), db.out.cpu().numpy())
    bad = torch.full((U, 1, 128), float("nan"), dtype=torch.float16, device="cuda")
    t0 = ca.num_tokens
    pl0 = ca.partial_len_t.clone()
    ca.append(bad, bad, validate="defer")
    with pytest.raises(ValueError):
        da.step_async(qs[0]).result()
    assert torch.equal(ca.partial_len_t, pl0) and ca.num_tokens == t0  # nothing appended
    ca.append(k[:, :1], v[:, :1], validate="defer")  # the cache keeps working
    da.step_async(qs[1]).result()
    assert ca.num_tokens == t0 + 1


def test_step_async_out_buffers_and_host_report(ck):
    """The serving-loop path -- bound report written into pinned host memory by the
    step's last kernel, outputs into caller buffers (out=), device float64 queries
    read in place -- equals the synchronous step bit for bit: outputs,
    certificates, page statistics; the report's certificates equal the device
    certificate array; float32 / host queries (the copy path) give the same."""
    rng = np.random.default_rng(22)
    U, n = 5, 2100
    k = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    v = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    ca, cb = ck.DeviceKVCache(U, n + 32), ck.DeviceKVCache(U, n + 32)
    ca.append(k, v)
    cb.append(k, v)
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=12)
    da = ck.CertifiedDecoder(ca, pol, n_heads=4, scratch=ck.ScratchCache(ca.max_blocks))
    db = ck.CertifiedDecoder(cb, pol, n_heads=4, scratch=ck.ScratchCache(cb.max_blocks))
    od = [torch.full((U, 4, 128), float("nan"), device="cuda") for _ in range(2)]
    kn = torch.from_numpy(rng.standard_normal((6, U, 1, 128))).half().cuda()
    for i in range(6):
        q = torch.from_numpy(rng.standard_normal((U, 4, 128))).cuda()
        pa = da.step_async(q, out=od[i % 2])
        if i % 2 == 0:  # the copy path: host data, or a strided device view
            qb = q.cpu().numpy()
        else:
            qw = torch.zeros((U, 4, 256), dtype=torch.float64, device="cuda")
            qw[..., ::2] = q
            qb = qw[..., ::2]
        rb = db.step(qb)
        ra = pa.result()
        assert ra.out.data_ptr() == od[i % 2].data_ptr()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ra.cert, rb.cert)
        np.testing.assert_array_equal(ra.page_stats, rb.page_stats)
        assert torch.equal(od[i % 2], db.out)
        rep = da.cert_buf.cpu().numpy().view(ck.engine.CERT_DTYPE).reshape(U, 4)
        np.testing.assert_array_equal(ra.cert, rep)
        ca.append(kn[i], kn[i], validate=False)
        cb.append(kn[i], kn[i], validate=False)
    # the float32 query (copy path) on the async side too
    q = torch.from_numpy(rng.standard_normal((U, 4, 128))).cuda()
    ra = da.step_async(q.float()).result()
    rb = db.step(q.float())
    np.testing.assert_array_equal(ra.cert, rb.cert)
    assert torch.equal(da.out, db.out)


@pytest.mark.parametrize("env", [{"CKV_NO_STASH": "1"}, {"CKV_CHUNKS": "2"}, {"CKV_SEPARATE_LRU": "1"},
                                 {"CKV_SEPARATE_UNION": "1"}],
                         ids=["no_stash", "chunks2", "separate_lru", "separate_union"])
def test_alternate_paths_bit_identical(ck, monkeypatch, env):
    """The A/B knobs switch between code paths that compute the same values: the
    phase-1 score stash (pass A's scores reused by pass B), unit-chunked overlap of
    the tail kernels, the fused vs separate LRU scratch accounting and the union
    list built by the last selection CTA vs its own launch.  Outputs,
    certificates and page statistics must be bit-identical to the default path."""
    rng = np.random.default_rng(33)
    U, n = 20, 3000
    k = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    v = torch.from_numpy(rng.standard_normal((U, n, 128))).half().cuda()
    qs = [torch.from_numpy(rng.standard_normal((U, 4, 128))).cuda() for _ in range(4)]
    kn = torch.from_numpy(rng.standard_normal((4, U, 1, 128))).half().cuda()
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=24)

    def run():
        cache = ck.DeviceKVCache(U, n + 16)
        cache.append(k, v)
        dec = ck.CertifiedDecoder(cache, pol, n_heads=4, scratch=ck.ScratchCache(cache.max_blocks))
        outs, certs, pages = [], [], []
        stashed = 0
        for i, q in enumerate(qs):
            r = dec.step(q)
            if getattr(dec, "stash_epoch", None) is not None:
                stashed += int(((dec.stash_epoch >> 4) == dec.st.epoch).sum())
            outs.append(dec.out.cpu().numpy().copy())
            certs.append(np.array(r.cert, copy=True))
            pages.append(None if r.page_stats is None else np.array(r.page_stats, copy=True))
            cache.append(kn[i], kn[i])
        return outs, certs, pages, stashed

    base = run()
    assert base[3] > 0  # the default path did use the stash
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    alt = run()
    for s in range(len(qs)):
        np.testing.assert_array_equal(alt[0][s], base[0][s], err_msg=f"output step {s}")
        np.testing.assert_array_equal(alt[1][s], base[1][s], err_msg=f"certificates step {s}")
        if base[2][s] is not None:
            np.testing.assert_array_equal(alt[2][s], base[2][s], err_msg=f"page stats step {s}")


# ---- the bound report of a run manifest (certkv run, cli.py:98-117) -------------------

def _walk(a, b, path, tol):
    """Recursive comparison: same keys in the same order, equal integers / booleans /
    strings, floats within ``tol`` relative (the unmodified reference keeps fp64
    metadata the device narrows)."""
    if isinstance(a, dict):
        assert isinstance(b, dict) and list(a) == list(b), (path, list(a), list(b))
        for k in a:
            _walk(a[k], b[k], f"{path}.{k}", tol)
    elif isinstance(a, list):
        assert isinstance(b, list) and len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _walk(x, y, f"{path}[{i}]", tol)
    elif isinstance(a, float) and not isinstance(b, bool):
        assert isinstance(b, (int, float)), path
        assert abs(a - b) <= tol * max(abs(a), abs(b)) + 1e-12, (path, a, b)
    else:
        assert type(a) is type(b) and a == b, (path, a, b)


def test_run_manifest_matches_reference_cli(ck, tmp_path, monkeypatch):
    """``run_manifest`` on the manifest the golden script ran through the unmodified
    reference CLI (tests/golden/telemetry_ref.jsonl): the same lines, key sets and key
    order (sorted, compact JSON), the same header apart from the kernel backend's
    name, identical decisions, events, rung counts, scratch hits / misses and page-in
    bytes, certificate floats within the narrowing tolerance."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    monkeypatch.chdir(root)
    out = str(tmp_path / "run.jsonl")
    ck.run_manifest("tests/golden/telemetry_manifest.json", out)
    ref = open(os.path.join(root, "tests", "golden", "telemetry_ref.jsonl")).read().splitlines()
    dev = open(out).read().splitlines()
    assert len(dev) == len(ref)
    r0, d0 = json.loads(ref[0]), json.loads(dev[0])
    assert r0.pop("kernel_backend") == "pure" and d0.pop("kernel_backend") == "b200"
    assert d0 == r0
    for i, (r, d) in enumerate(zip(ref[1:], dev[1:])):
        _walk(json.loads(r), json.loads(d), f"line{i + 1}", 5e-3)
