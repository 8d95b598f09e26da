"""Parity at the BASELINE.json configurations (VERDICT r1 "N1").

* C1 exactly (the reference's CPU case: 32 q / 8 KV heads, 4K, 16 steps) and
  the other frozen runs of the UNMODIFIED reference (tests/golden, produced by
  tests/golden/make_golden.py from /root/reference): device decisions must be
  identical except where the reference's own threshold distance
  (oracle/margins.py, frozen with the run) is below the stated tolerance;
  certificates and outputs within the tolerances below, which include the
  documented FP32 / FP16 metadata narrowing.
* The same runs against the oracle with the device's narrowing
  (OracleKV(narrow=True)): tight tolerances.
* Sampled units at the C2 / C3 / C5 shapes: the full 32-layer x 8-KV-head
  cache is built and stepped on the device; a sample of units (random ones,
  every Rung-3 unit up to a cap, and at C5 the corrupted unit and a neighbour
  of its layer) is copied from the device's FP16 Tier-2 into the oracle and
  compared head by head.

Every run prints "[parity <name>] head-steps=... decisions identical=..."
(also appended to $CKV_PARITY_LOG).
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.margins import TOL, TOL_REFERENCE, margins_from_oracle
from oracle.step import OraclePolicy, make_workload, run_workload as oracle_run
from parity_util import KINDS, Report, compare, dev_row, log, oracle_row

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RUNS = json.load(open(os.path.join(GOLD, "runs.json")))
D128 = sorted(n for n, s in RUNS.items() if s["workload"].get("head_dim") == 128)

# against the unmodified reference (fp64 metadata): value metadata FP16 moves eta
# (E_val) and the INT4 reconstructions (quantized outputs) by ~1e-3
NUM_REF = {"delta_h": 1e-5, "e_key_tight": 1e-4, "e_key_impl": 1e-4, "e_val": 5e-3,
           "est_tail_mass": 1e-4, "out_quant": 5e-3, "out_dense": 1e-5}
# against the oracle with the device's narrowing
NUM_NARROW = {"delta_h": 1e-5, "e_key_tight": 1e-4, "e_key_impl": 1e-4, "e_val": 1e-4,
              "est_tail_mass": 1e-4, "out_quant": 1e-4, "out_dense": 1e-5}
# C5 (outlier key channels x1000): the Phase-1 fixed-point quantum is 2^-21 of the
# largest |q_c sigma_c| of a block (k_pass_a), which the outlier channels
# raise ~1000-fold, so quantized scores carry ~1e-3 absolute error there: masses,
# tail mass / E_key and the score-based decisions get that tolerance; dense outputs
# at logits of a few hundred carry ~1e-7 x |s| of fp32 rounding
NUM_C5 = dict(NUM_NARROW, est_tail_mass=5e-3, e_key_tight=5e-3, e_key_impl=5e-3, out_dense=1e-4)
TOL_C5 = dict(TOL, cut=2e-3, ranking=2e-3, boundary=2e-3, canary=2e-3)
MAX_EXCEPTION_FRACTION = 0.05


@pytest.fixture(scope="module")
def ck():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    assert torch.cuda.is_available()
    return ck


def _device_run(ck, spec):
    cfg = ck.WorkloadConfig(ingest_binary16=True, **spec["workload"])
    wl = ck.generate_workload(cfg)
    kc, vc = spec["capacities"]
    rr = ck.run_workload(wl, ck.PolicyConfig(**spec["policy"]), kc, vc, keep_outputs=True,
                         keep_decisions=True)
    return cfg, rr


def _dev_rows(ck, cfg, rr):
    from paper_2605_20868_b200 import _lib
    rows = []
    for s, rec in enumerate(rr.step_records):
        for h, c in enumerate(rec["certificates"]):
            f = c["rung_flags"]
            rows.append({"promoted": rr.decisions[s][h][0], "vprom": rr.decisions[s][h][1],
                         "k_star": c["k_star"],
                         "flags": (f["rung1"], f["rung2"], f["rung3"], f["rung4"]),
                         "kind": c["returned_kind"], "delta_h": c["delta_h"],
                         "e_key_tight": c["e_key_tight"], "e_key_impl": c["e_key_impl"],
                         "e_val": c["e_val"], "est_tail_mass": c["est_tail_mass"],
                         "output": rr.outputs[s][h]})
    return rows


def _finish(rep, capped=True):
    """No failures; near-threshold exceptions are allowed (each one printed with
    its margins), and against the oracle with the device's own narrowing they
    must stay rare (a systematic drift would show up there first)."""
    log(rep)
    assert not rep.failures, rep.failures[:5]
    if capped:
        assert len(rep.exceptions) <= MAX_EXCEPTION_FRACTION * rep.n, rep.exceptions[:5]


@pytest.mark.parametrize("name", D128)
def test_device_vs_unmodified_reference(ck, name):
    spec = RUNS[name]
    z = np.load(os.path.join(GOLD, f"run_{name}.npz"))
    cfg, rr = _device_run(ck, spec)
    rep = Report(f"{name} vs reference")
    from oracle.margins import FIELDS
    for i, d in enumerate(_dev_rows(ck, cfg, rr)):
        row = z["cert"][i]
        p, v = z["promoted"][i], z["value_promotions"][i]
        ref = {"promoted": p[p >= 0].tolist(), "vprom": v[v >= 0].tolist(),
               "k_star": int(row[8]), "flags": tuple(bool(x) for x in row[10:14]),
               "kind": KINDS[int(row[9])], "delta_h": row[2], "e_key_tight": row[3],
               "e_key_impl": row[4], "e_val": row[5], "est_tail_mass": row[6],
               "output": z["outputs"][i]}
        margins = dict(zip(FIELDS, z["margins"][i]))
        compare(rep, f"step {int(row[0])} head {int(row[1])}", d, ref, margins, TOL_REFERENCE,
                NUM_REF)
    _finish(rep, capped=False)


@pytest.mark.parametrize("name", ["c1", "gauss16k", "sink8k_vtol", "greedy", "explore"])
def test_device_vs_oracle_narrow(ck, name):
    """Same runs against the oracle with the device's metadata widths: every
    number to the tight tolerances; telemetry identical when no decision sat
    near a threshold."""
    spec = RUNS[name]
    cfg, rr = _device_run(ck, spec)
    ow = make_workload(ingest_binary16=True, narrow=True, **spec["workload"])
    pol = OraclePolicy(**spec["policy"])
    ref = oracle_run(ow, pol, *spec["capacities"])
    rep = Report(f"{name} vs oracle(narrow)")
    rows = _dev_rows(ck, cfg, rr)
    i = 0
    for s, res in enumerate(ref["results"]):
        for h, r in enumerate(res):
            compare(rep, f"step {s} head {h}", rows[i], oracle_row(r),
                    margins_from_oracle(r, pol), TOL, NUM_NARROW)
            i += 1
    _finish(rep)
    if not rep.exceptions:
        for drec, orec in zip(rr.step_records, ref["records"]):
            assert drec["events"] == orec["events"]
            assert drec["key_scratch"] == orec["key_scratch"]
            assert drec["value_scratch"] == orec["value_scratch"]
            assert drec["bytes_paged_in"] == orec["bytes_paged_in"]
            assert drec["rung4_staging_bytes"] == orec["rung4_staging_bytes"]


# ---- sampled units at the C2 / C3 / C4 / C5 shapes ---------------------------------

# name: (context, adversarial, Tier-2 placement, v_tol).  C4 runs one sequence of its
# batch of 32 (256 units): 16K context, Tier-2 in pinned host RAM behind a scratch
# that holds every block (misses paged in by pass B), the tight v_tol that makes
# Rung 2 promote values.
SHAPES = {"c2": (32768, False, "device", None), "c3": (131072, False, "device", None),
          "c4": (16384, False, "host", 1e-3), "c5": (65536, True, "device", None)}
LAYERS, KV_HEADS, NH = 32, 8, 4


def _build(ck, ctx, adversarial, seed=77, tier2="device"):
    U = LAYERS * KV_HEADS
    cache = ck.DeviceKVCache(U, ctx + 64, tier2=tier2)
    g = torch.Generator(device="cuda").manual_seed(seed)
    chunk = max(16, min(4096, (1 << 22) // U))
    for pos in range(0, ctx, chunk):  # the bench's prefill recipe (bench.py)
        n = min(chunk, ctx - pos)
        kk = torch.randn((U, n, 128), generator=g, device="cuda")
        vv = torch.randn((U, n, 128), generator=g, device="cuda").half()
        if adversarial:
            kk[:, :, 3] *= 1000.0
            kk[:, :, 77] *= 1000.0
            if pos == 0 and n >= 32:
                kk[:, 16:32] = kk[:, 0:16] + 1e-4 * torch.randn_like(kk[:, 0:16])
        cache.append(kk.half(), vv, validate=False)
    faults = []
    if adversarial:
        rs = np.random.default_rng(5)
        for b in rs.choice(cache.num_blocks, size=8, replace=False):
            f = (int(b), int(rs.integers(0, 128)), float(rs.choice([-1.0, 1.0]) * 5.0e4))
            cache.corrupt_offset(0, *f)
            faults.append(f)
    q = torch.randn((U, NH, 128), generator=g, device="cuda", dtype=torch.float64)
    return cache, q, faults


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_sampled_units_at_baseline_shape(ck, name):
    from paper_2605_20868_b200 import _lib
    ctx, adversarial, tier2, v_tol = SHAPES[name]
    cache, q, faults = _build(ck, ctx, adversarial, tier2=tier2)
    U = cache.n_units
    groups = np.arange(U) % LAYERS  # kv-major units: step-wide Rung 4 per layer
    vkw = {} if v_tol is None else {"v_tol": v_tol}
    pol = ck.PolicyConfig(exploration_rate=0.0, **vkw)
    opol = OraclePolicy(exploration_rate=0.0, **vkw)
    scratch = ck.ScratchCache(cache.max_blocks) if tier2 == "host" else None
    dec = ck.CertifiedDecoder(cache, pol, n_heads=NH, rung4_group=groups, scratch=scratch)
    res = dec.step(q)
    if v_tol is not None:  # the tight v_tol promotes values somewhere in the step
        assert int(res.cert["n_value_promoted"].sum()) > 0
    if tier2 == "host":  # every promoted block was paged into its HBM slot
        assert int(res.page_stats[:, 1].sum()) > 0
    out = res.out.double().cpu().numpy()
    # the step-wide resolution against the device's own per-head requests
    r4 = np.array([[bool(int(res.cert[u, h]["flags"]) & (_lib.F_CANARY | _lib.F_NUMERIC))
                    for h in range(NH)] for u in range(U)])
    layer_r4 = np.zeros(LAYERS, bool)
    np.logical_or.at(layer_r4, groups, r4.any(1))
    assert np.array_equal(res.kinds == 2, np.repeat(layer_r4[groups][:, None], NH, 1))
    rs = np.random.default_rng(1)
    sample = set(int(u) for u in rs.choice(U, 2, replace=False))
    own_r3 = [int(u) for u in np.nonzero((res.kinds == 1).any(1))[0]]
    sample |= set(own_r3[:2])
    vprom = [int(u) for u in np.nonzero((res.cert["n_value_promoted"] > 0).any(1))[0]]
    sample |= set(vprom[:2])  # units whose heads promote values (C4's tight v_tol)
    if adversarial:
        assert layer_r4[0] and not layer_r4[1:].any()
        sample |= {0, LAYERS}  # the corrupted unit and another KV head of layer 0
    rep = Report(f"{name} sampled units {sorted(sample)} of {U} at {ctx}")
    tol, num = (TOL_C5, NUM_C5) if adversarial else (TOL, NUM_NARROW)
    for u in sorted(sample):
        k, v = cache.tier2_rows(u)
        vscale = float(v.float().pow(2).mean().sqrt())
        kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
        kv.append_tokens(k.double().cpu().numpy(), v.double().cpu().numpy())
        if adversarial and u == 0:
            for f in faults:
                kv.corrupt_offset(*f)
        for h in range(NH):
            qh = q[u, h].cpu().numpy()
            r = oracle.decode_step(qh, kv, opol)
            kind, o_ref = None, None
            if layer_r4[groups[u]]:  # step-wide Rung 4: every head of the layer is dense
                kind, o_ref = "dense_all_heads", oracle.dense_output(qh, kv)
            d = dev_row(res.cert[u, h], res.kinds[u, h], res.promoted(u, h),
                        res.value_promotions(u, h), out[u, h], _lib)
            ref = oracle_row(r, kind, o_ref)
            ref["vscale"] = vscale
            compare(rep, f"unit {u} head {h}", d, ref, margins_from_oracle(r, opol), tol, num)
    del dec, cache, scratch
    torch.cuda.empty_cache()
    _finish(rep)
