"""Bound-verification suites re-pointed at the device path (the reference's
``certkv verify``, verification.py:61-611).

Every property the reference checks against brute-force fp64 oracles is
checked here against what the CUDA path actually stores and returns:

* ``reconstruction_bounds`` -- INT8 keys / INT4 values fitted by the
  quantize-on-append kernel reconstruct every element to within half a
  quantization step of the stored (narrowed) metadata, plus the rounding the
  narrowing itself adds (verification.py:61-111);
* ``value_error_bound`` -- the weighted value error stays under sum rho*eta
  with the device's eta (fp32, rounded up), which stays under max eta
  (verification.py:117-151);
* ``output_soundness`` -- fast-path heads of ``run_decode_step``: the fp64
  two-pass recomputation of the mask-gated output from the device's own
  Tier-1 / Tier-2 lies within E_key(tight) + E_val of the exact output
  (verification.py:243-319); the device output's distance to that fp64
  recomputation is reported too;
* ``fallback_exactness`` -- dense rungs against the exact routine, the
  staging-cost formula, the canary fault injection (Rung 4) and Tier-2 loss as
  a hard error (verification.py:383-490);
* ``ranking_certificate`` -- whenever the depth-1 ranking + boundary
  certificate is issued on near-tie streams, the certified top block is the
  fp64 reference-key top block; with certification off the same streams
  mismatch (verification.py:493-556);
* the host-only lemmas (softmax perturbation, mass estimation, paper
  constants, storage accounting, GQA union) restated for completeness.

The device geometry is fixed (head_dim 128, block 16, value group 16, FP16
originals), so the reference's other head dims / group sizes are not swept;
inputs are generated binary16-exact.  ``run_suite`` keeps the reference's
suite names, default trial counts and ``PropertyResult`` lines.
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .cache import DeviceKVCache, TieredCache, storage_table
from .engine import (CertifiedDecoder, dense_attention, run_decode_step, rung3_per_head,
                     rung4_all_heads, rung4_staging_bytes)
from .errors import Tier2UnavailableError
from .harness import WorkloadConfig, generate_workload, gqa_union
from .policy import CAUSE_CANARY, PolicyConfig, e_key_bound

SLACK = 1e-12  # certifier.py:17 SOUNDNESS_SLACK
D, B, G = _lib.HEAD_DIM, _lib.BLOCK, _lib.GROUP


@dataclass
class PropertyResult:
    name: str
    trials: int
    violations: int
    details: dict = field(default_factory=dict)

    @property
    def ok(self):
        return self.violations == 0

    def line(self):
        extra = "".join(f" {k}={v}" for k, v in self.details.items())
        return (f"{self.name}: trials={self.trials} violations={self.violations}{extra} "
                f"[{'ok' if self.ok else 'VIOLATED'}]")


def _gen(seed, purpose=0):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, purpose))))


def _f16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def _softmax(x):
    w = np.exp(x - x.max(axis=-1, keepdims=True))
    return w / w.sum(axis=-1, keepdims=True)


# -- the device's stored blocks --------------------------------------------------


def _quantize_on_device(keys, values):
    """Append [n, 16, 128] fp16-exact key / value blocks to a one-unit device
    cache; return the stored Tier-1 (unpacked) and the annotations."""
    n = keys.shape[0]
    cache = DeviceKVCache(1, n * B)
    k = torch.from_numpy(keys.reshape(1, n * B, D)).to(cache.device).half()
    v = torch.from_numpy(values.reshape(1, n * B, D)).to(cache.device).half()
    cache.append(k, v)
    t1 = cache.read_tier1(0, 0, n)
    eta = cache.eta[0, :n].double().cpu().numpy()
    nu = cache.nu[0, :n].double().cpu().numpy()
    return t1, eta, nu


def _recon_keys(t1):
    """codes * scale + offset with the stored fp32 metadata, in fp64."""
    return (t1["kcodes"].astype(np.float64) * t1["kscale"].astype(np.float64)[:, None, :]
            + t1["koffset"].astype(np.float64)[:, None, :])


def _recon_values(t1):
    s = np.repeat(t1["vscale"].astype(np.float64), G, axis=-1)   # [n, 16, 128]
    o = np.repeat(t1["voffset"].astype(np.float64), G, axis=-1)
    return t1["vcodes"].astype(np.float64) * s + o


def reconstruction_bounds(trials=100_000, seed=0):
    """|recon - x| <= step/2 for every key and value element the device fitted.
    The bound is the stored step's half plus the rounding of the narrowing
    (fp32 key scale / offset: 2^-24 relative; fp16 value scale / offset: 2^-11
    relative); elements beyond the strict half-step alone are reported."""
    rng = _gen(seed, 10)
    checked = viol = strict = 0
    worst = 0.0
    remaining = trials
    while remaining > 0:
        n = min(4096, remaining)
        remaining -= n
        mag = 10.0 ** rng.uniform(-3, 3, (n, 1, 1))
        shift = rng.uniform(-4, 4, (n, 1, D))
        keys = _f16(rng.standard_normal((n, B, D)) * mag + shift)
        vmag = 10.0 ** rng.uniform(-3, 2, (n, 1, 1))
        vals = _f16(rng.standard_normal((n, B, D)) * vmag)
        t1, _, _ = _quantize_on_device(keys, vals)
        ks = t1["kscale"].astype(np.float64)[:, None, :]
        ko = np.abs(t1["koffset"].astype(np.float64))[:, None, :]
        err_k = np.abs(_recon_keys(t1) - keys)
        bound_k = ks / 2 + 2.0 ** -24 * (ko + 129.0 * ks) + 1e-12 * np.abs(keys)
        vs = np.repeat(t1["vscale"].astype(np.float64), G, axis=-1)
        vo = np.abs(np.repeat(t1["voffset"].astype(np.float64), G, axis=-1))
        err_v = np.abs(_recon_values(t1) - vals)
        bound_v = vs / 2 + 2.0 ** -11 * (vo + 15.0 * vs) + 2.0 ** -24
        viol += int((err_k > bound_k).sum() + (err_v > bound_v).sum())
        strict += int((err_k > ks / 2).sum() + (err_v > vs / 2).sum())
        worst = max(worst, float((err_k - ks / 2).max()), float((err_v - vs / 2).max()))
        checked += 2 * n
    return PropertyResult("reconstruction_bounds", checked, viol,
                          {"beyond_strict_half_step": strict,
                           "max_excess_over_half_step": float(max(worst, 0.0))})


def value_error_bound(trials=10_000, seed=0):
    """||sum_t w_t (v_hat_t - v_t)|| <= sum_b rho_b eta_b <= max_b eta_b with the
    device's reconstruction and its (rounded-up) eta annotations."""
    rng = _gen(seed, 20)
    done = viol = 0
    layouts = (2, 4, 8)
    i = 0
    while done < trials:
        nb = layouts[i % len(layouts)]
        i += 1
        n = min(512, trials - done)
        done += n
        mag = 10.0 ** rng.uniform(-2, 1, (n, 1, 1, 1))
        vals = _f16(rng.standard_normal((n, nb, B, D)) * mag)
        keys = np.zeros_like(vals)
        t1, eta, _ = _quantize_on_device(keys.reshape(-1, B, D), vals.reshape(-1, B, D))
        diff = (_recon_values(t1) - vals.reshape(-1, B, D)).reshape(n, nb * B, D)
        eta = eta.reshape(n, nb)
        scores = rng.standard_normal((n, nb * B)) * rng.uniform(0.3, 4.0, (n, 1))
        w = _softmax(scores)
        lhs = np.linalg.norm(np.einsum("nt,ntd->nd", w, diff), axis=-1)
        rho = w.reshape(n, nb, B).sum(-1)
        mid = (rho * eta).sum(-1)
        viol += int((lhs > mid + SLACK).sum() + (mid > eta.max(-1) + SLACK).sum())
    return PropertyResult("value_error_bound", done, viol)


# -- host-only lemmas (no device state involved) -------------------------------------


def softmax_perturbation(trials=100_000, seed=0):
    """Ratio envelope e^{+-2 Delta}, TV <= tanh(Delta), tail-restricted TV <=
    alpha (e^{2 Delta} - 1), and tightness at the ratio-polytope vertex."""
    rng = _gen(seed, 30)
    sizes = (2, 4, 8, 16, 32, 64)
    done = viol = 0
    i = 0
    while done < trials:
        t = sizes[i % len(sizes)]
        tail_only = i % 2 == 1
        i += 1
        n = min(4096, trials - done)
        done += n
        delta = rng.uniform(1e-4, 1.0, (n, 1))
        s = rng.standard_normal((n, t)) * rng.uniform(0.3, 5.0, (n, 1))
        pert = rng.uniform(-1.0, 1.0, (n, t)) * delta
        if tail_only:
            mask = rng.random((n, t)) < rng.uniform(0.1, 0.9, (n, 1))
            pert = pert * mask
        p, q = _softmax(s), _softmax(s + pert)
        env = np.exp(2.0 * delta)
        r = q / p
        viol += int(((r > env + SLACK) | (r < 1.0 / env - SLACK)).any(1).sum())
        tv = 0.5 * np.abs(p - q).sum(1)
        viol += int((tv > np.tanh(delta[:, 0]) + SLACK).sum())
        if tail_only:
            alpha = (p * mask).sum(1)
            viol += int((tv > alpha * (np.exp(2.0 * delta[:, 0]) - 1.0) + SLACK).sum())
    vertex = 0.0
    for d in (0.1, 0.18, 0.5, 1.0):
        up = math.exp(2.0 * d)
        a = 1.0 / (up + 1.0)
        pa, pb = np.array([a, 1.0 - a]), np.array([a * up, (1.0 - a) / up])
        vertex = max(vertex, abs(0.5 * np.abs(pa - pb).sum() - math.tanh(d)))
    viol += int(vertex > 1e-9)
    return PropertyResult("softmax_perturbation", done, viol, {"vertex_max_err": vertex})


def mass_estimation(trials=100_000, seed=0):
    """True block mass <= S'_b e^{m'_b - m' + 2 Delta}; true subset probability <=
    e^{2 Delta} x the quantized estimate."""
    rng = _gen(seed, 40)
    layouts = ((2, 4), (4, 8), (8, 8), (4, 16))
    done = viol = 0
    i = 0
    while done < trials:
        nb, bs = layouts[i % len(layouts)]
        i += 1
        n = min(4096, trials - done)
        done += n
        t = nb * bs
        delta = rng.uniform(1e-4, 1.0, (n, 1))
        s = rng.standard_normal((n, t)) * rng.uniform(0.3, 4.0, (n, 1))
        sq = s + rng.uniform(-1.0, 1.0, (n, t)) * delta
        bq = sq.reshape(n, nb, bs)
        mq = bq.max(-1)
        sumq = np.exp(bq - mq[..., None]).sum(-1)
        true_mass = np.exp(s.reshape(n, nb, bs) - s.max(-1)[:, None, None]).sum(-1)
        bound = sumq * np.exp(mq - sq.max(-1)[:, None] + 2.0 * delta)
        viol += int((true_mass > bound + SLACK).any(1).sum())
        subset = rng.random((n, t)) < rng.uniform(0.1, 0.9, (n, 1))
        pt = (_softmax(s) * subset).sum(1)
        pe = (_softmax(sq) * subset).sum(1)
        viol += int((pt > np.exp(2.0 * delta[:, 0]) * pe + SLACK).sum())
    return PropertyResult("mass_estimation", done, viol)


def paper_constants():
    """The operating-point constants: e^{2x0.18}, e^{3x0.18}, E_key at
    (v_max 1, Delta 0.18, tail 0.005) in both exponent modes, their ratio."""
    checks = {"exp_2delta": (math.exp(0.36), 1.433, 1e-3),
              "exp_3delta": (math.exp(0.54), 1.716, 1e-3),
              "e_key_tight": (e_key_bound(1.0, 0.18, 0.005, 2), 0.00615, 5e-4),
              "e_key_impl": (e_key_bound(1.0, 0.18, 0.005, 3), 0.00743, 5e-4)}
    bad = sum(abs(got - want) > tol for got, want, tol in checks.values())
    ratio = checks["e_key_impl"][0] / checks["e_key_tight"][0]
    bad += not 1.15 <= ratio <= 1.25
    det = {k: round(v[0], 6) for k, v in checks.items()}
    det["impl_widening"] = round(ratio, 4)
    return PropertyResult("paper_constants", len(checks) + 1, bad, det)


def storage_accounting():
    """288 B/token Tier-1 at d=128 (= the device's 4608-B record per 16-token
    block) and the d=64 column of the same formulas."""
    r = storage_table(128, 16, 16)
    want = {"key_codes_bytes": 128.0, "key_metadata_bytes": 64.0, "value_codes_bytes": 64.0,
            "value_metadata_bytes": 32.0, "tier1_total_bytes": 288.0, "dense_bytes": 512.0,
            "tier1_ratio": 0.5625}
    bad = sum(getattr(r, k) != v for k, v in want.items())
    bad += not 0.0 < r.annotation_bytes < 1.0
    bad += r.tier1_total_bytes * B != _lib.BLOCK_BYTES
    r64 = storage_table(64, 16, 16)
    bad += (r64.key_codes_bytes, r64.key_metadata_bytes, r64.value_codes_bytes,
            r64.value_metadata_bytes, r64.tier1_total_bytes, r64.dense_bytes) != \
        (64.0, 32.0, 32.0, 16.0, 144.0, 256.0)
    return PropertyResult("storage_accounting", len(want) + 3, int(bad))


def gqa_union_table():
    """Union fractions of the GQA working set (32 q-heads, K_max 128, Rung 1)
    within one point of the documented table, plus the degenerate forms."""
    want = {8192: 100.0, 32768: 99.0, 65536: 87.0, 131072: 64.0, 262144: 39.0}
    bad, det = 0, {}
    for n, pct in want.items():
        frac = gqa_union(n, 16, 128, 32, rung1_active=True)[1]
        det[f"n{n}"] = round(100 * frac, 1)
        bad += abs(100 * frac - pct) > 1.0
    bad += gqa_union(4096, 16, 2048, 32)[1] != 1.0
    bad += abs(gqa_union(65536, 16, 128, 1, rung1_active=True)[1] - 256 / 4096) > 1e-12
    return PropertyResult("gqa_union", len(want) + 2, int(bad), det)


# -- end-to-end properties through the certified call ---------------------------------


def _device_views(cache):
    """fp64 host views of one TieredCache's stored data: dequantized keys (fp32
    metadata), dequantized values (fp16 metadata), FP16 originals, partial."""
    dev = cache.dev
    nb = dev.num_blocks
    if nb:
        t1 = dev.read_tier1(0, 0, nb)
        kq, vq = _recon_keys(t1), _recon_values(t1)
    else:
        kq = vq = np.zeros((0, B, D))
    k, v = dev.tier2_rows(0)
    k = k.double().cpu().numpy()
    v = v.double().cpu().numpy()
    return kq, vq, k[:nb * B].reshape(nb, B, D), v[:nb * B].reshape(nb, B, D), \
        k[nb * B:], v[nb * B:]


def _masked_outputs(q, views, promoted, vprom):
    """fp64 two-pass outputs: the mask-gated one and the all-original one
    (verification.py:243-271 on the device's stored data)."""
    kq, vq, ko, vo, pk, pv = views
    nb = kq.shape[0]
    pm = np.zeros(nb, bool)
    pm[list(promoted)] = True
    vm = np.zeros(nb, bool)
    vm[list(vprom)] = True
    kg = np.where(pm[:, None, None], ko, kq).reshape(-1, D)
    vg = np.where(vm[:, None, None], vo, vq).reshape(-1, D)
    inv = 1.0 / math.sqrt(D)

    def attend(k, v):
        k = np.concatenate([k, pk])
        v = np.concatenate([v, pv])
        s = k @ q * inv
        w = np.exp(s - s.max())
        return (w / w.sum()) @ v

    return attend(kg, vg), attend(ko.reshape(-1, D), vo.reshape(-1, D))


def output_soundness(trials=10_000, seed=0, max_tokens=4096):
    """Fast-path heads: ||O_quant - O_ref|| <= E_key(tight) + E_val, both outputs
    recomputed in fp64 from the device's stored Tier-1 / Tier-2."""
    rng = _gen(seed, 50)
    n_caches = max(1, min(100, trials // 100))
    per = -(-trials // n_caches)
    viol = fast = done = 0
    worst, dev_err = math.inf, 0.0
    for _ in range(n_caches):
        n = int(np.exp(rng.uniform(np.log(4), np.log(max_tokens))))
        vscale = 10.0 ** rng.uniform(-2.0, 0.5)
        cache = TieredCache(16, D, 16, ingest_binary16=True, max_tokens=n + 16)
        cache.append_tokens(_f16(rng.standard_normal((n, D))),
                            _f16(rng.standard_normal((n, D)) * vscale))
        nb = cache.num_blocks
        policy = PolicyConfig(k_max=int(rng.choice([2, 4, 8, 32, 128])),
                              k_min=min(2, max(1, nb)) if nb else 0,
                              rung1_enabled=bool(rng.integers(2)), exploration_rate=0.0)
        views = _device_views(cache)
        for _ in range(per):
            if done >= trials:
                break
            done += 1
            q = rng.standard_normal(D)
            res = run_decode_step(q, cache, policy)
            cert = res.certificate
            if cert.is_dense:
                continue
            fast += 1
            o_quant, o_ref = _masked_outputs(q, views, res.decision.promoted, res.value_promotions)
            err = float(np.linalg.norm(o_quant - o_ref))
            bound = cert.e_key_tight + cert.e_val
            viol += err > bound + SLACK
            worst = min(worst, bound + SLACK - err)
            dev_err = max(dev_err, float(np.abs(res.output - o_quant).max()
                                         / max(np.abs(o_quant).max(), 1e-30)))
    return PropertyResult("output_soundness", done, int(viol),
                          {"fast_path_steps": fast,
                           "worst_margin": float(worst) if fast else None,
                           "device_vs_fp64_masked_output_max_rel": dev_err})


def _random_cache(rng, max_tokens=200):
    n = int(rng.integers(1, max_tokens))
    cache = TieredCache(16, D, 16, ingest_binary16=True, max_tokens=max_tokens + 16)
    cache.append_tokens(_f16(rng.standard_normal((n, D))), _f16(rng.standard_normal((n, D))))
    return cache


def sink_cache(seed=0, n_blocks=6):
    """verification.py:405-417's construction at d=128: block 0 dominates."""
    rng = _gen(seed, 60)
    w = rng.standard_normal(D)
    w /= np.linalg.norm(w)
    keys = rng.standard_normal((n_blocks * B, D))
    keys[:B] = 2.0 * np.sqrt(D) / 3.0 * w + 0.1 * keys[:B]
    cache = TieredCache(16, D, 16, ingest_binary16=True, max_tokens=n_blocks * B + 16)
    cache.append_tokens(_f16(keys), _f16(rng.standard_normal((n_blocks * B, D))))
    return cache, 3.0 * w + rng.standard_normal(D)


def corrupt_block_offset(cache, block, query):
    """Fault injection (verification.py:420-428): shift the stored key offset of
    the query's strongest channel by 10 (1 + sum |key scales|)."""
    ch = int(np.argmax(np.abs(query)))
    ks = cache.dev.read_tier1(0, block, 1)["kscale"][0].astype(np.float64)
    cache.dev.corrupt_offset(0, block, ch, float(10.0 * (1.0 + np.abs(ks).sum())))


def fallback_exactness(trials=1000, seed=0, dense_rtol=1e-5):
    """Dense rungs: the standalone rung-3 / rung-4 calls are the exact routine
    bit for bit; the certified call's in-step dense rung (k_dense, fp32 over the
    FP16 originals) matches it to ``dense_rtol``; the staging formula; metadata
    corruption trips the canary into Rung 4 with a dense output and a zero
    returned E_key; a lost Tier-2 block is a hard error."""
    rng = _gen(seed, 70)
    viol = 0
    worst = 0.0
    force_r3 = PolicyConfig(k_min=1, k_max=1, ranking_depth=2, rung1_enabled=False,
                            exploration_rate=0.0)
    for _ in range(trials):
        cache = _random_cache(rng)
        q = rng.standard_normal(D)
        exact = dense_attention(q, cache)
        viol += not np.array_equal(rung3_per_head(q, cache), exact)
        outs, staging = rung4_all_heads([q, q], [cache, cache])
        viol += sum(not np.array_equal(o, exact) for o in outs)
        viol += staging != 2 * cache.num_tokens * D * 2
        if cache.num_blocks:  # |F| = 1 < ranking depth 2: Rung 3 on the device
            r = run_decode_step(q, cache, force_r3)
            if r.certificate.returned_kind != "dense_per_head":
                viol += 1
            else:
                e = float(np.abs(r.output - exact).max() / max(np.abs(exact).max(), 1e-30))
                worst = max(worst, e)
                viol += e > dense_rtol
    viol += rung4_staging_bytes([131072] * 8, 128) != 536870912
    cache, q = sink_cache(seed)
    pol = PolicyConfig(exploration_rate=0.0)
    viol += any(e.rung == 4 for e in run_decode_step(q, cache, pol).events)
    corrupt_block_offset(cache, 0, q)
    tripped = run_decode_step(q, cache, pol)
    viol += not [e for e in tripped.events if e.rung == 4 and e.cause == CAUSE_CANARY]
    exact = dense_attention(q, cache)
    e = float(np.abs(tripped.output - exact).max() / np.abs(exact).max())
    worst = max(worst, e)
    viol += e > dense_rtol
    viol += tripped.certificate.returned_e_key != 0.0
    cache, q = sink_cache(seed + 1)
    cache.dev.drop_tier2(0, 0)
    try:
        run_decode_step(q, cache, PolicyConfig(exploration_rate=0.0))
        viol += 1
    except Tier2UnavailableError:
        pass
    return PropertyResult("fallback_exactness", trials + 4, int(viol),
                          {"in_step_dense_max_rel": worst})


def _reference_top_block(q, cache):
    """fp64 top block by reference-key log-mass, ties to the lower index."""
    nb = cache.num_blocks
    k, _ = cache.tier2_rows(0)
    s = (k[:nb * B].double().cpu().numpy() @ q / math.sqrt(D)).reshape(nb, B)
    m = s.max(1)
    lm = m + np.log(np.exp(s - m[:, None]).sum(1))
    return int(np.lexsort((np.arange(nb), -lm))[0])


def ranking_certificate(trials=10_000, seed=0):
    """Depth-1 ranking + boundary certificate on near-tie streams (d=128):
    every certified head-step's top block is the fp64 oracle's; the naive
    policy (no certification) mismatches on >= 1% of the same stream."""
    runs = max(1, min(100, trials // 100))
    steps = -(-trials // runs)
    policy = PolicyConfig(k_min=2, k_max=4, exploration_rate=0.0)
    naive = PolicyConfig.naive()
    cert_steps = r3_steps = viol = naive_steps = naive_miss = 0
    for run in range(runs):
        cfg = WorkloadConfig(kind="near_tie", n_tokens=96, head_dim=D, steps=steps,
                             seed=seed + run, ingest_binary16=True)
        for active in (True, False):
            wl = generate_workload(cfg)
            cache = wl.cache
            dec = CertifiedDecoder(cache, policy if active else naive, n_heads=1)
            for step in range(steps):
                q = wl.queries[step, 0]
                top = _reference_top_block(q, cache)
                res = dec.step(torch.from_numpy(q).reshape(1, 1, D).to(cache.device))
                nb = cache.num_blocks
                lm1 = dec.lm1[0, 0, :nb].double().cpu().numpy()
                lm2 = dec.lm2[0, 0, :nb].double().cpu().numpy()
                prom = set(int(b) for b in res.promoted(0, 0))
                if active:
                    if int(res.kinds[0, 0]) != 0 or int(res.cert[0, 0]["flags"]) & (
                            _lib.F_RANKING | _lib.F_BOUNDARY | _lib.F_CANARY):
                        r3_steps += 1
                    else:
                        cert_steps += 1
                        cand = sorted(prom)
                        best = min(cand, key=lambda b: (-lm2[b], b))
                        viol += best != top
                else:
                    naive_steps += 1
                    att = np.where(np.isin(np.arange(nb), list(prom)), lm2, lm1)
                    naive_miss += int(np.lexsort((np.arange(nb), -att))[0]) != top
                cache.append(torch.from_numpy(wl.new_keys[step])[:, None, :],
                             torch.from_numpy(wl.new_values[step])[:, None, :])
    rate = naive_miss / naive_steps if naive_steps else 0.0
    fails = viol + (cert_steps == 0 or r3_steps == 0) + (rate < 0.01)
    return PropertyResult("ranking_certificate", cert_steps + naive_steps, int(fails),
                          {"certified_steps": cert_steps, "rung3_steps": r3_steps,
                           "naive_mismatch_rate": round(rate, 4)})


# -- registry (verification.py:561-611) ---------------------------------------------------

SUITES = {
    "bounds": ("reconstruction_bounds", "value_error_bound", "softmax_perturbation",
               "mass_estimation", "output_soundness", "paper_constants"),
    "fallback": ("fallback_exactness", "ranking_certificate"),
    "storage": ("storage_accounting", "gqa_union"),
}

DEFAULT_TRIALS = {"reconstruction_bounds": 100_000, "value_error_bound": 10_000,
                  "softmax_perturbation": 100_000, "mass_estimation": 100_000,
                  "output_soundness": 10_000, "fallback_exactness": 1_000,
                  "ranking_certificate": 10_000}

RUNNERS = {"reconstruction_bounds": reconstruction_bounds, "value_error_bound": value_error_bound,
           "softmax_perturbation": softmax_perturbation, "mass_estimation": mass_estimation,
           "output_soundness": output_soundness, "paper_constants": paper_constants,
           "storage_accounting": storage_accounting, "gqa_union": gqa_union_table,
           "fallback_exactness": fallback_exactness, "ranking_certificate": ranking_certificate}


def run_suite(suite="all", trials=None, seed=0):
    """One named suite (or "all"): a list of PropertyResult."""
    if suite == "all":
        names = [n for grp in ("bounds", "fallback", "storage") for n in SUITES[grp]]
    elif suite in SUITES:
        names = list(SUITES[suite])
    else:
        raise ValueError(f"unknown suite {suite!r}; choose from {sorted(SUITES)} or 'all'")
    out = []
    for name in names:
        fn = RUNNERS[name]
        if name in DEFAULT_TRIALS:
            out.append(fn(trials=DEFAULT_TRIALS[name] if trials is None else trials, seed=seed))
        else:
            out.append(fn())
    return out
