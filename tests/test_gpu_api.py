"""GPU tests of the drop-in API surface: reference-style scratch objects in
run_decode_step, cache reset with a bound scratch, deferred append rejections,
and the evicting LRU at long context (state kept in global memory).

All calls go through the C ABI (libcertkv_b200.so)."""

from collections import OrderedDict

import numpy as np
import pytest
import torch

import oracle
from oracle.step import OraclePolicy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    assert torch.cuda.is_available()
    return ck


def test_run_decode_step_updates_caller_scratches(ck):
    """key_scratch / value_scratch passed the reference way (one ScratchCache per
    kind, harness.py:186-187) receive exactly the oracle's LRU accounting, and
    page_reports holds PageInReport objects (cache.py:230-240)."""
    rng = np.random.default_rng(11)
    k = rng.standard_normal((1500, 128)).astype(np.float16).astype(np.float64)
    v = rng.standard_normal((1500, 128)).astype(np.float16).astype(np.float64)
    cache = ck.TieredCache(16, 128, 16, ingest_binary16=True, max_tokens=2048)
    cache.append_tokens(k, v)
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=True)
    kv.append_tokens(k, v)
    ks, vs = ck.ScratchCache(20), ck.ScratchCache(5)
    oks, ovs = oracle.OracleScratch(20), oracle.OracleScratch(5)
    pol = ck.PolicyConfig(exploration_rate=0.0, k_max=8, v_tol=0.002)
    opol = OraclePolicy(exploration_rate=0.0, k_max=8, v_tol=0.002)
    for step in range(6):
        q = rng.standard_normal(128)
        a = ck.run_decode_step(q, cache, pol, key_scratch=ks, value_scratch=vs, step=step)
        b = oracle.decode_step(q, kv, opol, oks, ovs, step=step)
        assert sorted(a.decision.promoted) == b["promoted"].tolist()
        assert sorted(a.value_promotions) == b["value_promotions"].tolist()
        for kind in ("keys", "values"):
            rep = a.page_reports[kind]
            assert isinstance(rep, ck.cache.PageInReport)
            ob = b["pages"][kind]
            assert (rep.hits, rep.misses, rep.bytes) == (ob["hits"], ob["misses"], ob["bytes"])
            assert sum(r.bytes for r in [rep]) == ob["bytes"]
    assert (ks.hits, ks.misses, ks.bytes_paged_in) == (oks.hits, oks.misses, oks.bytes_paged_in)
    assert (vs.hits, vs.misses, vs.bytes_paged_in) == (ovs.hits, ovs.misses, ovs.bytes_paged_in)
    assert ks.hit_rate == pytest.approx(oks.hits / (oks.hits + oks.misses))
    assert vs.misses > 0 and ks.hits > 0


def test_reset_reinitialises_bound_scratch(ck):
    """After reset() and a different refill, a host-Tier-2 cache with a bound
    scratch gives the same step as a fresh cache (no stale resident slots)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    U, N = 2, 1200
    k1 = torch.randn((U, N, 128), generator=g, device="cuda").half()
    v1 = torch.randn((U, N, 128), generator=g, device="cuda").half()
    k2 = torch.randn((U, N, 128), generator=g, device="cuda").half()
    v2 = torch.randn((U, N, 128), generator=g, device="cuda").half()
    q = torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
    pol = ck.PolicyConfig(exploration_rate=0.0, v_tol=0.002)

    def run(cache, sc):
        dec = ck.CertifiedDecoder(cache, pol, n_heads=4, scratch=sc)
        r = dec.step(q)
        return r.out.clone(), r.cert.copy(), r.page_stats.copy()

    reused = ck.DeviceKVCache(U, N + 64, tier2="host")
    sc = ck.ScratchCache(4096)
    reused.append(k1, v1)
    run(reused, sc)
    reused.reset()
    assert sc.misses == 0  # counters restart with the emptied scratch
    reused.append(k2, v2)
    out_a, cert_a, ps_a = run(reused, sc)
    fresh = ck.DeviceKVCache(U, N + 64, tier2="host")
    fresh.append(k2, v2)
    out_b, cert_b, ps_b = run(fresh, ck.ScratchCache(4096))
    assert torch.equal(out_a, out_b)
    assert np.array_equal(cert_a, cert_b)
    assert np.array_equal(ps_a, ps_b) and ps_a[:, 1].sum() > 0  # every promoted block misses again


def test_deferred_rejection_reported_once(ck):
    """A rejected deferred append surfaces exactly once, through the first step
    result that observes it; steps enqueued later stay clean."""
    g = torch.Generator(device="cuda").manual_seed(5)
    U = 2
    cache = ck.DeviceKVCache(U, 1024)
    cache.append(torch.randn((U, 300, 128), generator=g, device="cuda").half(),
                 torch.randn((U, 300, 128), generator=g, device="cuda").half())
    dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4)
    q = torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
    good = torch.randn((U, 1, 128), generator=g, device="cuda").half()
    bad = good.clone()
    bad[1, 0, 3] = float("nan")
    pend = [dec.step_async(q)]
    cache.append(bad, good, validate="defer")
    for _ in range(4):
        pend.append(dec.step_async(q))
        cache.append(good, good, validate="defer")
    errors = 0
    for p in pend:
        try:
            p.result()
        except ValueError as e:
            assert "non-finite" in str(e)
            errors += 1
    assert errors == 1
    torch.cuda.synchronize()
    cache.resync()
    assert cache.num_tokens == 304  # the bad token was dropped, the 4 good ones kept
    with pytest.raises(ValueError, match="non-finite"):
        cache.append(bad, good)
    cache.append(good, good)  # and the next validated append is clean
    assert cache.num_tokens == 305


def _lru_sim(state, cap, requests):
    """ScratchCache.request (cache.py:261-286) over per-head ascending lists."""
    hits = misses = 0
    for req in requests:
        for b in sorted(set(req)):
            if b in state:
                state.move_to_end(b)
                hits += 1
            else:
                misses += 1
                if cap > 0:
                    state[b] = True
                    while len(state) > cap:
                        state.popitem(last=False)
    return hits, misses


def test_evicting_lru_at_long_context(ck):
    """Evicting scratch at 270K tokens (16.9K blocks: the LRU state no longer
    fits in shared memory, k_lru works on it in global memory): per-step hits /
    misses equal a host LRU fed with the device's own promotion decisions."""
    g = torch.Generator(device="cuda").manual_seed(9)
    U, N = 2, 270_000
    cache = ck.DeviceKVCache(U, N + 64)
    for pos in range(0, N, 30_000):
        n = min(30_000, N - pos)
        cache.append(torch.randn((U, n, 128), generator=g, device="cuda").half(),
                     torch.randn((U, n, 128), generator=g, device="cuda").half(), validate=False)
    assert cache.max_blocks >= 16384
    kcap, vcap = 1500, 300
    sc = ck.ScratchCache(kcap, vcap)
    pol = ck.PolicyConfig(exploration_rate=0.0, v_tol=2e-4)
    dec = ck.CertifiedDecoder(cache, pol, n_heads=4, scratch=sc)
    states = [(OrderedDict(), OrderedDict()) for _ in range(U)]
    for step in range(3):
        q = torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
        r = dec.step(q)
        for u in range(U):
            kh, km = _lru_sim(states[u][0], kcap, [r.promoted(u, h).tolist() for h in range(4)])
            vh, vm = _lru_sim(states[u][1], vcap, [r.value_promotions(u, h).tolist() for h in range(4)])
            assert r.page_stats[u].tolist() == [kh, km, vh, vm], (step, u)
    assert sum(len(s[0]) for s in states) == U * kcap  # the key scratch did evict
