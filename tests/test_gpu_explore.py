"""Exploration draws on the device (csrc/explore_draw.cu) against numpy's own
``rng.choice(len(tail), count, replace=False)`` in the reference's head order
(fallback.py:212-218), and the generator state it leaves behind; plus the
spot check running inside ``step_async`` with the generator attached."""

import numpy as np
import pytest
import torch

from oracle import explore_rng as X

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    return ck


def _gen(seed):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 1))))


def _same_state(a, b):
    sa, sb = a.bit_generator.state, b.bit_generator.state
    return ((sa["state"]["counter"] == sb["state"]["counter"]).all()
            and (sa["state"]["key"] == sb["state"]["key"]).all()
            and (sa["buffer"] == sb["buffer"]).all()
            and (sa["buffer_pos"], sa["has_uint32"], sa["uinteger"])
            == (sb["buffer_pos"], sb["has_uint32"], sb["uinteger"]))


def _cache(ck, U, N, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    cache = ck.DeviceKVCache(U, N + 64)
    for pos in range(0, N, 32768):
        n = min(32768, N - pos)
        cache.append(torch.randn((U, n, 128), generator=g, device="cuda").half(),
                     torch.randn((U, n, 128), generator=g, device="cuda").half(), validate=False)
    return cache, g


# (units, context, rate, seed, steps): Floyd at small and C3 sizes (the C3 stream
# with seed 2 meets a Lemire rejection in its first 3 steps), the tail shuffle past
# 10000 tail blocks, and the maximum rate
CASES = [(4, 3000, 0.02, 0, 3), (256, 131072, 0.02, 2, 3), (8, 170000, 0.02, 1, 2),
         (6, 20000, 0.05, 3, 3)]


@pytest.mark.parametrize("U,N,rate,seed,steps", CASES)
def test_device_draws_match_numpy(ck, U, N, rate, seed, steps):
    cache, g = _cache(ck, U, N, seed)
    dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=rate), n_heads=4)
    rng, ref, model = _gen(seed), _gen(seed), _gen(seed)
    rejections = 0
    for s in range(steps):
        q = torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
        res = dec.step(q, rng=rng)
        nb = cache.num_blocks
        pos = dec.explore_pos.cpu().numpy()
        kps = [int(res.cert[u, h]["k_star"]) for u in range(U) for h in range(4)]
        for i, kp in enumerate(kps):
            u, h = divmod(i, 4)
            pop, cnt = nb - kp, min(nb - kp, round(rate * nb))
            want = sorted(ref.choice(pop, size=cnt, replace=False)) if cnt > 0 else []
            assert int(res.explore_counts[u, h]) == cnt
            assert sorted(pos[u, h, :cnt].tolist()) == want, (s, u, h)
        _, r = X.explore_draws(model, kps, rate, nb)
        rejections += r
        assert _same_state(rng, ref), s
        cache.append(torch.randn((U, 1, 128), generator=g, device="cuda").half(),
                     torch.randn((U, 1, 128), generator=g, device="cuda").half())
    print(f"units={U} ctx={N}: {rejections} Lemire rejections in {steps} steps")
    if (U, N, seed) == (256, 131072, 2):
        assert rejections >= 1  # the rejection path was exercised


def test_step_async_with_exploration(ck):
    """An attached generator: every async step draws on the device in stream
    order; the results and the final state equal the synchronous steps'."""
    U, N = 8, 6000
    outs = {}
    for mode in ("sync", "async"):
        cache, g = _cache(ck, U, N, 7)
        dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.03), n_heads=4)
        rng = _gen(11)
        qs = [torch.randn((U, 4, 128), generator=g, device="cuda", dtype=torch.float64)
              for _ in range(4)]
        certs, counts = [], []
        if mode == "async":
            dec.attach_rng(rng)
            pend = [dec.step_async(q) for q in qs[:1]]
            for q in qs[1:]:
                pend.append(dec.step_async(q))
            res = [p.result() for p in pend]
            dec.detach_rng()
        else:
            res = [dec.step(q, rng=rng) for q in qs]
        outs[mode] = ([r.cert.tobytes() for r in res], [r.explore_counts.tolist() for r in res],
                      rng.bit_generator.state["buffer_pos"],
                      int(rng.bit_generator.state["state"]["counter"][0]))
    assert outs["sync"] == outs["async"]
