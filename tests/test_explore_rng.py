"""The uint32-level model of the reference's exploration draws
(oracle/explore_rng.py) against numpy itself; the device draws are checked
against numpy in tests/test_gpu_explore.py."""

import numpy as np
import pytest

from oracle import explore_rng as X


def _gen(seed):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 1))))


def test_philox_block_matches_numpy():
    g = _gen(5)
    st = g.bit_generator.state
    raw = [int(g.bit_generator.random_raw()) for _ in range(12)]
    ctr = [int(x) for x in st["state"]["counter"]]
    out = []
    for n in range(1, 4):
        c = ctr[:]
        c[0] += n
        out += X.philox4x64_10(c, st["state"]["key"])
    assert out == raw


@pytest.mark.parametrize("pop,size", [(1, 1), (2, 2), (5, 3), (100, 0), (100, 2), (7936, 164),
                                      (9999, 400), (10001, 199), (10001, 201), (10369, 212),
                                      (20000, 1000), (32000, 1600)])
def test_choice_matches_numpy(pop, size):
    for seed in range(3):
        a, b = _gen(seed), _gen(seed)
        if seed % 2:  # leave a buffered high half behind first
            a.integers(0, 7)
            b.integers(0, 7)
        ref = a.choice(pop, size=size, replace=False)
        s = X.Stream(b)
        got = X.choice(s, pop, size)
        s.close()
        assert list(ref) == got
        sa, sb = a.bit_generator.state, b.bit_generator.state
        assert (sa["state"]["counter"] == sb["state"]["counter"]).all()
        assert (sa["buffer"] == sb["buffer"]).all()
        assert (sa["buffer_pos"], sa["has_uint32"], sa["uinteger"]) == \
            (sb["buffer_pos"], sb["has_uint32"], sb["uinteger"])


def test_step_draws_match_sequential_choices():
    a, b = _gen(9), _gen(9)
    heads = [3, 10, 0, 50, 7, 7]
    got, _ = X.explore_draws(b, heads, 0.05, 400)
    for kp, g in zip(heads, got):
        pop, cnt = 400 - kp, min(400 - kp, round(0.05 * 400))
        assert sorted(a.choice(pop, size=cnt, replace=False)) == g
    assert a.bit_generator.state["buffer_pos"] == b.bit_generator.state["buffer_pos"]
