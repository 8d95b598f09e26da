"""Exploration draws of the reference, restated at the level of the uint32
stream -- the model the device's exploration draws (csrc/explore_draw.cu)
are checked against.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference draws ``rng.choice(len(tail), count, replace=False)`` per
q-head (fallback.py:212-218) from the workload's numpy Philox generator
(harness.py:348).  numpy 2.x implements that as (random/_generator.pyx
choice(), src/distributions): Philox4x64-10 64-bit outputs, uint32 draws taken
low half first with the high half buffered, ``random_bounded_uint64`` by
Lemire's multiply-shift with rejection, then Floyd's algorithm + shuffle, or a
tail Fisher-Yates when ``pop > 10000 and size > pop // 50``.  ``choice`` below
reproduces the result and the generator's final state bit for bit
(tests/test_explore_rng.py checks it against numpy itself) and counts the
Lemire rejections, which the device has to account for.
"""

import numpy as np

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK64 = (1 << 64) - 1


def philox4x64_10(ctr, key):
    """One Philox4x64 block, 10 rounds (Random123 constants)."""
    c, k = [int(x) for x in ctr], [int(x) for x in key]
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK64, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK64]
        k = [(k[0] + W0) & MASK64, (k[1] + W1) & MASK64]
    return c


class Stream:
    """uint32 draws as numpy's Philox bit generator hands them out, driving the
    generator itself (random_raw) so its state stays the reference's."""

    def __init__(self, rng):
        self.bg = rng.bit_generator
        st = self.bg.state
        self.has, self.uint = st["has_uint32"], st["uinteger"]
        self.draws = self.rejections = 0

    def u32(self):
        self.draws += 1
        if self.has:
            self.has = 0
            return self.uint
        x = int(self.bg.random_raw())
        self.has, self.uint = 1, x >> 32
        return x & 0xFFFFFFFF

    def bounded(self, n):
        """random_bounded_uint64(0, n) for n < 2^32 - 1 (Lemire, with rejection)."""
        if n == 0:
            return 0
        ex = n + 1
        m = self.u32() * ex
        if (m & 0xFFFFFFFF) < ex:
            thr = (0xFFFFFFFF - n) % ex
            while (m & 0xFFFFFFFF) < thr:
                self.rejections += 1
                m = self.u32() * ex
        return m >> 32

    def close(self):
        st = self.bg.state
        st["has_uint32"], st["uinteger"] = self.has, self.uint
        self.bg.state = st


def choice(stream, pop, size):
    """rng.choice(pop, size, replace=False) on the stream (shuffle=True)."""
    if pop > 10000 and size > pop // 50:  # tail shuffle over arange(pop)
        data = {}
        for i in range(pop - 1, max(pop - size, 1) - 1, -1):
            j = stream.bounded(i)
            data[i], data[j] = data.get(j, j), data.get(i, i)
        return [data.get(p, p) for p in range(pop - size, pop)]
    out, seen = [], set()
    for j in range(pop - size, pop):  # Floyd
        v = stream.bounded(j)
        v = j if v in seen else v
        seen.add(v)
        out.append(v)
    for i in range(size - 1, 0, -1):  # shuffle=True: draws only consume the stream here
        k = stream.bounded(i)
        out[i], out[k] = out[k], out[i]
    return out


def explore_draws(rng, heads, rate, n_blocks):
    """The draws of one step: ``heads`` = K' per q-head in the reference's head
    order; returns ([sorted positions per head], rejections) and advances rng."""
    s = Stream(rng)
    res = []
    for kp in heads:
        pop = n_blocks - int(kp)
        count = min(pop, int(round(rate * n_blocks))) if n_blocks else 0
        res.append(sorted(choice(s, pop, count)) if count > 0 else [])
    s.close()
    return res, s.rejections
