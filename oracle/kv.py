"""One KV head's tiered store and the LRU scratch, restated from cache.py.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.
"""

from collections import OrderedDict

import numpy as np

from . import quant


class Tier2Lost(RuntimeError):
    """Mirror of cache.Tier2UnavailableError (cache.py:29-34)."""


class PagingFault(RuntimeError):
    """Mirror of cache.PagingError (cache.py:37-39)."""


def _f32_up(x):
    """float32 rounded toward +inf, as a Python float (the device's annotation width)."""
    f = np.float32(x)
    if float(f) < x:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


class OracleKV:
    """Block-organised store for one KV head (cache.py:49-224).

    Full blocks keep the INT8/INT4 payload plus metadata; ``narrow`` selects
    which metadata the reconstruction views use (see oracle/__init__.py).
    Tier-2 keeps the fp32 (binary16-rounded when ``ingest_binary16``)
    originals of full blocks; the trailing partial block stays at reference
    precision until it fills (cache.py:102-120).
    """

    def __init__(self, block_size, head_dim, group_size=16,
                 ingest_binary16=False, narrow=False):
        if head_dim % group_size:
            raise ValueError(
                f"group size {group_size} does not divide head dim {head_dim}")
        self.block_size = int(block_size)
        self.head_dim = int(head_dim)
        self.group_size = int(group_size)
        self.ingest_binary16 = bool(ingest_binary16)
        self.narrow = bool(narrow)
        # raw fp64 fit results (what the reference stores)
        self.kcodes, self.kscale, self.koffset = [], [], []
        self.vcodes, self.vscale, self.voffset = [], [], []
        self.eta, self.nu = [], []
        self.tier2_k, self.tier2_v = [], []
        self._pk, self._pv = [], []
        self.v_max = 0.0
        self._cache = {}

    # -- ingest / fill (cache.py:76-120) -------------------------------
    def _ingest(self, vec, what):
        x = np.asarray(vec, dtype=np.float64).reshape(-1)
        if x.shape[0] != self.head_dim:
            raise ValueError(f"{what} has length {x.shape[0]}, expected {self.head_dim}")
        if not np.all(np.isfinite(x)):
            raise ValueError(f"non-finite {what} entry")
        if self.ingest_binary16:
            x = x.astype(np.float16)
        return x.astype(np.float32)

    def append_token(self, key, value):
        self._pk.append(self._ingest(key, "key"))
        self._pv.append(self._ingest(value, "value"))
        if len(self._pk) == self.block_size:
            self._fill()

    def append_tokens(self, keys, values):
        keys = np.atleast_2d(np.asarray(keys))
        values = np.atleast_2d(np.asarray(values))
        if keys.shape != values.shape:
            raise ValueError("keys and values must have matching shapes")
        for k, v in zip(keys, values):
            self.append_token(k, v)

    def _fill(self):
        k32 = np.stack(self._pk)
        v32 = np.stack(self._pv)
        kc, ks, ko = quant.fit_key_block(k32)
        vc, vs, vo = quant.fit_value_block(v32, self.group_size)
        us, uo = self.value_meta(vs, vo)
        eta, nu = quant.value_annotations(
            v32, quant.dequant_values(vc, us, uo, self.group_size))
        if self.narrow:  # the device stores them as float32 rounded up
            eta, nu = _f32_up(eta), _f32_up(nu)
        self.kcodes.append(kc); self.kscale.append(ks); self.koffset.append(ko)
        self.vcodes.append(vc); self.vscale.append(vs); self.voffset.append(vo)
        self.eta.append(eta); self.nu.append(nu)
        self.tier2_k.append(k32); self.tier2_v.append(v32)
        self.v_max = max(self.v_max, nu)
        self._pk, self._pv = [], []
        self._cache = {}

    # -- metadata as used by reconstruction --------------------------------
    def key_meta(self, b):
        s, o = self.kscale[b], self.koffset[b]
        return quant.narrow_key_meta(s, o) if self.narrow else (s, o)

    def value_meta(self, s, o):
        return quant.narrow_value_meta(s, o) if self.narrow else (s, o)

    # -- shape (cache.py:124-134) -----------------------------------------
    @property
    def num_blocks(self):
        return len(self.kcodes)

    @property
    def partial_len(self):
        return len(self._pk)

    @property
    def num_tokens(self):
        return self.num_blocks * self.block_size + self.partial_len

    # -- reads (cache.py:138-206) -----------------------------------------
    def check_tier2(self, b):
        if self.tier2_k[b] is None or self.tier2_v[b] is None:
            raise Tier2Lost(f"full-precision originals for block {b} are unavailable")

    def orig_keys32(self, b):
        self.check_tier2(b)
        return self.tier2_k[b]

    def orig_values32(self, b):
        self.check_tier2(b)
        return self.tier2_v[b]

    def deq_key_rows(self):
        """(N_full, d) fp64 reconstruction of every full block's keys."""
        if "dk" not in self._cache:
            if self.num_blocks:
                rows = [quant.dequant_keys(self.kcodes[b], *self.key_meta(b))
                        for b in range(self.num_blocks)]
                self._cache["dk"] = np.concatenate(rows, axis=0)
            else:
                self._cache["dk"] = np.empty((0, self.head_dim))
        return self._cache["dk"]

    def deq_value_block32(self, b):
        """Tail values as the attend pass sees them: fp64 recon cast to fp32
        (cache.py:115-116)."""
        us, uo = self.value_meta(self.vscale[b], self.voffset[b])
        return quant.dequant_values(self.vcodes[b], us, uo,
                                    self.group_size).astype(np.float32)

    def tier2_key_rows(self):
        for b in range(self.num_blocks):
            self.check_tier2(b)
        if not self.num_blocks:
            return np.empty((0, self.head_dim))
        return np.concatenate(self.tier2_k, axis=0).astype(np.float64)

    def tier2_value_rows(self):
        for b in range(self.num_blocks):
            self.check_tier2(b)
        if not self.num_blocks:
            return np.empty((0, self.head_dim))
        return np.concatenate(self.tier2_v, axis=0).astype(np.float64)

    def partial_keys(self):
        if not self._pk:
            return np.empty((0, self.head_dim))
        return np.stack(self._pk).astype(np.float64)

    def partial_values(self):
        if not self._pv:
            return np.empty((0, self.head_dim))
        return np.stack(self._pv).astype(np.float64)

    def etas(self):
        return np.asarray(self.eta, dtype=np.float64)

    def key_scales_used(self):
        """(N_B, d) key scales as the Delta bound sees them."""
        if not self.num_blocks:
            return np.empty((0, self.head_dim))
        return np.stack([self.key_meta(b)[0] for b in range(self.num_blocks)])

    def corrupt_offset(self, b, channel, shift):
        """Fault injection equivalent of verification.py:420-428: shift one
        stored key offset (the device adds the shift to its fp32 offset)."""
        self.koffset[b] = self.koffset[b].copy()
        if self.narrow:
            o32 = np.float32(self.koffset[b][channel]) + np.float32(shift)
            self.koffset[b][channel] = float(o32)
        else:
            self.koffset[b][channel] += shift
        self._cache = {}


class OracleScratch:
    """Bounded LRU of promoted payloads with byte accounting (cache.py:243-291).

    Indices are processed in ascending order; a hit moves to MRU, a miss is
    loaded, admitted at MRU and the LRU entry is evicted past capacity; a
    zero-capacity scratch serves but retains nothing.
    """

    def __init__(self, capacity):
        if capacity < 0:
            raise ValueError("capacity must be non-negative")
        self.capacity = int(capacity)
        self.resident = OrderedDict()
        self.hits = self.misses = self.bytes_paged_in = 0

    def request(self, indices, loader, bytes_per_block):
        hits = misses = nbytes = 0
        payloads = {}
        for b in sorted(set(int(i) for i in indices)):
            if b in self.resident:
                self.resident.move_to_end(b)
                hits += 1
                payloads[b] = self.resident[b]
                continue
            payload = loader(b)
            misses += 1
            nbytes += bytes_per_block
            payloads[b] = payload
            if self.capacity > 0:
                self.resident[b] = payload
                while len(self.resident) > self.capacity:
                    self.resident.popitem(last=False)
        self.hits += hits
        self.misses += misses
        self.bytes_paged_in += nbytes
        return {"hits": hits, "misses": misses, "bytes": nbytes,
                "payloads": payloads}


def promote(scratch, kv, indices, kind):
    """cache.py:294-312: page originals of full blocks into ``scratch``."""
    idx = [int(i) for i in indices]
    for b in idx:
        if b < 0 or b >= kv.num_blocks:
            raise ValueError(f"block {b} is not a full block (cache has {kv.num_blocks})")
    if kind == "keys":
        loader = kv.orig_keys32
    elif kind == "values":
        loader = kv.orig_values32
    else:
        raise ValueError(f"unknown payload kind {kind!r}")
    return scratch.request(idx, loader, kv.block_size * kv.head_dim * 2)
