"""Device-resident tiered KV cache (Tier-1 INT8/INT4 + FP16 Tier-2).

``DeviceKVCache`` holds ``n_units`` KV-head caches (units = layers x KV heads
x sequences) in HBM; ``TieredCache`` is the single-KV-head drop-in for the
reference class (cache.py:49-224) built on a one-unit DeviceKVCache.

HBM layout per unit (see include/certkv_b200.h):
  tier1       u8  [max_blocks, 4608]   one contiguous record per 16-token block
  eta/nu/kscale_max f32 [max_blocks]   annotations (eta/nu: quantizer.py:207-217)
  partial_k/v f16 [16, 128]            trailing partial block
  tier2_k/v   f16 [max_blocks*16, 128] originals, in HBM or in pinned host RAM
"""

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import Tier2UnavailableError

D, B, G = _lib.HEAD_DIM, _lib.BLOCK, _lib.GROUP


def _k2_index():
    """natural [t][c] -> position in the fragment-ordered Tier-2 key block
    (k2_offset in csrc/common.cuh)."""
    t = np.arange(B)[:, None]
    c = np.arange(D)[None, :]
    kt, cc = c >> 4, c & 15
    lane = (t & 7) * 4 + ((cc & 7) >> 1)
    reg = (t >> 3) + 2 * (cc >> 3)
    return (kt * 256 + lane * 8 + reg * 2 + (cc & 1)).reshape(-1)


K2_INDEX = _k2_index()


def _v2_index():
    """natural [t][c] -> position in the fragment-ordered Tier-2 value block
    (v2_offset in csrc/common.cuh)."""
    t = np.arange(B)[:, None]
    c = np.arange(D)[None, :]
    g, r = c >> 4, c & 15
    lane = (r & 7) * 4 + ((t & 7) >> 1)
    reg = (r >> 3) + 2 * (t >> 3)
    return (g * 256 + lane * 8 + reg * 2 + (t & 1)).reshape(-1)


V2_INDEX = _v2_index()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class DeviceKVCache:
    """``n_units`` tiered KV caches on one GPU.

    Appends go through the quantize-on-append kernel (K1): tokens are FP16
    (binary16 ingest, the paper's Tier-2 width), every completed 16-token
    block is fitted in fp64 and written once (cache.py:102-120).
    """

    def __init__(self, n_units, max_tokens, device="cuda", tier2="device"):
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceKVCache needs a CUDA device (no CPU fallback)")
        if tier2 not in ("device", "host"):
            raise ValueError("tier2 must be 'device' or 'host'")
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.n_units = int(n_units)
        self.max_blocks = max(32, -(-int(max_tokens) // (B * 32)) * 32)  # multiple of 32 blocks
        self.tier2_location = tier2
        U, NB = self.n_units, self.max_blocks
        kw = dict(device=self.device)
        self.tier1 = torch.zeros((U, NB, _lib.BLOCK_BYTES), dtype=torch.uint8, **kw)
        self.eta = torch.zeros((U, NB), dtype=torch.float32, **kw)
        self.nu = torch.zeros((U, NB), dtype=torch.float32, **kw)
        self.kscale_max = torch.ones((U, NB), dtype=torch.float32, **kw)
        self.v_max_t = torch.zeros((U,), dtype=torch.float32, **kw)
        self.n_blocks_t = torch.zeros((U,), dtype=torch.int32, **kw)
        self.partial_len_t = torch.zeros((U,), dtype=torch.int32, **kw)
        self.partial_k = torch.zeros((U, B, D), dtype=torch.float16, **kw)
        self.partial_v = torch.zeros((U, B, D), dtype=torch.float16, **kw)
        if tier2 == "device":
            self.tier2_k = torch.zeros((U, NB * B, D), dtype=torch.float16, **kw)
            self.tier2_v = torch.zeros((U, NB * B, D), dtype=torch.float16, **kw)
        else:
            self.tier2_k = torch.zeros((U, NB * B, D), dtype=torch.float16).pin_memory()
            self.tier2_v = torch.zeros((U, NB * B, D), dtype=torch.float16).pin_memory()
        self.tier2_valid = torch.zeros((U, NB), dtype=torch.uint8, **kw)
        self.status = torch.zeros((8,), dtype=torch.int32, **kw)
        self.c = _lib.CkvCache(
            n_units=U, max_blocks=NB, tier1=_ptr(self.tier1), eta=_ptr(self.eta),
            nu=_ptr(self.nu), kscale_max=_ptr(self.kscale_max), v_max=_ptr(self.v_max_t),
            n_blocks=_ptr(self.n_blocks_t), partial_len=_ptr(self.partial_len_t),
            partial_k=_ptr(self.partial_k), partial_v=_ptr(self.partial_v),
            tier2_k=_ptr(self.tier2_k), tier2_v=_ptr(self.tier2_v),
            tier2_valid=_ptr(self.tier2_valid), status=_ptr(self.status))
        self._tokens = 0  # host mirror: every unit receives the same appends
        self._nonfinite_reported = 0  # rejected appends already raised (status word 0)
        self._scratches = weakref.WeakSet()  # ScratchCaches bound to this cache

    # -- shape ------------------------------------------------------------
    @property
    def num_tokens(self):
        return self._tokens

    def resync(self):
        """Re-read the token count from the device (after a deferred append was
        rejected there, the host mirror counted tokens the device refused)."""
        nb = int(self.n_blocks_t[0].item())
        self._tokens = nb * B + int(self.partial_len_t[0].item())

    @property
    def num_blocks(self):
        return self._tokens // B

    @property
    def partial_len(self):
        return self._tokens % B

    @property
    def tier1_bytes_per_token(self):
        return _lib.BLOCK_BYTES / B

    # -- writes -----------------------------------------------------------
    def append(self, keys, values, validate=True):
        """Append n tokens to every unit: keys/values [n_units, n, 128].

        Inputs are cast to FP16 (binary16 ingest, cache.py:82-84).  With
        ``validate`` the sticky device status is read back and a non-finite
        entry raises ValueError; the kernel never mutates the cache when any
        input is non-finite.  ``validate="defer"`` skips that host sync: the
        device still rejects the block, and the ValueError is raised by the
        next decode step's result (which reads the status with the
        certificates).
        """
        k = torch.as_tensor(keys, device=self.device)
        v = torch.as_tensor(values, device=self.device)
        if k.dim() == 2:
            k, v = k[:, None, :], v[:, None, :]
        if k.shape != v.shape:
            raise ValueError("keys and values must have matching shapes")
        if k.dim() != 3 or k.shape[0] != self.n_units or k.shape[2] != D:
            raise ValueError(f"expected [n_units={self.n_units}, n, {D}], got {tuple(k.shape)}")
        n = int(k.shape[1])
        if n == 0:
            return
        if (self._tokens + n) // B > self.max_blocks:
            raise ValueError(f"append of {n} tokens exceeds the cache capacity "
                             f"({self.max_blocks * B} tokens)")
        k16, v16 = self._to_half(k), self._to_half(v)
        defer = validate == "defer"
        if validate and not defer and (k.dtype != torch.float16):
            # a finite fp32/fp64 value can overflow binary16: the reference
            # rejects non-finite inputs before the cast (cache.py:80-81)
            if not bool(torch.isfinite(k).all()) or not bool(torch.isfinite(v).all()):
                raise ValueError("non-finite key/value entry")
        code = self.lib.ckv_append(ctypes.byref(self.c), _ptr(k16), _ptr(v16), n,
                                   _stream(self.device))
        _lib.check(code, "ckv_append")
        if validate and not defer:
            st = self.status.cpu()
            if self.take_rejections(st):
                raise ValueError("non-finite key/value entry")
            if st[_lib.ST_CAPACITY]:
                raise ValueError("cache capacity exceeded")
        self._tokens += n
        self._keep = (k16, v16)  # keep inputs alive until the stream consumes them

    def _to_half(self, x):
        if x.dtype == torch.float16:
            return x.contiguous()
        if x.dtype != torch.float64:
            return x.float().to(torch.float16).contiguous()  # fp32 -> fp16: one rounding
        x = x.contiguous()
        y = torch.empty(x.shape, dtype=torch.float16, device=self.device)
        code = self.lib.ckv_f64_to_f16(_ptr(x), _ptr(y), x.numel(), _stream(self.device))
        _lib.check(code, "ckv_f64_to_f16")
        return y

    def take_rejections(self, status):
        """True if ``status`` (a host copy of the status words) shows appends
        rejected for a non-finite entry that were not reported yet; marks them
        reported, so every rejection raises exactly once."""
        n = int(status[_lib.ST_NONFINITE])
        if n > self._nonfinite_reported:
            self._nonfinite_reported = n
            return True
        return False

    def reset(self):
        """Empty every unit.  LRU scratches bound to this cache are re-initialised
        (nothing stays resident), so a refilled cache never hits stale slots."""
        _lib.check(self.lib.ckv_reset(ctypes.byref(self.c), _stream(self.device)), "ckv_reset")
        self.tier2_valid.zero_()
        self._tokens = 0
        self._nonfinite_reported = 0
        for sc in list(self._scratches):
            sc._init_device(self)

    # -- reads / parity views ------------------------------------------------
    def read_tier1(self, unit, b0=0, nb=None):
        """Unpacked Tier-1 of blocks [b0, b0+nb) of one unit as numpy arrays:
        key codes i8 [nb,16,128], key scale/offset f32 [nb,128], value codes
        u8 [nb,16,128], value scale/offset f16 [nb,16,8]."""
        if nb is None:
            nb = self.num_blocks - b0
        dev = self.device
        kc = torch.empty((max(nb, 1), B, D), dtype=torch.int8, device=dev)
        ks = torch.empty((max(nb, 1), D), dtype=torch.float32, device=dev)
        ko = torch.empty_like(ks)
        vc = torch.empty((max(nb, 1), B, D), dtype=torch.uint8, device=dev)
        vs = torch.empty((max(nb, 1), B, D // G), dtype=torch.float16, device=dev)
        vo = torch.empty_like(vs)
        code = self.lib.ckv_read_tier1(ctypes.byref(self.c), unit, b0, nb, _ptr(kc), _ptr(ks),
                                       _ptr(ko), _ptr(vc), _ptr(vs), _ptr(vo), _stream(dev))
        _lib.check(code, "ckv_read_tier1")
        return {k: t[:nb].cpu().numpy() for k, t in
                dict(kcodes=kc, kscale=ks, koffset=ko, vcodes=vc, vscale=vs, voffset=vo).items()}

    def etas(self, unit=0):
        return self.eta[unit, :self.num_blocks].double().cpu().numpy()

    def nus(self, unit=0):
        return self.nu[unit, :self.num_blocks].double().cpu().numpy()

    def v_max(self, unit=0):
        return float(self.v_max_t[unit].item())

    def corrupt_offset(self, unit, block, channel, shift):
        """Fault injection (verification.py:420-428): shift one stored key offset."""
        code = self.lib.ckv_fault_offset(ctypes.byref(self.c), unit, block, channel,
                                         ctypes.c_float(shift), _stream(self.device))
        _lib.check(code, "ckv_fault_offset")

    def drop_tier2(self, unit, block):
        """Simulate Tier-2 loss for one block (cache.py:138-142)."""
        _lib.check(self.lib.ckv_tier2_drop(ctypes.byref(self.c), unit, block,
                                           _stream(self.device)), "ckv_tier2_drop")

    def tier2_rows(self, unit):
        """Originals of all full blocks + partial, fp16 tensors on the device."""
        nfull = self.num_blocks * B
        k = self.tier2_k[unit, :nfull]
        v = self.tier2_v[unit, :nfull]
        if self.tier2_location == "host":
            k = k.to(self.device, non_blocking=True)
            v = v.to(self.device, non_blocking=True)
        idx = torch.as_tensor(K2_INDEX, device=k.device)
        k = k.reshape(-1, B * D)[:, idx].reshape(-1, D)  # fragment order -> [token][channel]
        v = v.reshape(-1, B * D)[:, torch.as_tensor(V2_INDEX, device=v.device)].reshape(-1, D)
        p = self.partial_len
        if p:
            k = torch.cat([k, self.partial_k[unit, :p]], 0)
            v = torch.cat([v, self.partial_v[unit, :p]], 0)
        return k, v

    def check_tier2(self, unit):
        nb = self.num_blocks
        if nb and not bool(self.tier2_valid[unit, :nb].all()):
            bad = int(torch.nonzero(self.tier2_valid[unit, :nb] == 0)[0].item())
            raise Tier2UnavailableError(
                f"full-precision originals for block {bad} are unavailable; "
                "cannot serve a fallback or promotion")


@dataclass
class PageInReport:
    """Accounting outcome of one promotion request (cache.py:230-240).  The
    device keeps the payloads in HBM, so ``payloads`` stays empty."""
    hits: int = 0
    misses: int = 0
    bytes: int = 0
    payloads: dict = field(default_factory=dict, repr=False)

    def to_dict(self):
        return {"hits": self.hits, "misses": self.misses, "bytes": self.bytes}


class ScratchCache:
    """LRU accounting + capacity for promoted originals of every unit, on device
    (cache.py:243-291 semantics; ckv_scratch in the C ABI).

    Bound to a DeviceKVCache (``CertifiedDecoder(..., scratch=)``) it holds the
    key LRU (``capacity``) and the value LRU (``value_capacity``) of every unit.
    Used the reference way -- one ScratchCache per payload kind passed to
    ``run_decode_step(key_scratch=, value_scratch=)`` -- it is the accounting
    view of that kind: ``hits`` / ``misses`` / ``bytes_paged_in`` / ``hit_rate``
    count the requests made through it."""

    def __init__(self, capacity, value_capacity=None):
        if capacity < 0 or (value_capacity is not None and value_capacity < 0):
            raise ValueError("capacity must be non-negative")
        self.capacity = int(capacity)
        self.value_capacity = int(capacity if value_capacity is None else value_capacity)
        self._bound = None
        self._acc = [0, 0, 0]  # hits, misses, bytes as a single-kind view (unbound)

    def _account(self, hits, misses, nbytes):
        self._acc[0] += int(hits)
        self._acc[1] += int(misses)
        self._acc[2] += int(nbytes)

    def bind(self, cache, n_heads=4, kcap=258):
        """Allocate the device LRU state (and, with Tier-2 in host RAM, the HBM
        slot pool + miss lists of the side-stream page-in) for ``cache``."""
        if self._bound is not None and self._bound() is cache:
            return
        lib = cache.lib
        U, NB = cache.n_units, cache.max_blocks
        wk = lib.ckv_lru_words(NB, self.capacity)
        wv = lib.ckv_lru_words(NB, self.value_capacity)
        dev = cache.device
        self.key_lru = torch.empty((U, wk), dtype=torch.int32, device=dev)
        self.value_lru = torch.empty((U, wv), dtype=torch.int32, device=dev)
        self.counters = torch.zeros((U, 6), dtype=torch.int64, device=dev)
        self.key_slots = self.value_slots = self.miss_list = self.miss_n = None
        miss_cap = 0
        if cache.tier2_location == "host":
            if self.capacity > 0:
                self.key_slots = torch.empty((U, min(self.capacity, NB), B * D), dtype=torch.float16,
                                             device=dev)
            if self.value_capacity > 0:
                self.value_slots = torch.empty((U, min(self.value_capacity, NB), B * D),
                                               dtype=torch.float16, device=dev)
            miss_cap = n_heads * (kcap + NB)
            self.miss_list = torch.empty((U, 2, miss_cap), dtype=torch.int32, device=dev)
            self.miss_n = torch.zeros((U, 2), dtype=torch.int32, device=dev)
        self.c = _lib.CkvScratch(key_capacity=min(self.capacity, NB), value_capacity=min(self.value_capacity, NB),
                                 key_lru=_ptr(self.key_lru), value_lru=_ptr(self.value_lru),
                                 counters=_ptr(self.counters), key_slots=_ptr(self.key_slots),
                                 value_slots=_ptr(self.value_slots), miss_list=_ptr(self.miss_list),
                                 miss_n=_ptr(self.miss_n), miss_cap=miss_cap)
        self._init_device(cache)
        self._bound = weakref.ref(cache)
        cache._scratches.add(self)

    def _init_device(self, cache):
        """Empty LRU (nothing resident) and zero counters."""
        _lib.check(cache.lib.ckv_scratch_init(cache.n_units, cache.max_blocks, ctypes.byref(self.c),
                                              _stream(cache.device)), "ckv_scratch_init")

    def totals(self):
        """(key hits, key misses, key bytes, value hits, value misses, value bytes)."""
        if self._bound is None:
            return [*self._acc, 0, 0, 0]
        return self.counters.sum(0).cpu().tolist()

    @property
    def hits(self):
        t = self.totals()
        return t[0] + t[3]

    @property
    def misses(self):
        t = self.totals()
        return t[1] + t[4]

    @property
    def bytes_paged_in(self):
        t = self.totals()
        return t[2] + t[5]

    @property
    def hit_rate(self):
        tot = self.hits + self.misses
        return self.hits / tot if tot else 0.0


class TieredCache:
    """Single KV head drop-in for the reference TieredCache (cache.py:49-224).

    Device path geometry is fixed: head_dim 128, block_size 16, group 16.
    Storage is FP16 (binary16 ingest, cache.py:82-84).
    """

    def __init__(self, block_size, head_dim, group_size=16, ingest_binary16=False,
                 max_tokens=65536, device="cuda", tier2="device"):
        if head_dim % group_size != 0:
            raise ValueError(f"group size {group_size} does not divide head dim {head_dim}")
        if (block_size, head_dim, group_size) != (B, D, G):
            raise ValueError("the device path supports block_size=16, head_dim=128, group_size=16")
        if not ingest_binary16:
            # the reference default keeps float32 originals (cache.py:52, 82-84); the
            # device keeps FP16 Tier-2 only, so refuse rather than round silently
            raise ValueError("the device path stores FP16 originals: pass ingest_binary16=True")
        self.block_size, self.head_dim, self.group_size = B, D, G
        self.ingest_binary16 = True
        self.dev = DeviceKVCache(1, max_tokens, device=device, tier2=tier2)

    def _row(self, vec, what):
        x = np.asarray(vec, dtype=np.float64).reshape(-1)
        if x.shape[0] != self.head_dim:
            raise ValueError(f"{what} has length {x.shape[0]}, expected {self.head_dim}")
        if not np.all(np.isfinite(x)):
            raise ValueError(f"non-finite {what} entry")
        return x

    def append_token(self, key, value):
        k, v = self._row(key, "key"), self._row(value, "value")
        self.dev.append(torch.from_numpy(k)[None, None], torch.from_numpy(v)[None, None])

    def append_tokens(self, keys, values):
        keys = np.atleast_2d(np.asarray(keys, dtype=np.float64))
        values = np.atleast_2d(np.asarray(values, dtype=np.float64))
        if keys.shape != values.shape:
            raise ValueError("keys and values must have matching shapes")
        if keys.shape[1] != self.head_dim:
            raise ValueError(f"key has length {keys.shape[1]}, expected {self.head_dim}")
        if not (np.all(np.isfinite(keys)) and np.all(np.isfinite(values))):
            raise ValueError("non-finite key/value entry")
        if keys.shape[0]:
            self.dev.append(torch.from_numpy(keys)[None], torch.from_numpy(values)[None])

    @property
    def num_blocks(self):
        return self.dev.num_blocks

    @property
    def partial_len(self):
        return self.dev.partial_len

    @property
    def num_tokens(self):
        return self.dev.num_tokens

    @property
    def v_max(self):
        return self.dev.v_max(0)

    def etas(self):
        return self.dev.etas(0)


# -- storage accounting (cache.py:315-388) ----------------------------------


@dataclass(frozen=True)
class StorageReport:
    head_dim: int
    block_size: int
    group_size: int
    key_codes_bytes: float
    key_metadata_bytes: float
    value_codes_bytes: float
    value_metadata_bytes: float
    annotation_bytes: float
    tier1_total_bytes: float
    tier1_exact_bytes: float
    dense_bytes: float
    tier1_ratio: float

    def to_dict(self):
        return dict(self.__dict__)


def storage_table(head_dim, block_size, group_size):
    """Per-token Tier-1 components; the device record realises exactly these
    widths (4608 B per 16-token block at d=128, g=16 -> 288 B/token)."""
    d, b, g = float(head_dim), float(block_size), float(group_size)
    parts = (d, 8.0 * d / b, d / 2.0, 4.0 * d / g)
    total = sum(parts)
    return StorageReport(int(head_dim), int(block_size), int(group_size), *parts,
                         annotation_bytes=4.0 / b, tier1_total_bytes=total,
                         tier1_exact_bytes=total + 4.0 / b, dense_bytes=4.0 * d,
                         tier1_ratio=total / (4.0 * d))


def storage_report(cache):
    return storage_table(cache.head_dim, cache.block_size, cache.group_size)
