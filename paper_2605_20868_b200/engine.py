"""Certified decode step driver (host side of the C ABI) and the reference API.

``CertifiedDecoder.step`` is the batched certified attention call: one C call
launches pass A / select / pass B / combine, the step-wide Rung 4 resolution
(harness.py:362-372), the terminal dense fallback (exact fp32 attention over
the FP16 Tier-2 originals, flagged units only) and the LRU scratch accounting
for every (unit, q-head); the host then reads back the certificate array.

``run_decode_step`` / ``run_workload`` keep the reference signatures
(harness.py:186-394) on top of it.
"""

import ctypes
import dataclasses
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .cache import DeviceKVCache, PageInReport, ScratchCache, TieredCache, _ptr, _stream
from .errors import EmptyCacheError, Tier2UnavailableError
from .policy import (KINDS, RETURNED_DENSE_ALL_HEADS, RETURNED_QUANTIZED, Certificate,
                     PolicyConfig, RungFlags, events_from_flags)

D, B = _lib.HEAD_DIM, _lib.BLOCK

CERT_DTYPE = np.dtype([("delta_h", "f8"), ("e_key_tight", "f8"), ("e_key_impl", "f8"),
                       ("e_val", "f8"), ("est_tail_mass", "f8"), ("v_max", "f8"),
                       ("canary_gap", "f8"), ("partial_mass", "f8"), ("k_star", "i4"),
                       ("k_star0", "i4"), ("k_coverage", "i4"), ("n_value_promoted", "i4"),
                       ("flags", "u4"), ("returned_kind", "i4")])
assert CERT_DTYPE.itemsize == ctypes.sizeof(_lib.CkvCert)


@dataclass
class StepOutput:
    """Result of one batched certified decode step."""
    out: torch.Tensor            # [U, nh, 128] float32 (dense rungs applied)
    explore_counts = None        # [U, nh] exploration samples (when the spot check ran)
    cert: np.ndarray             # [U, nh] CERT_DTYPE
    kinds: np.ndarray            # [U, nh] 0 quantized, 1 dense per head, 2 dense all heads
    page_stats: np.ndarray | None
    staging_bytes: int
    decoder: "CertifiedDecoder" = field(repr=False)

    def promoted(self, u, h):
        """Promoted block ids of (unit, head) in mass order (the decision)."""
        kp = int(self.cert[u, h]["k_star"])
        return self.decoder.order[u, h, :kp].cpu().numpy()

    def value_promotions(self, u, h):
        nv = int(self.cert[u, h]["n_value_promoted"])
        return self.decoder.vlist[u, h, :nv].cpu().numpy()


class PendingStep:
    """Handle of a step enqueued by ``CertifiedDecoder.step_async``."""

    def __init__(self, dec, cert_h, stat_h, ps_h, event, n_tokens, en_h=None, out=None):
        self._args = (cert_h, stat_h, ps_h, n_tokens, en_h, out)
        self._dec, self._ev, self._res, self._exc = dec, event, None, None

    def done(self):
        return self._ev.query()

    def _decode(self):
        """Decode the pinned copies once; an error (Tier-2 loss, a rejected
        deferred append) is kept and raised by ``result()`` of this step."""
        if self._res is None and self._exc is None:
            self._ev.synchronize()
            try:
                self._res = self._dec._output(*self._args)
            except (ValueError, Tier2UnavailableError) as e:
                self._exc = e

    def result(self):
        """Wait for this step's certificates (not for later steps) and decode them."""
        self._decode()
        if self._exc is not None:
            raise self._exc
        return self._res


class CertifiedDecoder:
    """Certified decode over every unit of a DeviceKVCache.

    ``rung4_group`` is the number of consecutive units that share a step-wide
    Rung 4 (a canary trip in any of them makes all their heads dense); the
    reference's single-layer run makes it every unit (harness.py:362-372).

    ``plan_units`` / ``dense_splits``: by default the launch shapes adapt to this
    decoder's unit count and to how many units turn dense in a step.  A shard of
    a KV-head-sharded job that passes the whole job's unit count and a fixed
    dense split count computes, for its units, bit for bit what one decoder over
    every unit computes (the decomposition of every reduction is the same).
    """

    def __init__(self, cache: DeviceKVCache, policy: PolicyConfig, n_heads=4, scratch=None,
                 rung4_group=None, plan_units=None, dense_splits=0):
        if not 1 <= n_heads <= _lib.MAX_QHEADS:
            raise ValueError("device path supports 1..4 query heads per KV head")
        self.cache, self.policy, self.nh = cache, policy, int(n_heads)
        self.lib = cache.lib
        self.pol_c = policy.to_c()
        st = _lib.CkvStep()
        _lib.check(self.lib.ckv_plan(int(plan_units or cache.n_units), cache.max_blocks, self.nh,
                                     ctypes.byref(self.pol_c), ctypes.byref(st)), "ckv_plan")
        st.plan_units = int(plan_units or 0)
        st.dense_splits = int(dense_splits)
        U, NB, nh, dev = cache.n_units, cache.max_blocks, self.nh, cache.device
        self.q = torch.zeros((U, nh, D), dtype=torch.float64, device=dev)
        self.out = self._out0 = torch.zeros((U, nh, D), dtype=torch.float32, device=dev)
        self.cert_buf = torch.zeros((U, nh, CERT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        self.lm1 = torch.zeros((U, nh, NB), dtype=torch.float32, device=dev)
        self.split_state = torch.zeros((U, st.n_splits, 4, _lib.SPLIT_FLOATS),
                                       dtype=torch.float32, device=dev)
        self.order = torch.zeros((U, nh, st.kcap), dtype=torch.int32, device=dev)
        self.work = torch.zeros((U, st.wcap), dtype=torch.int32, device=dev)
        self.n_work = torch.zeros((U,), dtype=torch.int32, device=dev)
        self.vlist = torch.zeros((U, nh, NB), dtype=torch.int32, device=dev)
        self.lm2 = torch.zeros((U, nh, NB), dtype=torch.float32, device=dev)
        self.head_state = torch.zeros((U, nh, _lib.HEAD_FLOATS), dtype=torch.float32, device=dev)
        self.chunk_state = torch.zeros((U, st.n_chunks, 4, _lib.CHUNK_FLOATS),
                                       dtype=torch.float32, device=dev)
        self.page_stats = torch.zeros((U, 4), dtype=torch.int32, device=dev)
        self.dense_list = torch.zeros((2 * U + 1,), dtype=torch.int32, device=dev)
        self.unit_done = torch.zeros((U,), dtype=torch.int32, device=dev)
        # st.queue (persistent pass B) stays NULL: measured 443 us vs 416 us for one
        # CTA per (chunk, unit) at C3 -- the per-chunk ring drain is not overlapped
        st.ecap = max(1, int(round(0.05 * NB)) + 1)
        self.explore_n = torch.zeros((U, nh), dtype=torch.int32, device=dev)
        self.explore_pos = torch.zeros((U, nh, st.ecap), dtype=torch.int32, device=dev)
        self.rng_words = torch.zeros((16,), dtype=torch.int64, device=dev)
        self.rng_host = torch.zeros((16,), dtype=torch.int64).pin_memory()
        self.explore_work = torch.zeros((4 * U * nh + 64,), dtype=torch.int32, device=dev)
        self._attached = None
        st.explore_rate = float(policy.exploration_rate)
        st.explore_work = _ptr(self.explore_work)
        self.dense_part = torch.zeros((U, st.n_dsplit_cap, 4, 132), dtype=torch.float32, device=dev)
        for name, t in (("q", self.q), ("out", self.out), ("cert", self.cert_buf),
                        ("lm1", self.lm1), ("split_state", self.split_state),
                        ("order", self.order), ("work", self.work), ("n_work", self.n_work),
                        ("vlist", self.vlist), ("lm2", self.lm2),
                        ("head_state", self.head_state), ("chunk_state", self.chunk_state),
                        ("page_stats", self.page_stats), ("dense_list", self.dense_list),
                        ("dense_part", self.dense_part), ("explore_pos", self.explore_pos),
                        ("unit_done", self.unit_done)):
            setattr(st, name, _ptr(t))
        if os.environ.get("CKV_SEPARATE_UNION"):  # A/B knob: union list by its own launch
            st.unit_done = None
        # per-unit completion epochs: pass A -> selection -> pass B -> combine run as
        # programmatic dependent launches that overlap on finished units
        self.flow = torch.zeros((6 * U + 4,), dtype=torch.int32, device=dev)
        if not os.environ.get("CKV_NO_FLOW"):
            st.flow = _ptr(self.flow)
        # phase-1 score stash: pass A keeps the quantized scores of blocks likely to be
        # promoted (predicted from the previous step's tail threshold) so pass B needs
        # only the value part of their Tier-1 record (exact either way)
        if not os.environ.get("CKV_NO_STASH"):
            self.stash = torch.empty((U, NB, 4 * 16), dtype=torch.float32, device=dev)
            self.stash_epoch = torch.full((U, NB), -1, dtype=torch.int32, device=dev)
            st.stash = _ptr(self.stash)
            st.stash_epoch = _ptr(self.stash_epoch)
            st.stash_margin = float(os.environ.get("CKV_STASH_MARGIN", "0.1"))
        st.epoch = 0
        # step-wide Rung 4 (harness.py:362-372) acts on groups of units: one
        # group = the reference's single step (None), contiguous runs of
        # ``rung4_group`` units (int), or explicit group ids per unit (array,
        # e.g. the (layer, sequence) of every unit -- shared across ranks)
        if rung4_group is None or np.isscalar(rung4_group):
            g = int(rung4_group or U)
            groups = np.arange(U) // g
        else:
            groups = np.asarray(rung4_group, dtype=np.int64).reshape(-1)
            if groups.shape[0] != U or groups.min() < 0:
                raise ValueError("rung4_group must give a non-negative group id per unit")
        self.unit_group_host = groups
        self.n_groups = int(groups.max()) + 1
        self.unit_group = torch.as_tensor(groups, dtype=torch.int32).to(dev)
        self.group_flags = torch.zeros((self.n_groups,), dtype=torch.int32, device=dev)
        st.rung4_group = 1
        st.unit_group = _ptr(self.unit_group)
        st.group_flags = _ptr(self.group_flags)
        st.n_groups = self.n_groups
        self.st = st
        self.scratch = scratch
        if scratch is not None:
            scratch.bind(cache, n_heads=self.nh, kcap=st.kcap)
        # the step's bound report is written by its last kernel straight into pinned
        # host memory (ckv_step.host_report): no device-to-host copies in the stream
        self._report = self._report_buffer()
        self.cert_host, self.status_host, self.ps_host, self.explore_n_host = self._report[1]

    def _report_buffer(self):
        """A pinned host_report buffer and its views (cert, status, page_stats,
        explore_n) in the library's layout (ckv_report_layout)."""
        U, nh = self.cache.n_units, self.nh
        lay = (ctypes.c_int64 * 4)()
        self.lib.ckv_report_layout(U, nh, lay)
        buf = torch.zeros((int(lay[0]),), dtype=torch.uint8).pin_memory()
        cert = buf[:U * nh * CERT_DTYPE.itemsize].view(U, nh, CERT_DTYPE.itemsize)
        status = buf[lay[1]:lay[1] + 32].view(torch.int32)
        ps = buf[lay[2]:lay[2] + U * 16].view(torch.int32).view(U, 4)
        en = buf[lay[3]:lay[3] + U * nh * 4].view(torch.int32).view(U, nh)
        return buf, (cert, status, ps, en)

    # -- the device step -----------------------------------------------------
    def launch(self, queries=None, reduce_flags=None, explore=False, report=None, out=None):
        """Enqueue the whole step (no host sync); returns immediately.

        ``reduce_flags(group_flags)`` -- e.g. an all-reduce(MAX) across the
        ranks of a KV-head sharded job -- runs between the Rung-4 requests and
        their resolution, in stream order (ckv_decode_flags / _finish).
        ``report``: a pinned buffer from ``_report_buffer`` the step's last kernel
        writes the bound report into (None: the report stays on the device).
        ``out``: the device tensor the outputs go to (None: ``self._out0``);
        ``self.out`` names the latest step's."""
        if out is None:
            out = self._out0
        elif (out.device != self._out0.device or out.dtype != torch.float32
              or out.shape != self._out0.shape or not out.is_contiguous()):
            raise ValueError("out must be a contiguous float32 device tensor of shape "
                             f"{tuple(self._out0.shape)}")
        self.out = out
        self.st.out = out.data_ptr()
        if queries is not None:
            qt = queries if isinstance(queries, torch.Tensor) else torch.as_tensor(queries)
            if (qt.device == self.q.device and qt.dtype == torch.float64 and qt.is_contiguous()
                    and qt.numel() == self.q.numel()):
                # a device float64 query tensor is read in place (no copy kernel in the
                # step's stream); record_stream keeps the allocator from reusing it
                # before the step has read it, whichever stream allocated it
                self.st.q = qt.data_ptr()
                qt.record_stream(torch.cuda.current_stream(self.cache.device))
            else:
                self.q.copy_(qt.reshape(self.q.shape), non_blocking=True)
                self.st.q = self.q.data_ptr()
        else:  # the caller filled self.q
            self.st.q = self.q.data_ptr()
        sc = ctypes.byref(self.scratch.c) if self.scratch is not None else None
        args = (ctypes.byref(self.cache.c), ctypes.byref(self.pol_c), ctypes.byref(self.st))
        nbk, stream = self.cache.num_blocks, _stream(self.cache.device)
        self.st.epoch = (self.st.epoch + 1) & 0x3ffffff
        # exploration: samples drawn on the device from the generator state in rng_words
        self.st.explore_rng = _ptr(self.rng_words) if explore else None
        self.st.explore_n = _ptr(self.explore_n) if explore else None
        self.st.host_report = report.data_ptr() if report is not None else None
        if reduce_flags is None:
            _lib.check(self.lib.ckv_decode_step(*args, sc, nbk, stream), "ckv_decode_step")
            return
        _lib.check(self.lib.ckv_decode_begin(*args, sc, nbk, stream), "ckv_decode_begin")
        _lib.check(self.lib.ckv_decode_flags(*args, nbk, stream), "ckv_decode_flags")
        reduce_flags(self.group_flags)
        _lib.check(self.lib.ckv_decode_finish(ctypes.byref(self.cache.c), ctypes.byref(self.st),
                                              sc, nbk, stream), "ckv_decode_finish")

    def step(self, queries, rng=None):
        """Certified attention for all units: queries [U, nh, 128] (float64).

        The fast path, the step-wide Rung 4 resolution and the dense fallback
        all run on the device; the host reads back the certificate array once
        (and raises on a Tier-2 loss).  With ``policy.exploration_rate > 0``
        and the workload's numpy Philox Generator ``rng`` the exploration spot
        check runs too: the device draws the sampled tail positions from the
        generator's state exactly as fallback.py:212-218 does (heads in
        unit-major q-head order; csrc/explore_draw.cu), rescores those blocks,
        and ``rng`` is advanced as the reference's draws would advance it.
        """
        if self.cache.num_tokens == 0:
            raise EmptyCacheError("cannot attend over an empty cache")
        explore = self.policy.exploration_rate > 0 and rng is not None
        if explore and self._attached is None:
            self._rng_upload(rng)
        self.launch(queries, explore=explore or self._attached is not None, report=self._report[0])
        out = self._finish(explore or self._attached is not None)
        if explore and self._attached is None:
            self._rng_download(rng)
        return out

    # -- exploration generator on the device ------------------------------------
    def _rng_upload(self, rng):
        if not isinstance(getattr(rng, "bit_generator", None), np.random.Philox):
            raise ValueError("the exploration generator must be a numpy Generator over Philox "
                             "(the reference's philox4x64 stream, harness.py:93-95)")
        self.rng_host.numpy()[:] = pack_philox_state(rng.bit_generator.state).view(np.int64)
        self.rng_words.copy_(self.rng_host, non_blocking=True)

    def _rng_download(self, rng):
        self.rng_host.copy_(self.rng_words)  # synchronous
        st = rng.bit_generator.state
        rng.bit_generator.state = unpack_philox_state(self.rng_host.numpy().view(np.uint64), st)

    def attach_rng(self, rng):
        """Keep the exploration generator on the device across steps (step_async
        with exploration): the state is uploaded once and advanced by every
        step; ``detach_rng`` writes it back into ``rng``."""
        if self.policy.exploration_rate <= 0:
            raise ValueError("the policy's exploration_rate is 0")
        self._rng_upload(rng)
        self._attached = rng

    def detach_rng(self):
        rng, self._attached = self._attached, None
        if rng is not None:
            torch.cuda.current_stream(self.cache.device).synchronize()
            self._rng_download(rng)
        return rng

    def step_async(self, queries, reduce_flags=None, out=None):
        """Enqueue a certified step and return a ``PendingStep`` without a host
        sync: the step's last kernel writes its bound report into one of two
        pinned buffers, so the host can read step i's report while the device
        runs step i+1.  The output stays on the device, dense rungs already
        applied: in ``out`` (a float32 device tensor [U, n_heads, 128] of the
        caller, e.g. one of two buffers that leave for the host while the next
        step runs) or in the decoder's own ``self.out``, valid in stream order
        until the next step overwrites it.  Exploration runs when a generator
        is attached (``attach_rng``)."""
        if self.cache.num_tokens == 0:
            raise EmptyCacheError("cannot attend over an empty cache")
        explore = self._attached is not None
        k = self._ring_i = (getattr(self, "_ring_i", 1) + 1) % 2
        if not hasattr(self, "_ring"):
            self._ring = [self._report_buffer() + (torch.cuda.Event(),) for _ in range(2)]
            self._ring_pending = [None, None]
        prev = self._ring_pending[k]
        if prev is not None:
            prev._decode()  # the step that last used this report buffer, before it is rewritten
        buf, (cert_h, stat_h, ps_h, en_h), ev = self._ring[k]
        self.launch(queries, reduce_flags, explore=explore, report=buf, out=out)
        ev.record(torch.cuda.current_stream(self.cache.device))
        pend = PendingStep(self, cert_h, stat_h, ps_h, ev, self.cache.num_tokens,
                           en_h if explore else None, self.out)
        self._ring_pending[k] = pend
        return pend

    def _finish(self, explore=False):
        # the step's last kernel wrote the report into self._report (host_report)
        torch.cuda.current_stream(self.cache.device).synchronize()  # the step's only host sync
        return self._output(self.cert_host, self.status_host, self.ps_host, self.cache.num_tokens,
                            self.explore_n_host if explore else None)

    def _output(self, cert_h, stat_h, ps_h, n_tokens, en_h=None, out_t=None):
        if self.cache.take_rejections(stat_h):  # a deferred append check (DeviceKVCache.append)
            self.cache.resync()
            raise ValueError("non-finite key/value entry (append rejected on the device)")
        if stat_h[_lib.ST_TIER2]:  # per-step word: this step needed a lost block
            raise Tier2UnavailableError("full-precision originals of a promoted block are unavailable")
        cert = cert_h.numpy().view(CERT_DTYPE).reshape(self.cache.n_units, self.nh).copy()
        kinds = cert["returned_kind"].copy()
        # Rung-4 staging bytes (fallback.py:235-238): every unit of a flagged group
        flagged = np.unique(self.unit_group_host[(kinds == 2).any(axis=1)])
        n_units = int(np.isin(self.unit_group_host, flagged).sum()) if flagged.size else 0
        staging = n_units * 2 * n_tokens * D * 2
        ps = ps_h.numpy().copy() if self.scratch is not None else None
        out = StepOutput(self.out if out_t is None else out_t, cert, kinds, ps, staging, self)
        if en_h is not None:
            out.explore_counts = en_h.numpy().copy()
        return out


def pack_philox_state(state):
    """numpy Philox bit_generator.state -> the 16 uint64 words of
    ckv_step.explore_rng (counter, key, buffer, buffer_pos, has_uint32, uinteger)."""
    w = np.zeros(16, dtype=np.uint64)
    w[0:4] = np.asarray(state["state"]["counter"], dtype=np.uint64)
    w[4:6] = np.asarray(state["state"]["key"], dtype=np.uint64)
    w[6:10] = np.asarray(state["buffer"], dtype=np.uint64)
    w[10] = int(state["buffer_pos"])
    w[11] = int(state["has_uint32"])
    w[12] = int(state["uinteger"])
    return w


def unpack_philox_state(words, template):
    """Inverse of pack_philox_state, into a copy of ``template``."""
    st = dict(template)
    st["state"] = {"counter": np.asarray(words[0:4], dtype=np.uint64).copy(),
                   "key": np.asarray(words[4:6], dtype=np.uint64).copy()}
    st["buffer"] = np.asarray(words[6:10], dtype=np.uint64).copy()
    st["buffer_pos"] = int(words[10])
    st["has_uint32"] = int(words[11])
    st["uinteger"] = int(words[12])
    return st


# -- reference-shaped per-head API --------------------------------------------


@dataclass
class SelectionView:
    promoted: frozenset
    k_star: int
    est_tail_mass: float
    clamped: bool
    k_coverage: int
    partial_mass: float
    order: np.ndarray


@dataclass
class HeadStepResult:
    """Same fields as harness.HeadStepResult (harness.py:166-178)."""
    output: np.ndarray
    certificate: Certificate
    events: list
    page_reports: dict
    decision: SelectionView
    value_promotions: frozenset
    attend: object
    delta_h: float
    rung4_requested: bool = False


def certificate_from_row(row, head, step, kind=None):
    fl = int(row["flags"])
    kind = int(row["returned_kind"]) if kind is None else int(kind)
    return Certificate(
        head=int(head), step=int(step), delta_h=float(row["delta_h"]),
        e_key_tight=float(row["e_key_tight"]), e_key_impl=float(row["e_key_impl"]),
        e_val=float(row["e_val"]), est_tail_mass=float(row["est_tail_mass"]),
        v_max=float(row["v_max"]), k_star=int(row["k_star"]), returned_kind=KINDS[kind],
        rung_flags=RungFlags(rung1=bool(fl & _lib.F_RUNG1), rung2=bool(fl & _lib.F_RUNG2),
                             rung3=bool(fl & (_lib.F_RANKING | _lib.F_BOUNDARY)),
                             rung4=bool(fl & (_lib.F_CANARY | _lib.F_NUMERIC | _lib.F_EXPLORE))))


def run_decode_step(query, cache, policy, key_scratch=None, value_scratch=None, rng=None,
                    head=0, step=0):
    """One q-head through the certified pipeline (harness.py:186-300)."""
    if not isinstance(cache, TieredCache):
        raise TypeError("run_decode_step expects a paper_2605_20868_b200.TieredCache")
    q = np.asarray(query, dtype=np.float64).reshape(-1)
    if q.shape[0] != cache.head_dim:
        raise ValueError(f"query has length {q.shape[0]}, expected {cache.head_dim}")
    scratch = None
    if key_scratch is not None or value_scratch is not None:
        # one device LRU state per (key scratch, value scratch) pair, held by the
        # cache (with the pair, so the ids stay unique while it lives); the
        # caller's objects receive the per-kind accounting of every request
        kc = key_scratch.capacity if key_scratch is not None else 1 << 30
        vc = value_scratch.capacity if value_scratch is not None else 1 << 30
        reg = cache.__dict__.setdefault("_scratch_pairs", {})
        key = (id(key_scratch), id(value_scratch))
        if key not in reg:
            reg[key] = (key_scratch, value_scratch, ScratchCache(kc, vc))
        scratch = reg[key][2]
    dkey = ("dec", policy, id(scratch))
    dec = cache.__dict__.get(dkey)
    if dec is None:
        dec = CertifiedDecoder(cache.dev, policy, n_heads=1, scratch=scratch)
        cache.__dict__[dkey] = dec
    res = dec.step(torch.from_numpy(q).reshape(1, 1, D).to(cache.dev.device), rng=rng)
    row = res.cert[0, 0]
    kind = int(res.kinds[0, 0])
    cert = certificate_from_row(row, head, step, kind)
    reports = {}
    if scratch is not None:
        ps = res.page_stats[0]  # this step's (key hits, key misses, value hits, value misses)
        nbytes = B * D * 2
        if key_scratch is not None:
            reports["keys"] = PageInReport(int(ps[0]), int(ps[1]), int(ps[1]) * nbytes)
            key_scratch._account(ps[0], ps[1], int(ps[1]) * nbytes)
        if value_scratch is not None:
            reports["values"] = PageInReport(int(ps[2]), int(ps[3]), int(ps[3]) * nbytes)
            value_scratch._account(ps[2], ps[3], int(ps[3]) * nbytes)
    if res.explore_counts is not None:
        n = int(res.explore_counts[0, 0])
        reports["exploration"] = PageInReport(0, n, n * B * D * 2)
    prom = res.promoted(0, 0)
    vprom = frozenset(int(b) for b in res.value_promotions(0, 0))
    decision = SelectionView(frozenset(int(b) for b in prom), int(row["k_star"]),
                             float(row["est_tail_mass"]),
                             bool(int(row["flags"]) & _lib.F_CLAMPED), int(row["k_coverage"]),
                             float(row["partial_mass"]), prom)
    out = res.out[0, 0].double().cpu().numpy()
    return HeadStepResult(out, cert, events_from_flags(int(row["flags"]), head, step), reports,
                          decision, vprom, None, float(row["delta_h"]),
                          rung4_requested=bool(int(row["flags"]) & (_lib.F_CANARY | _lib.F_NUMERIC
                                                                    | _lib.F_EXPLORE)))


def dense_attention(query, cache):
    """Exact attention over the originals of a TieredCache (attention.py:327-342)."""
    dev = cache.dev
    if dev.num_tokens == 0:
        raise EmptyCacheError("cannot attend over an empty cache")
    dev.check_tier2(0)
    k, v = dev.tier2_rows(0)
    q = torch.as_tensor(np.asarray(query, dtype=np.float64)).to(dev.device)
    s = (k.double() @ q) / np.sqrt(D)
    w = torch.softmax(s, 0)
    return (w @ v.double()).cpu().numpy()


# -- the dense rungs as standalone calls (fallback.py:230-255) ----------------


def rung3_per_head(query, cache):
    """Dense recomputation of one head: the exact routine (dense_attention)."""
    return dense_attention(query, cache)


def rung4_staging_bytes(token_counts, head_dim):
    """FP16 K and V staged for an all-head dense recomputation: 2 * N * d * 2
    bytes per distinct cache (fallback.py:235-238)."""
    return int(sum(2 * int(n) * int(head_dim) * 2 for n in token_counts))


def rung4_all_heads(queries, caches):
    """Dense outputs for every query head (one cache per head, grouped heads
    repeat their cache) and the staging bytes, charged once per distinct cache."""
    if len(queries) != len(caches):
        raise ValueError("need one cache reference per query head")
    outs = [dense_attention(q, c) for q, c in zip(queries, caches)]
    distinct = list({id(c): c for c in caches}.values())
    return outs, rung4_staging_bytes([c.num_tokens for c in distinct], distinct[0].head_dim)
