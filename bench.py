"""Certified decode-attention steps/s at Llama-3.1-8B attention shape, 128K context.

One step = one full decode step of the model's attention: every (layer, KV
head) unit (32 layers x 8 KV heads, 4 q-heads each) runs the certified path
(Phase-1 INT8 scoring, selection + Rung 1/2, page-in accounting, Phase-2
mask-gated attend, E_key/E_val certificates, ranking/boundary/canary, dense
fallback for flagged heads) and then appends one new token per unit
(quantize-on-append).  KV heads are sharded across ranks (N GPUs); per step the
ranks all-gather outputs + certificates over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0).  `--impl reference` times the reference's own
CPU implementation on the host cores instead: the unmodified certkv package
with its compiled kernel backend, built into oracle/_ref by oracle/build_ref.sh
(the oracle/ NumPy port only if that build is missing).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Certified decode-attention steps/s (Llama-3.1-8B, 128K ctx); % HBM peak"
UNIT = "steps/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


# BASELINE.json configs C2-C5 (C1 is the reference's CPU case: the parity tests
# and the cpu_baseline leg).  The default bench line is C3, the headline.
PRESETS = {
    "c2": dict(ctx=32768, batch=1, tier2="device", scratch=-1, v_tol=None, adversarial=False,
               desc="C2: Llama-3.1-8B attention, 32 layers x GQA 32/8, d=128, 32768 ctx, batch 1"),
    "c3": dict(ctx=131072, batch=1, tier2="device", scratch=-1, v_tol=None, adversarial=False,
               desc="C3: Llama-3.1-8B attention, 32 layers x GQA 32/8, d=128, 131072 ctx, batch 1, "
                    "KV-head sharded"),
    # the north-star placement of C3: Tier-2 originals in pinned host RAM, the
    # reference's default 2048-block scratch per KV head (harness.py:339), misses
    # paged in over PCIe
    "c3host": dict(ctx=131072, batch=1, tier2="host", scratch=2048, v_tol=None, adversarial=False,
                   desc="C3 with Tier-2 in pinned host RAM: Llama-3.1-8B attention, 32 layers x "
                        "GQA 32/8, d=128, 131072 ctx, batch 1, 2048-block LRU scratch per KV head "
                        "in HBM, misses paged in over PCIe"),
    "c4": dict(ctx=16384, batch=32, tier2="host", scratch=-1, v_tol=1e-3, adversarial=False,
               desc="C4: Llama-3.1-8B attention, 32 layers x GQA 32/8, d=128, 16384 ctx, batch 32, "
                    "tight v_tol (value promotions), Tier-2 in pinned host RAM (page-in)"),
    "c5": dict(ctx=65536, batch=1, tier2="device", scratch=-1, v_tol=None, adversarial=True,
               desc="C5: 65536 ctx, outlier key channels (x1000 on 2 channels), near-tie twin "
                    "blocks, corrupted key offsets in layer 0 (canary -> Rung 4 -> dense)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(PRESETS))
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--q-per-kv", type=int, default=4)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--tier2", default=None, choices=["device", "host"])
    ap.add_argument("--scratch", type=int, default=None,
                    help="LRU scratch capacity in blocks (-1: every block, 0: off)")
    ap.add_argument("--v-tol", type=float, default=None)
    ap.add_argument("--explore", type=float, default=0.0,
                    help="exploration_rate of the policy (0 or 0.01..0.05; the reference default "
                         "is 0.02, the paper's benchmarks run with 0)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="shards plan their launches for the whole job (bit-identical to N=1)")
    ap.add_argument("--no-variant", action="store_true",
                    help="skip the c3host variant measured after the default c3 line")
    args = ap.parse_args()
    pre = PRESETS[args.config]
    for k in ("ctx", "batch", "tier2", "scratch", "v_tol"):
        if getattr(args, k) is None:
            setattr(args, k, pre[k])
    args.adversarial = pre["adversarial"]
    args.desc = pre["desc"]
    return args


def peak_hbm():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML thread
    polls every ~4 ms between start() and stop() (the timed region is ~20 ms at the
    default K, too short for nvidia-smi's 200-ms loop); nvidia-smi when NVML is absent."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index, dev=None):
        self.index, self.rows, self.proc, self.nv, self.h = index, [], None, None, None
        try:
            if os.environ.get("CKV_BENCH_CLOCKS") == "smi":
                raise ImportError
            import pynvml
            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(dev).uuid)
                self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                         pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap)
        except Exception:
            self.nv = None

    def start(self):
        if self.nv is not None:
            self.stop_flag = False
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _poll(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.rows.append([sm, self.smax] + [bool(r & b) for b in self.bits])
            except Exception:
                pass
            time.sleep(0.004)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                self.rows.append([float(parts[0]), float(parts[1])] + [p == "Active" for p in parts[3:]])

    def stop(self):
        if self.nv is not None:
            self.stop_flag = True
            self.t.join(timeout=2)
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        rows = list(self.rows)
        sm = sorted(r[0] for r in rows)
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[2 + i]})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": rows[0][1] if rows else None,
                "reasons": reasons, "samples": len(rows),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


# -------------------------------------------------------------------------
# CPU arm: the unmodified reference (oracle/_ref, built by oracle/build_ref.sh)
# or, if that build is absent, the oracle port
# -------------------------------------------------------------------------

_W = {}


def _worker_init(ctx, seed, n_heads):
    import numpy as np
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    import oracle
    rng = np.random.default_rng(seed)
    kv = oracle.OracleKV(16, 128, 16, ingest_binary16=True, narrow=False)
    kv.append_tokens(rng.standard_normal((ctx, 128)), rng.standard_normal((ctx, 128)))
    _W.update(kv=kv, rng=rng, n_heads=n_heads)


def _worker_step(_):
    """One unit-step of the oracle port: n_heads certified q-heads, then
    quantize-on-append of the new token (harness.py:351-382)."""
    import oracle
    from oracle.step import OraclePolicy
    kv, rng = _W["kv"], _W["rng"]
    pol = OraclePolicy(exploration_rate=0.0)
    t0 = time.perf_counter()
    for _h in range(_W["n_heads"]):
        oracle.decode_step(rng.standard_normal(128), kv, pol)
    kv.append_token(rng.standard_normal(128), rng.standard_normal(128))
    return time.perf_counter() - t0


def _port_reference(args, total_units, steps, warmup, workers):
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_worker_init,
                  initargs=(args.ctx, 1234, args.q_per_kv)) as pool:
        pool.map(_worker_step, range(workers))
        for _ in range(warmup):
            pool.map(_worker_step, range(workers))
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_worker_step, range(workers))
        dt = (time.perf_counter() - t0) / steps
    return dt * total_units / workers


def cpu_reference(args, total_units, steps, warmup, workers):
    """Seconds per full decode step on `workers` host processes (one unit each,
    single-threaded), scaled from `workers` unit-steps to `total_units`.
    Returns (steps/s, kind, detail)."""
    from oracle import ref_arm
    if ref_arm.available():
        r = ref_arm.time_reference(args.ctx, args.q_per_kv, total_units, steps, warmup, workers,
                                   v_tol=args.v_tol, adversarial=args.adversarial,
                                   explore=args.explore)
        return 1.0 / r["sec_per_step"], "reference", {
            "impl": "unmodified certkv (oracle/_ref) harness.run_workload, kernel backend "
                    f"'{r['backend']}'", "unit_step_s": r["round_s"], "prefill_s": r["prefill_s"],
            "host": ref_arm.host_info()}
    sec = _port_reference(args, total_units, steps, warmup, workers)
    return 1.0 / sec, "port", {"impl": "oracle/ NumPy port (oracle/_ref not built)",
                               "host": ref_arm.host_info()}


# -------------------------------------------------------------------------
# our arm
# -------------------------------------------------------------------------

def run_gpu(args, ck, dev, world, rank, local, K, W, dist, total_units, e2e_wanted=True,
            clocks_wanted=True):
    """Build the cache of this rank's units, warm up, time K certified steps (CUDA
    events, max over ranks), then the end-to-end loop through the public API.
    Returns the measurements and the live objects (cache, decoder, scratch)."""
    import numpy as np
    import torch
    from paper_2605_20868_b200 import _lib
    # KV-head sharding: units are kv-major (sharding.unit_index); rank r owns whole KV heads
    if args.kv_heads % world:
        raise SystemExit("kv_heads must be divisible by the number of GPUs")
    U = total_units // world
    max_tokens = args.ctx + 3 * K + 2 * W + max(K, 40) + 64  # timed + pass-A + e2e appends
    cache = ck.DeviceKVCache(U, max_tokens, device=dev, tier2=args.tier2)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    chunk = max(16, min(4096, (1 << 22) // U))
    t0 = time.perf_counter()
    for pos in range(0, args.ctx, chunk):
        n = min(chunk, args.ctx - pos)
        kk = torch.randn((U, n, 128), generator=g, device=dev)
        vv = torch.randn((U, n, 128), generator=g, device=dev).half()
        if args.adversarial:
            kk[:, :, 3] *= 1000.0    # outlier key channels
            kk[:, :, 77] *= 1000.0
            if pos == 0 and n >= 32:  # near-tie twin blocks 0 and 1
                kk[:, 16:32] = kk[:, 0:16] + 1e-4 * torch.randn_like(kk[:, 0:16])
        cache.append(kk.half(), vv, validate=False)
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    if args.adversarial and rank == 0:
        # corrupt stored key offsets of 8 blocks of unit 0 (layer 0), random channel and
        # sign, so some promoted block's scores move by far more than Delta every step
        # (verification.py:420-428): the canary trips and layer 0 returns dense
        rs = np.random.default_rng(5)
        for b in rs.choice(cache.num_blocks, size=8, replace=False):
            cache.corrupt_offset(0, int(b), int(rs.integers(0, 128)),
                                 float(rs.choice([-1.0, 1.0]) * 5.0e4))

    pkw = {"exploration_rate": args.explore}
    if args.v_tol is not None:
        pkw["v_tol"] = args.v_tol
    pol = ck.PolicyConfig(**pkw)
    cap = cache.max_blocks if args.scratch < 0 else args.scratch
    scratch = ck.ScratchCache(cap) if args.scratch != 0 else None
    from paper_2605_20868_b200 import sharding
    my_units = sharding.shard_units(args.layers, args.kv_heads, args.batch, world, rank)
    # step-wide Rung 4 per (layer, sequence), shared by the ranks holding that layer's KV heads
    groups = np.asarray(list(my_units)) % (args.layers * args.batch)
    det = dict(plan_units=total_units, dense_splits=64) if args.deterministic else {}
    dec = ck.CertifiedDecoder(cache, pol, n_heads=args.q_per_kv, scratch=scratch,
                              rung4_group=groups, **det)
    assert dec.n_groups == args.layers * args.batch
    if args.explore > 0:  # the spot check's generator, drawn from on the device every step
        dec.attach_rng(np.random.Generator(np.random.Philox(np.random.SeedSequence((rank, 1)))))
    nq = W + K
    qpool = torch.randn((nq, U, args.q_per_kv, 128), generator=g, device=dev, dtype=torch.float64)
    kpool = torch.randn((nq, U, 1, 128), generator=g, device=dev).half()
    vpool = torch.randn((nq, U, 1, 128), generator=g, device=dev).half()
    ev_a = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(K)]
    for a, b in ev_a:  # torch creates the CUDA event lazily: force it before handing it over
        a.record()
        b.record()

    reduce_flags = None
    if world > 1:
        def reduce_flags(flags):  # per-layer Rung-4 request, MAX over ranks (NCCL, no host sync)
            sharding.reduce_group_flags(flags)

    def exchange():
        if world > 1:  # the bound report: outputs + certificates of every rank, one all-gather
            sharding.gather_bound_report(dec.out, dec.cert_buf)

    launches = {"n": 0}
    dense_heads = {"n": 0}
    stats = {"rung4": 0, "nv": 0.0, "pagein": 0, "steps": 0, "hits": 0, "misses": 0}
    last = {}
    pending = {"p": None}

    def collect():
        p = pending["p"]
        if p is not None:
            res = p.result()
            dense_heads["n"] += int((res.kinds != 0).sum())
            stats["rung4"] += int((res.kinds == 2).sum())
            stats["nv"] += float(res.cert["n_value_promoted"].mean())
            if res.page_stats is not None:
                stats["pagein"] += int(res.page_stats[:, 1].sum() + res.page_stats[:, 3].sum()) * 4096
                stats["hits"] += int(res.page_stats[:, 0].sum() + res.page_stats[:, 2].sum())
                stats["misses"] += int(res.page_stats[:, 1].sum() + res.page_stats[:, 3].sum())
            stats["steps"] += 1
            last["res"] = res
            pending["p"] = None

    def one_step(i, timed_ev=None):
        # the host decodes step i-1's certificates while the device runs step i
        if timed_ev is not None:
            dec.st.prof_begin = timed_ev[0].cuda_event
            dec.st.prof_end = timed_ev[1].cuda_event
        p = dec.step_async(qpool[i], reduce_flags)
        dec.st.prof_begin = None
        dec.st.prof_end = None
        launches["n"] += lib.ckv_last_launches()
        exchange()
        cache.append(kpool[i], vpool[i], validate=False)
        launches["n"] += lib.ckv_last_launches()
        collect()
        pending["p"] = p

    lib = cache.lib
    for i in range(W):
        one_step(i)
    torch.cuda.synchronize()
    collect()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local, dev) if (rank == 0 and clocks_wanted) else None
    if sampler:
        sampler.start()
        if sampler.nv is None:
            time.sleep(0.3)  # nvidia-smi start-up
    launches["n"] = 0
    dense_heads["n"] = 0
    stats.update(rung4=0, nv=0.0, pagein=0, steps=0, hits=0, misses=0)
    nb_timed = cache.num_blocks
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start.record()
    for i in range(K):
        one_step(W + i)
    t_end.record()
    torch.cuda.synchronize()
    collect()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / K
    clocks = sampler.stop() if sampler else None
    n_launch = launches["n"]
    n_dense = dense_heads["n"]
    # pass A's own duration (the roofline kernel), from CUDA events the library
    # records around its launch on the step's stream -- in K further steps, since
    # an event between pass A and the selection stops the selection's programmatic
    # launch from overlapping pass A's last wave
    saved = dict(stats), launches["n"], dense_heads["n"]
    for i in range(K):
        one_step(W + i, ev_a[i])
    torch.cuda.synchronize()
    collect()
    stats.clear()
    stats.update(saved[0])
    launches["n"], dense_heads["n"] = saved[1], saved[2]
    pa_ms = sum(a.elapsed_time(b) for a, b in ev_a) / K
    if world > 1:
        t = torch.tensor([ms, pa_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, pa_ms = float(t[0]), float(t[1])

    # ---- end to end through the public API with host buffers -----------------
    e2e = None
    if e2e_wanted:
        # steady state over E >= K steps: the wall clock from the host having read step
        # 0's bound report to it having read step E-1's (every one of those E-1 steps
        # pays its H2D inputs, its bound report and its output D2H); NP pinned input
        # sets cycled
        E, NP = max(K, 60), min(K, 8)
        # the device-timed loop's own inputs (same data: same dense / Rung-4 work)
        qh = qpool[W:W + NP].cpu().pin_memory()
        kh = kpool[W:W + NP].cpu().pin_memory()
        vh = vpool[W:W + NP].cpu().pin_memory()
        oh = torch.empty((U, args.q_per_kv, 128), dtype=torch.float32).pin_memory()
        for i in range(2):  # warm the pinned paths
            dec.step(qh[i].to(dev, non_blocking=True))
            oh.copy_(dec.out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        serial = os.environ.get("CKV_E2E_SERIAL") == "1"
        comp = torch.cuda.current_stream(dev)
        cs = torch.cuda.Stream(device=dev)  # copy stream: PCIe transfers beside the kernels
        # double-buffered device staging: step i+1's inputs land while step i runs,
        # step i's output leaves while step i+1 runs
        qd = [torch.empty_like(dec.q) for _ in range(2)]
        kd = [torch.empty((U, 1, 128), dtype=torch.float16, device=dev) for _ in range(2)]
        vd = [torch.empty_like(kd[0]) for _ in range(2)]
        od = [torch.empty_like(dec.out) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]

        def stage_in(i):  # H2D of step i's queries and new token on the copy stream
            j, b = i % NP, i % 2
            with torch.cuda.stream(cs):
                cs.wait_event(ev_used[b])  # step i-2 is done with these buffers
                qd[b].copy_(qh[j], non_blocking=True)
                kd[b].copy_(kh[j], non_blocking=True)
                vd[b].copy_(vh[j], non_blocking=True)
                ev_in[b].record(cs)

        for ev in ev_used + ev_d2h:
            ev.record(comp)
        ev_step = [torch.cuda.Event(enable_timing=True) for _ in range(E)]
        esampler = ClockSampler(local, dev) if (rank == 0 and clocks_wanted) else None
        if esampler:
            esampler.start()
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        prev = None
        if not serial:
            stage_in(0)
        for i in range(E):
            j, b = i % NP, i % 2
            if serial:
                dec.q.copy_(qh[j], non_blocking=True)            # H2D: this step's queries
                p = dec.step_async(None, reduce_flags)          # + D2H of the certificates
                exchange()
                oh.copy_(dec.out, non_blocking=True)             # D2H: the attention outputs
                kd[0].copy_(kh[j], non_blocking=True)            # H2D: the step's new token
                vd[0].copy_(vh[j], non_blocking=True)
                cache.append(kd[0], vd[0], validate="defer")
            else:
                if i + 1 < E:
                    stage_in(i + 1)
                comp.wait_event(ev_in[b])
                comp.wait_event(ev_d2h[b])                      # step i-2's output has left od[b]
                p = dec.step_async(qd[b], reduce_flags, out=od[b])  # + the bound report to host
                exchange()
                ev_out[b].record(comp)
                ev_step[i].record(comp)
                cache.append(kd[b], vd[b], validate="defer")
                ev_used[b].record(comp)
                with torch.cuda.stream(cs):                     # D2H: the attention outputs
                    cs.wait_event(ev_out[b])
                    oh.copy_(od[b], non_blocking=True)
                    ev_d2h[b].record(cs)
            if prev is not None:
                prev.result()  # host reads step i-1's bound report while step i runs
                if i == 1:  # steady state: from step 0's report to step E-1's
                    e0 = time.perf_counter()
            prev = p
        torch.cuda.synchronize()
        prev.result()
        e_ms = (time.perf_counter() - e0) * 1000.0 / (E - 1)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        h2d = qh[0].numel() * 8 + kh[0].numel() * 2 + vh[0].numel() * 2
        d2h = oh.numel() * 4 + dec.cert_buf.numel()
        e2e = {"value": 1000.0 / e_ms, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms, "steps": E}
        if not serial:  # the device's own step interval inside this loop (diagnostic)
            e2e["device_ms_per_step"] = ev_step[0].elapsed_time(ev_step[E - 1]) / (E - 1)
        if esampler:  # E steps back to back run long enough to meet the board's power cap
            e2e["clocks"] = esampler.stop()

    return dict(ms=ms, pa_ms=pa_ms, clocks=clocks, n_launch=n_launch, n_dense=n_dense,
                stats=stats, last=last, dec=dec, cache=cache, scratch=scratch, e2e=e2e,
                prefill_s=prefill_s, nb_timed=nb_timed, U=U, qpool=qpool)



def _lru_ring(max_blocks, cap):
    """Ring size of an LRU state (lru_ring in csrc/common.cuh)."""
    if cap >= max_blocks:
        return 0
    need, r = 2 * cap + max_blocks + 1024, 1
    while r < need:
        r <<= 1
    return r


def pcie_peak_gbs(dev, nbytes=1 << 30):
    """Pinned host -> HBM DMA bandwidth of this box (1 GiB, best of 5)."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = None
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / 1000.0
        best = t if best is None else min(best, t)
    return nbytes / best / 1e9


def pcie_stats(args, R, ms):
    """Host-Tier-2 configurations are PCIe-bound: bytes read from pinned host RAM
    per step (misses paged into HBM slots by pass B + the dense rungs' blocks
    that are not resident in a slot), the LRU hit rate of the timed steps, and the
    achieved H2D rate against this box's measured DMA bandwidth."""
    import numpy as np
    import torch
    dec, cache, sc, st = R["dec"], R["cache"], R["scratch"], R["stats"]
    steps = max(1, st["steps"])
    pagein = st["pagein"] / steps
    dense_host, n = 0, 3
    maxb = cache.max_blocks
    for i in range(n):  # a few synchronous steps: slot tables as the dense kernel saw them
        res = dec.step(R["qpool"][i])
        units = np.nonzero((res.kinds != 0).any(1))[0]
        nb = cache.num_blocks
        for kind, lru, cap in ((0, sc.key_lru, sc.c.key_capacity), (1, sc.value_lru, sc.c.value_capacity)):
            off = 4 + maxb + _lru_ring(maxb, cap)
            for u in units:
                resident = int((lru[int(u), off:off + nb] >= 0).sum()) if cap > 0 else 0
                dense_host += (nb - resident) * 4096
    dense_host /= n
    total = pagein + dense_host
    peak = pcie_peak_gbs(cache.device)
    achieved = total / (ms / 1000.0) / 1e9
    hm = st["hits"] + st["misses"]
    return {"bound": "pcie", "pagein_bytes_per_step": pagein,
            "dense_host_bytes_per_step": dense_host, "h2d_bytes_per_step": total,
            "achieved_gbs": achieved, "peak_gbs_measured": peak, "frac": achieved / peak,
            "scratch_hit_rate": st["hits"] / hm if hm else 0.0,
            "scratch_blocks_per_kv_head": sc.c.key_capacity,
            "note": "pinned-host Tier-2 read zero-copy by pass B (misses, filling their HBM "
                    "slots) and by k_dense (dense rungs); peak = pinned DMA H2D of 1 GiB, best of 5"}


def run_variant(args, ck, dev, dist, total_units, name="c3host", K=8, W=3, explore=0.0):
    """Another preset on the same box after the main line (fewer steps)."""
    import copy
    va = copy.copy(args)
    pre = PRESETS[name]
    for k in ("ctx", "batch", "tier2", "scratch", "v_tol"):
        setattr(va, k, pre[k])
    va.adversarial, va.desc, va.config, va.explore = pre["adversarial"], pre["desc"], name, explore
    R = run_gpu(va, ck, dev, 1, 0, 0, K, W, dist, total_units, e2e_wanted=False,
                clocks_wanted=False)
    out = {"workload": pre["desc"] + (f", exploration_rate {explore} (device draws)" if explore else ""),
           "value": 1000.0 / R["ms"], "unit": UNIT,
           "ms_per_step": R["ms"], "steps": K, "warmup": W, "pass_a_ms": R["pa_ms"],
           "hbm_frac_step": total_units * va.ctx * 288.0 / (R["ms"] / 1000.0) / 1e9 / peak_hbm()[0],
           "dense_heads_in_timed_region": R["n_dense"]}
    if va.tier2 == "host":
        out["pcie"] = pcie_stats(va, R, R["ms"])
    return out


def main():
    args = parse()
    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knob for exercising the sharded path on a single GPU (every rank on cuda:0, gloo)
    if os.environ.get("CKV_BENCH_ONE_DEVICE"):
        local = 0
    K, W = args.steps, max(3, args.warmup)
    total_units = args.layers * args.kv_heads * args.batch
    pol_desc = f"PolicyConfig(exploration_rate={args.explore}) defaults"
    if args.v_tol is not None:
        pol_desc = f"PolicyConfig(exploration_rate={args.explore}, v_tol={args.v_tol})"
    tier1_gb = total_units * args.ctx * 288 / 1e9
    config = {"workload": args.desc if args.ctx == PRESETS[args.config]["ctx"] else
              f"{args.config.upper()} shape at {args.ctx} ctx, batch {args.batch}",
              "ctx": args.ctx, "layers": args.layers, "kv_heads": args.kv_heads,
              "q_heads": args.kv_heads * args.q_per_kv, "batch": args.batch,
              "parallelism": f"kv-head shard x{args.gpus}",
              "policy": pol_desc,
              "l2": f"inputs larger than L2 (Tier-1 {tier1_gb:.2f} GB/step)",
              "tier2": args.tier2}

    if args.impl == "reference":
        if rank != 0:
            return
        try:
            ncpu = len(os.sched_getaffinity(0))
        except Exception:
            ncpu = os.cpu_count() or 1
        workers = max(1, min(ncpu, 32, total_units))
        rate, kind, detail = cpu_reference(args, total_units, K, W, workers)
        line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": K,
                "warmup": W, "ms_per_step": 1000.0 / rate, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": rate, "unit": UNIT, "cores": workers, "kind": kind,
                                 "sample": f"{workers} of {total_units} units (one per process, "
                                           f"single-threaded) at {args.ctx} ctx, {args.q_per_kv} "
                                           f"q-heads each, {K} timed steps after {W} warm-up; "
                                           f"scaled x{total_units / workers:.1f}",
                                 **detail},
                "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        if os.environ.get("CKV_BENCH_ONE_DEVICE"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    from paper_2605_20868_b200 import _lib
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    R = run_gpu(args, ck, dev, world, rank, local, K, W, dist, total_units,
                e2e_wanted=not args.no_e2e)
    ms, pa_ms, e2e, U = R["ms"], R["pa_ms"], R["e2e"], R["U"]
    dec, cache, stats, last = R["dec"], R["cache"], R["stats"], R["last"]
    pcie = pcie_stats(args, R, ms) if args.tier2 == "host" else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = peak_hbm()
    tier1_bytes_launch = U * R["nb_timed"] * _lib.BLOCK_BYTES  # Tier-1 read by one pass A
    achieved = tier1_bytes_launch / (pa_ms / 1000.0) / 1e9
    step_bytes = total_units * args.ctx * 288.0
    step_frac = step_bytes / (ms / 1000.0) / 1e9 / peak
    # DRAM bytes per pass-A launch from an ncu capture of THIS configuration
    # (tools/traffic.py -> profiles/traffic_r02.json, keyed by the workload shape)
    traffic = None
    tkey = f"{args.config}:{args.ctx}:{args.batch}:{args.tier2}:{U}"
    tfile = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(tfile):
        try:
            ent = json.load(open(tfile)).get(tkey)
            if ent:
                traffic = ent["k_pass_a"]["dram_bytes_per_launch"]
        except Exception:
            traffic = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, kind, detail = cpu_reference(args, total_units, 2, 1, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"1 of {total_units} units at {args.ctx} ctx ({args.q_per_kv} q-heads "
                         f"+ append), 2 timed unit-steps on one core, scaled x{total_units}",
               **detail}

    value = 1000.0 / ms
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int8/int4 codes, fp32 accumulate", "data": "synthetic",
        "config": config,
        "hbm_frac_step": step_frac,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_pass_a (Tier-1 stream, Phase 1 + speculative Phase 2)",
                     "peak_kind": peak_kind, "pass_a_ms": pa_ms},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": R["n_launch"],
        "k_star_mean": float(last["res"].cert["k_star"].mean()),
        "promoted_union_blocks_per_unit": float(dec.n_work.float().mean().item()),
        "dense_heads_in_timed_region": R["n_dense"],
        "rung4_heads_in_timed_region": stats["rung4"],
        "value_promoted_per_head_mean": stats["nv"] / max(1, stats["steps"]),
        "pagein_bytes_per_step": stats["pagein"] / max(1, stats["steps"]),
        "clocks": R["clocks"],
        "prefill_s": R["prefill_s"],
    }
    if pcie is not None:
        line["pcie"] = pcie
    if args.config == "c3" and world == 1 and not args.no_variant:
        # the north-star placement of the same workload: Tier-2 in pinned host RAM,
        # the reference's 2048-block scratch, misses over PCIe (bench --config c3host)
        del R, dec, cache, last
        torch.cuda.empty_cache()
        line["variant_c3host"] = run_variant(args, ck, dev, dist, total_units)
        torch.cuda.empty_cache()
        line["variant_c3_explore"] = run_variant(args, ck, dev, dist, total_units, name="c3",
                                                 explore=0.02)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
