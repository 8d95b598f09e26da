"""The reference's own CPU implementation of the path, timed on the host cores.

BASELINE INFRASTRUCTURE ONLY (bench.py's ``--impl reference`` arm and its
``cpu_baseline`` leg).  It drives the UNMODIFIED reference package built by
``oracle/build_ref.sh`` into ``oracle/_ref`` (certkv with its compiled Cython
kernel backend) through its public API: ``certkv.TieredCache.append_tokens``
for the prefill and ``certkv.harness.run_workload`` (harness.py:339-394) for
the decode steps -- per step every q-head of the unit through
``run_decode_step``, the step-wide Rung 4, the telemetry record and the
quantize-on-append of the new token.

One worker process holds one unit (one KV head with its q-heads, i.e. one
``run_workload`` over a single-KV-head workload); ``workers`` processes run in
parallel, each single-threaded (the reference is single-threaded apart from
BLAS, and more BLAS threads slowed it).  A full decode step of the
benchmarked model is ``total_units`` unit-steps, so the measured time per
parallel round is scaled by ``total_units / workers``.
"""

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")

_W = {}


def available():
    return os.path.isfile(os.path.join(REF, "certkv", "__init__.py"))


def _limit_threads():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _import_certkv():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import certkv
    return certkv


def _init(ctx, q_per_kv, seed, n_steps, v_tol, adversarial, explore=0.0):
    _limit_threads()
    import numpy as np
    certkv = _import_certkv()
    from certkv.fallback import PolicyConfig
    from certkv.harness import Workload, WorkloadConfig
    rng = np.random.default_rng(seed)
    total = ctx + n_steps
    keys = rng.standard_normal((total, 128))
    values = rng.standard_normal((total, 128))
    if adversarial:  # bench.py's C5 shape: outlier key channels, near-tie twin blocks
        keys[:, 3] *= 1000.0
        keys[:, 77] *= 1000.0
        keys[16:32] = keys[0:16] + 1e-4 * rng.standard_normal((16, 128))
    queries = rng.standard_normal((n_steps, q_per_kv, 128))
    t0 = time.perf_counter()
    cache = certkv.TieredCache(16, 128, group_size=16, ingest_binary16=True)
    cache.append_tokens(keys[:ctx], values[:ctx])
    cfg = WorkloadConfig(kind="gaussian", n_tokens=ctx, head_dim=128, query_heads=q_per_kv,
                         kv_heads=1, steps=n_steps, seed=seed, ingest_binary16=True)
    wl = Workload(cfg, [cache], queries, keys[ctx:, None, :].astype(np.float32),
                  values[ctx:, None, :].astype(np.float32))
    pol = PolicyConfig(exploration_rate=explore) if v_tol is None else \
        PolicyConfig(exploration_rate=explore, v_tol=v_tol)
    _W.update(wl=wl, pol=pol, next=0, prefill_s=time.perf_counter() - t0,
              backend=certkv._kernels.get_backend().NAME)


def _run(n):
    """``run_workload`` over the next ``n`` steps of this worker's stream."""
    import dataclasses
    from certkv.harness import Workload, run_workload
    wl, i = _W["wl"], _W["next"]
    part = Workload(dataclasses.replace(wl.config, steps=n), wl.caches,
                    wl.queries[i:i + n], wl.new_keys[i:i + n], wl.new_values[i:i + n])
    t0 = time.perf_counter()
    run_workload(part, _W["pol"], key_capacity=2048, value_capacity=2048)
    _W["next"] = i + n
    return time.perf_counter() - t0, _W["prefill_s"], _W["backend"]


def host_info():
    info = {"cpu_model": None, "cores_visible": None, "threads_per_process": 1}
    try:
        info["cores_visible"] = len(os.sched_getaffinity(0))
    except Exception:
        info["cores_visible"] = os.cpu_count()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["threadpools"] = [{k: p.get(k) for k in ("internal_api", "num_threads", "version")}
                               for p in threadpool_info()]
    except Exception:
        pass
    return info


def _worker(w, args, barrier, out):
    ctx, q_per_kv, seed, n, v_tol, adversarial, warmup, steps, explore = args
    _init(ctx, q_per_kv, seed + w, n, v_tol, adversarial, explore)
    barrier.wait()
    if warmup:
        _run(warmup)
    barrier.wait()  # every unit starts its timed steps together
    out.put(_run(steps))


def time_reference(ctx, q_per_kv, total_units, steps, warmup, workers, v_tol=None,
                   adversarial=False, seed=1234, explore=0.0):
    """Seconds per full decode step (``total_units`` unit-steps) of the unmodified
    reference: ``workers`` processes (one unit each) run ``warmup`` then ``steps``
    steps concurrently; the slowest worker's time counts."""
    import multiprocessing as mp
    ctxm = mp.get_context("fork")
    barrier = ctxm.Barrier(workers)
    out = ctxm.Queue()
    args = (ctx, q_per_kv, seed, warmup + steps, v_tol, adversarial, warmup, steps, explore)
    procs = [ctxm.Process(target=_worker, args=(w, args, barrier, out)) for w in range(workers)]
    for p in procs:
        p.start()
    res = [out.get() for _ in procs]
    for p in procs:
        p.join()
    dt = max(r[0] for r in res) / steps  # one parallel round = `workers` unit-steps
    sec_per_step = dt * total_units / workers
    return {"sec_per_step": sec_per_step, "round_s": dt, "prefill_s": max(r[1] for r in res),
            "backend": res[0][2]}
