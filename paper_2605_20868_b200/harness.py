"""Workloads, the decode step loop and the bound report (harness.py of the
reference, 41-499), driven through the batched device decoder.

``run_workload`` keeps the reference's per-step order: every q-head is
certified (here all at once on the GPU), a canary trip anywhere makes the
whole step dense (harness.py:362-372), a telemetry record is emitted, then one
new token is appended per KV head (quantize-on-append on the device).
"""

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import DeviceKVCache, ScratchCache
from .engine import CertifiedDecoder, certificate_from_row
from .policy import RETURNED_QUANTIZED, events_from_flags

RNG_ALGORITHM = "philox4x64"
WORKLOAD_KINDS = ("gaussian", "sink", "needle", "near_tie")


@dataclass(frozen=True)
class WorkloadConfig:
    """Fields and defaults of the reference WorkloadConfig (harness.py:41-81).

    The device path runs head_dim 128, block 16, group 16 with FP16 originals
    (binary16 ingest) and at most 4 q-heads per KV head; any other geometry --
    including the reference's own defaults (head_dim=64, float32 ingest) --
    raises ValueError instead of being coerced.
    """
    kind: str = "gaussian"
    n_tokens: int = 1024
    head_dim: int = 64
    block_size: int = 16
    group_size: int = 16
    query_heads: int = 1
    kv_heads: int = 1
    steps: int = 8
    seed: int = 0
    ingest_binary16: bool = False

    def __post_init__(self):
        if self.kind not in WORKLOAD_KINDS:
            raise ValueError(f"unknown workload kind {self.kind!r}")
        if self.n_tokens < 1:
            raise ValueError("n_tokens must be at least 1")
        if self.steps < 1:
            raise ValueError("steps must be at least 1")
        if self.query_heads % self.kv_heads != 0:
            raise ValueError("kv_heads must divide query_heads")
        if self.head_dim % self.group_size != 0:
            raise ValueError("group_size must divide head_dim")
        if (self.head_dim, self.block_size, self.group_size) != (_lib.HEAD_DIM, _lib.BLOCK,
                                                                 _lib.GROUP):
            raise ValueError("the device path supports head_dim=128, block_size=16, "
                             f"group_size=16 (got {self.head_dim}, {self.block_size}, "
                             f"{self.group_size})")
        if not self.ingest_binary16:
            raise ValueError("the device path stores FP16 originals: ingest_binary16 must be True")
        if self.query_heads // self.kv_heads > _lib.MAX_QHEADS:
            raise ValueError("the device path supports up to 4 query heads per KV head")

    @property
    def group_factor(self):
        return self.query_heads // self.kv_heads

    def kv_index(self, query_head):
        return query_head // self.group_factor

    def to_dict(self):
        return dataclasses.asdict(self)

    @classmethod
    def from_dict(cls, data):
        unknown = set(data) - {f.name for f in dataclasses.fields(cls)}
        if unknown:
            raise ValueError(f"unknown workload fields: {sorted(unknown)}")
        return cls(**data)


@dataclass
class Workload:
    config: WorkloadConfig
    cache: DeviceKVCache
    queries: np.ndarray      # float64 [steps, query_heads, d]
    new_keys: np.ndarray     # float32 [steps, kv_heads, d]
    new_values: np.ndarray


def _philox(seed, purpose):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, purpose))))


def synth_arrays(cfg):
    """Seeded K/V/queries, identical draws to generate_workload (harness.py:97-148)."""
    d = cfg.head_dim
    rng = _philox(cfg.seed, 0)
    total = cfg.n_tokens + cfg.steps
    keys = rng.standard_normal((cfg.kv_heads, total, d))
    values = rng.standard_normal((cfg.kv_heads, total, d))
    queries = rng.standard_normal((cfg.steps, cfg.query_heads, d))
    kappa = 3.0
    dirs = np.empty((cfg.kv_heads, d))
    for kv in range(cfg.kv_heads):
        w = rng.standard_normal(d)
        dirs[kv] = w / np.linalg.norm(w)
    if cfg.kind != "gaussian":
        for h in range(cfg.query_heads):
            queries[:, h, :] += kappa * dirs[cfg.kv_index(h)]
    b = cfg.block_size
    if cfg.kind == "sink":
        span = min(b, cfg.n_tokens)
        for kv in range(cfg.kv_heads):
            keys[kv, :span] = 2.0 * np.sqrt(d) / kappa * dirs[kv] + 0.1 * keys[kv, :span]
    elif cfg.kind == "needle":
        for kv in range(cfg.kv_heads):
            keys[kv, cfg.n_tokens // 2] = 2.5 * np.sqrt(d) / kappa * dirs[kv]
    elif cfg.kind == "near_tie":
        if cfg.n_tokens < 2 * b:
            raise ValueError("near_tie needs at least two full blocks")
        for kv in range(cfg.kv_heads):
            base = 2.0 * np.sqrt(d) / kappa * dirs[kv] + 0.5 * keys[kv, :b]
            keys[kv, :b] = base
            keys[kv, b:2 * b] = base + 1e-4 * rng.standard_normal((b, d))
    return keys, values, queries


def generate_workload(config, device="cuda", tier2="device"):
    """Build the device caches (one unit per KV head) and the query stream."""
    cfg = config
    keys, values, queries = synth_arrays(cfg)
    cache = DeviceKVCache(cfg.kv_heads, cfg.n_tokens + cfg.steps, device=device, tier2=tier2)
    cache.append(torch.from_numpy(keys[:, :cfg.n_tokens]), torch.from_numpy(values[:, :cfg.n_tokens]))
    return Workload(cfg, cache, queries,
                    np.swapaxes(keys[:, cfg.n_tokens:], 0, 1).astype(np.float32),
                    np.swapaxes(values[:, cfg.n_tokens:], 0, 1).astype(np.float32))


def gqa_union(n_tokens, block_size, k_max, query_heads, rung1_active=True):
    """Expected per-cache promoted working set (harness.py:303-315)."""
    if min(n_tokens, block_size, k_max, query_heads) <= 0:
        raise ValueError("all union parameters must be positive")
    nb = -(-int(n_tokens) // int(block_size))
    k_eff = min((2 if rung1_active else 1) * int(k_max), nb)
    fraction = 1.0 - (1.0 - k_eff / nb) ** int(query_heads)
    return nb * fraction, fraction


@dataclass
class RunResult:
    header: dict
    step_records: list
    summary: dict


def _mean(xs):
    return float(np.mean(xs)) if xs else 0.0


def _max(xs):
    return float(np.max(xs)) if xs else 0.0


def step_record(step, certs, events, kscr, vscr, bytes_paged, staging, union_fractions):
    """Telemetry record of one step, schema of harness.py:397-447."""
    rc = {f"rung{i}": 0 for i in (1, 2, 3, 4)}
    cc = {}
    for e in events:
        rc[f"rung{e.rung}"] += 1
        cc[e.cause] = cc.get(e.cause, 0) + 1
    return {
        "step": step,
        "e_key_step_mean": _mean([c.e_key_impl for c in certs]),
        "e_key_step_max": _max([c.e_key_impl for c in certs]),
        "e_key_step_mean_returned": _mean([c.returned_e_key for c in certs]),
        "e_key_step_max_returned": _max([c.returned_e_key for c in certs]),
        "e_val_step_mean": _mean([c.e_val for c in certs]),
        "e_val_step_max": _max([c.e_val for c in certs]),
        "e_val_step_mean_returned": _mean([c.returned_e_val for c in certs]),
        "e_val_step_max_returned": _max([c.returned_e_val for c in certs]),
        "k_star_mean": _mean([c.k_star for c in certs]),
        "est_tail_mass_mean": _mean([c.est_tail_mass for c in certs]),
        "delta_h_max": _max([c.delta_h for c in certs]),
        "rung_counts": rc,
        "cause_counts": cc,
        "events": [e.to_dict() for e in events],
        "certificates": [c.to_dict() for c in certs],
        "key_scratch": kscr,
        "value_scratch": vscr,
        "bytes_paged_in": bytes_paged,
        "rung4_staging_bytes": staging,
        "union_fraction_mean": _mean(union_fractions),
    }


def aggregate_telemetry(step_records, config, layers=1):
    """Run summary (harness.py:450-499)."""
    steps = len(step_records)
    head_steps = steps * config.query_heads * layers
    rt = {f"rung{i}": 0 for i in (1, 2, 3, 4)}
    ct = {}
    for rec in step_records:
        for k, v in rec["rung_counts"].items():
            rt[k] += v
        for k, v in rec["cause_counts"].items():
            ct[k] = ct.get(k, 0) + v
    certs = [c for rec in step_records for c in rec["certificates"]]

    def stats(key):
        vals = [c[key] for c in certs]
        return {"mean": _mean(vals), "max": _max(vals)}

    dense = sum(1 for c in certs if c["returned_kind"] != RETURNED_QUANTIZED)
    return {
        "steps": steps, "head_steps": head_steps, "layers": layers,
        "rung_counts": rt, "cause_counts": ct,
        "rates": {"rung3_per_head_step": rt["rung3"] / head_steps if head_steps else 0.0,
                  "rung4_per_step": rt["rung4"] / steps if steps else 0.0,
                  "dense_fraction": dense / head_steps if head_steps else 0.0},
        "e_key_candidate": stats("e_key_impl"),
        "e_key_tight_candidate": stats("e_key_tight"),
        "e_key_returned": stats("returned_e_key"),
        "e_val": stats("e_val"),
        "e_val_returned": stats("returned_e_val"),
        "k_star_mean": _mean([c["k_star"] for c in certs]),
        "est_tail_mass_mean": _mean([c["est_tail_mass"] for c in certs]),
        "bytes_paged_in_total": sum(r["bytes_paged_in"] for r in step_records),
        "rung4_staging_bytes_total": sum(r["rung4_staging_bytes"] for r in step_records),
        "union_fraction_mean": _mean([r["union_fraction_mean"] for r in step_records]),
    }


def _scr(h, m):
    return {"hits": int(h), "misses": int(m), "hit_rate": h / (h + m) if h + m else 0.0,
            "bytes_paged_in": int(m) * _lib.BLOCK * _lib.HEAD_DIM * 2}


def run_workload(workload, policy, key_capacity=2048, value_capacity=2048, layers=1,
                 keep_outputs=False, keep_decisions=False):
    """Drive a workload through decode (harness.py:339-394).

    ``keep_outputs`` adds ``result.outputs`` (per step, [query_heads, d]);
    ``keep_decisions`` adds ``result.decisions`` (per step, per q-head: the
    promoted block ids and the value-promoted block ids, ascending)."""
    cfg = workload.config
    if cfg.group_factor > _lib.MAX_QHEADS:
        raise ValueError("device path supports up to 4 query heads per KV head")
    cache = workload.cache
    explore_rng = _philox(cfg.seed, 1)  # harness.py:348
    scratch = ScratchCache(key_capacity, value_capacity)
    dec = CertifiedDecoder(cache, policy, n_heads=cfg.group_factor, scratch=scratch)
    gf = cfg.group_factor
    records, outputs, decisions = [], [], []
    for step in range(cfg.steps):
        q = torch.from_numpy(workload.queries[step].reshape(cfg.kv_heads, gf, cfg.head_dim))
        res = dec.step(q.to(cache.device), rng=explore_rng)
        certs, events = [], []
        for h in range(cfg.query_heads):
            u, j = divmod(h, gf)
            row = res.cert[u, j]
            certs.append(certificate_from_row(row, h, step, res.kinds[u, j]))
            events.extend(events_from_flags(int(row["flags"]), h, step))
        ps = res.page_stats.sum(0)
        fr = []
        if cache.num_blocks:
            for u in range(cfg.kv_heads):
                un = set()
                for j in range(gf):
                    un.update(int(b) for b in res.promoted(u, j))
                fr.append(len(un) / cache.num_blocks)
        bytes_paged = int(ps[1] + ps[3]) * _lib.BLOCK * _lib.HEAD_DIM * 2
        if res.explore_counts is not None:
            bytes_paged += int(res.explore_counts.sum()) * _lib.BLOCK * _lib.HEAD_DIM * 2
        records.append(step_record(step, certs, events, _scr(ps[0], ps[1]), _scr(ps[2], ps[3]),
                                   bytes_paged, res.staging_bytes, fr))
        if keep_outputs:
            outputs.append(res.out.double().cpu().numpy().reshape(cfg.query_heads, -1).copy())
        if keep_decisions:
            decisions.append([(sorted(int(b) for b in res.promoted(*divmod(h, gf))),
                               sorted(int(b) for b in res.value_promotions(*divmod(h, gf))))
                              for h in range(cfg.query_heads)])
        cache.append(torch.from_numpy(workload.new_keys[step])[:, None, :],
                     torch.from_numpy(workload.new_values[step])[:, None, :])
    header = {"config": cfg.to_dict(), "policy": policy.to_dict(), "seed": cfg.seed,
              "rng": RNG_ALGORITHM, "scratch": {"key_capacity": key_capacity,
                                                "value_capacity": value_capacity},
              "layers": layers}
    rr = RunResult(header, records, aggregate_telemetry(records, cfg, layers=layers))
    if keep_outputs:
        rr.outputs = outputs
    if keep_decisions:
        rr.decisions = decisions
    return rr


def _jsonable(obj):
    if isinstance(obj, dict):
        return {k: _jsonable(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_jsonable(v) for v in obj]
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.floating):
        return float(obj)
    if isinstance(obj, np.ndarray):
        return [_jsonable(v) for v in obj.tolist()]
    return obj


def dump_line(obj):
    """One deterministic JSONL line (cli.py:80-95: sorted keys, compact separators)."""
    import json
    return json.dumps(_jsonable(obj), sort_keys=True, separators=(",", ":"))


def write_telemetry(result, path, config_path="", seed_override=None, version="0.1.0"):
    """The bound report as the reference CLI writes it (cli.py:98-117): a header
    line, one line per step record, one summary line."""
    header = dict(result.header)
    header["kind"] = "header"
    header["manifest"] = {"config_path": config_path, "seed_override": seed_override}
    header["rng"] = RNG_ALGORITHM
    header["kernel_backend"] = "b200"
    header["version"] = version
    with open(path, "w") as fh:
        fh.write(dump_line(header) + "\n")
        for record in result.step_records:
            fh.write(dump_line({"kind": "step", **record}) + "\n")
        fh.write(dump_line({"kind": "summary", **result.summary}) + "\n")
    return path


_CONFIG_SECTIONS = {"workload", "policy", "scratch", "seed", "layers"}
_SCRATCH_FIELDS = {"key_capacity", "value_capacity"}


def resolve_manifest(config_path, seed=None):
    """A run manifest (JSON) resolved as the reference CLI resolves it
    (cli.py:36-77): the same sections, seed override, scratch defaults of 2048
    blocks and error messages (``ValueError`` here for the CLI's ConfigError)."""
    import json
    from .policy import PolicyConfig
    try:
        with open(config_path) as fh:
            raw = json.load(fh)
    except OSError as exc:
        raise ValueError(f"cannot read config: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ValueError(f"malformed JSON at line {exc.lineno}, column {exc.colno}: {exc.msg}") from exc
    if not isinstance(raw, dict):
        raise ValueError("config root must be a JSON object")
    unknown = set(raw) - _CONFIG_SECTIONS
    if unknown:
        raise ValueError(f"unknown config sections: {sorted(unknown)}")
    workload_raw = dict(raw.get("workload", {}))
    if seed is not None:
        workload_raw["seed"] = seed
    elif "seed" in raw:
        workload_raw.setdefault("seed", raw["seed"])
    workload = WorkloadConfig.from_dict(workload_raw)
    policy = PolicyConfig.from_dict(raw.get("policy", {}))
    scratch = dict(raw.get("scratch", {}))
    unknown = set(scratch) - _SCRATCH_FIELDS
    if unknown:
        raise ValueError(f"unknown scratch fields: {sorted(unknown)}")
    return (workload, policy, int(scratch.get("key_capacity", 2048)),
            int(scratch.get("value_capacity", 2048)), int(raw.get("layers", 1)))


def run_manifest(config_path, out_path, seed=None):
    """``certkv run`` (cli.py:98-117) on the device path: resolve the manifest,
    run the workload, write the bound report (header, one line per step, summary)
    to ``out_path``.  Returns the RunResult."""
    workload_cfg, policy, key_cap, value_cap, layers = resolve_manifest(config_path, seed)
    result = run_workload(generate_workload(workload_cfg), policy, key_capacity=key_cap,
                          value_capacity=value_cap, layers=layers)
    write_telemetry(result, out_path, config_path=config_path, seed_override=seed)
    return result
