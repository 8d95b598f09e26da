"""KV-head sharding across GPUs — host-side logic.

All state of the certified path is per unit (one (layer, KV head, sequence)
cache; harness.py:150-155, 346-347), so a rank that owns a set of KV heads
computes their outputs and certificates with no data from other ranks.  The
only exchange per step is the bound report: outputs + certificates gathered
with one collective, and the step-wide Rung-4 flag (harness.py:362-372)
reduced with MAX per layer so every rank can recompute its own flagged units
densely from its local Tier-2.
"""

import numpy as np
import torch
import torch.distributed as dist

CERT_BYTES = 88


def unit_index(layer, seq, kv, layers, batch):
    """kv-major unit numbering: contiguous ranges are KV-head subsets."""
    return (kv * layers + layer) * batch + seq


def shard_units(layers, kv_heads, batch, world, rank):
    """Units owned by ``rank``: the KV heads [rank*kv/world, (rank+1)*kv/world)."""
    if kv_heads % world:
        raise ValueError(f"{kv_heads} KV heads cannot be sharded over {world} ranks")
    per = kv_heads // world
    lo = rank * per * layers * batch
    return range(lo, lo + per * layers * batch)


def layer_of_units(units, layers, batch):
    """Layer index of every unit in ``units`` (kv-major numbering)."""
    u = np.asarray(list(units))
    return (u // batch) % layers


def pack_step(out, cert_bytes):
    """One flat uint8 buffer: outputs (fp32) then certificates (raw structs)."""
    return torch.cat([out.contiguous().view(torch.uint8).reshape(-1),
                      cert_bytes.contiguous().reshape(-1)])


def unpack_gathered(buf, world, n_local, n_heads, head_dim=128):
    """Inverse of pack_step for an all-gathered buffer -> (out [world*n_local, nh, d],
    cert bytes [world*n_local, nh, CERT_BYTES])."""
    per_out = n_local * n_heads * head_dim * 4
    per_cert = n_local * n_heads * CERT_BYTES
    parts = buf.view(world, per_out + per_cert)
    out = parts[:, :per_out].contiguous().view(torch.float32).reshape(world * n_local, n_heads, head_dim)
    cert = parts[:, per_out:].reshape(world * n_local, n_heads, CERT_BYTES)
    return out, cert


def _host_staged(t, group):
    """gloo collectives run on host tensors: stage device tensors through RAM."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def gather_bound_report(out, cert_bytes, group=None):
    """All-gather of the packed step (NCCL over NVLink; gloo via host memory)."""
    world = dist.get_world_size(group)
    local = pack_step(out, cert_bytes)
    staged = _host_staged(local, group)
    src = local.cpu() if staged else local
    buf = torch.empty(world * src.numel(), dtype=torch.uint8, device=src.device)
    dist.all_gather_into_tensor(buf, src, group=group)
    return buf.to(local.device) if staged else buf


def reduce_group_flags(flags, group=None):
    """Step-wide Rung-4 requests, MAX over the ranks, in place (stream-ordered
    with NCCL; host-staged with gloo)."""
    if _host_staged(flags, group):
        f = flags.cpu()
        dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
        flags.copy_(f)
    else:
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)


def rung4_layers(flags_per_unit, layers_of_units, layers, group=None, device="cpu"):
    """Per-layer OR of local Rung-4 requests, reduced with MAX across ranks."""
    f = torch.zeros(layers, dtype=torch.int32, device=device)
    for fl, ly in zip(flags_per_unit, layers_of_units):
        if fl:
            f[int(ly)] = 1
    if dist.is_initialized():
        dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
    return f.cpu().numpy().astype(bool)
