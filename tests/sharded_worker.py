"""Worker of tests/test_gpu_sharded.py (launched with torch.distributed.run, gloo,
every rank on cuda:0): runs the KV-head-sharded certified step exactly as
bench.py does -- each rank owns whole KV heads (kv-major units), the per-layer
Rung-4 request is all-reduced (MAX) between ckv_decode_flags and
ckv_decode_finish, outputs + certificates are all-gathered as the bound report
-- and rank 0 compares the gathered result with one unsharded decoder over
every unit, bit for bit.  A corrupted key offset in a unit of rank 1 (layer 2)
must make layer 2 dense on rank 0 as well."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_20868_b200 import sharding  # noqa: E402

L, KV, BATCH, NH, CTX, STEPS = 4, 4, 1, 4, 2500, 3
U = L * KV * BATCH
CORRUPT = (sharding.unit_index(2, 0, 3, L, BATCH), 5, 7, 5.0e4)  # kv head 3 = rank 1 at world 2


def run(ck, units, dev, reduce_flags=None):
    g = torch.Generator().manual_seed(11)  # the same data on every rank
    K = torch.randn((U, CTX + STEPS, 128), generator=g).half()
    V = torch.randn((U, CTX + STEPS, 128), generator=g).half()
    Q = torch.randn((STEPS, U, NH, 128), generator=g, dtype=torch.float64)
    idx = torch.as_tensor(list(units))
    cache = ck.DeviceKVCache(len(units), CTX + STEPS + 16, device=dev)
    cache.append(K[idx, :CTX].to(dev), V[idx, :CTX].to(dev))
    if CORRUPT[0] in units:
        cache.corrupt_offset(list(units).index(CORRUPT[0]), *CORRUPT[1:])
    groups = np.asarray(list(units)) % (L * BATCH)  # the (layer, sequence) of every unit
    dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=NH,
                              rung4_group=groups, plan_units=U, dense_splits=64)
    outs, certs, kinds = [], [], []
    for s in range(STEPS):
        res = dec.step_async(Q[s, idx].to(dev), reduce_flags).result()
        outs.append(dec.out.clone())
        certs.append(dec.cert_buf.clone())
        kinds.append(res.kinds.copy())
        cache.append(K[idx, CTX + s:CTX + s + 1].to(dev), V[idx, CTX + s:CTX + s + 1].to(dev))
    return outs, certs, kinds


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_20868_b200 as ck
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    mine = sharding.shard_units(L, KV, BATCH, world, rank)

    outs, certs, kinds = run(ck, mine, dev, sharding.reduce_group_flags)
    gathered = []
    for o, c in zip(outs, certs):  # device tensors: the library stages them for gloo
        buf = sharding.gather_bound_report(o, c)
        gathered.append(sharding.unpack_gathered(buf.cpu(), world, len(mine), NH))
    if rank == 0:
        ref_o, ref_c, ref_k = run(ck, range(U), dev)
        for s in range(STEPS):
            o, c = gathered[s]
            assert torch.equal(o, ref_o[s].cpu()), f"step {s}: outputs differ"
            assert torch.equal(c, ref_c[s].cpu()), f"step {s}: certificates differ"
            kind = ref_k[s]
            layer2 = [u for u in range(U) if u % L == 2]
            assert (kind[layer2] == 2).all(), "layer 2 is not dense on every rank"
            assert not (kind[[u for u in range(U) if u % L != 2]] == 2).any()
            assert (kinds[s][[i for i, u in enumerate(mine) if u % L == 2]] == 2).all()
        print(f"SHARDED OK world={world} units={U} steps={STEPS}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
