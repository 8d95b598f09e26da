"""Multi-process (world_size 2, gloo on CPU) coverage of the KV-head sharded
path: unit partitioning, the packed all-gather of outputs + certificates and
the per-layer Rung-4 flag reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_20868_b200 import sharding


def test_shard_partition_covers_units_once():
    layers, kv, batch = 32, 8, 2
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            units = list(sharding.shard_units(layers, kv, batch, world, r))
            seen.extend(units)
            kvs = {(u // batch) // layers for u in units}
            assert len(kvs) == kv // world  # whole KV heads per rank
        assert sorted(seen) == list(range(layers * kv * batch))
    with pytest.raises(ValueError):
        sharding.shard_units(32, 8, 1, 3, 0)


def test_unit_index_roundtrip():
    layers, batch = 4, 3
    for kv in range(2):
        for ly in range(layers):
            for s in range(batch):
                u = sharding.unit_index(ly, s, kv, layers, batch)
                assert sharding.layer_of_units([u], layers, batch)[0] == ly


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers, kv, batch, nh = 4, 2, 1, 4
        units = list(sharding.shard_units(layers, kv, batch, world, rank))
        n_local = len(units)
        out = torch.full((n_local, nh, 128), float(rank + 1))
        cert = torch.full((n_local, nh, sharding.CERT_BYTES), rank + 7, dtype=torch.uint8)
        buf = sharding.gather_bound_report(out, cert)
        o, c = sharding.unpack_gathered(buf, world, n_local, nh)
        ok = bool((o[:n_local] == 1).all() and (o[n_local:] == 2).all()
                  and (c[:n_local] == 7).all() and (c[n_local:] == 8).all())
        # rank 1 requests Rung 4 in layer 2 only
        lyr = sharding.layer_of_units(units, layers, batch)
        flags = [(rank == 1 and ly == 2) for ly in lyr]
        f = sharding.rung4_layers(flags, lyr, layers)
        ok = ok and f.tolist() == [False, False, True, False]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gather_and_rung4_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
