"""Fraction of blocks pass A stashes vs the union pass B needs (C3-shaped, 64 units)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
import paper_2605_20868_b200 as ck
U, ctx = 64, 131072
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, ctx + 64, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
for pos in range(0, ctx, 4096):
    cache.append(torch.randn((U, 4096, 128), generator=g, device=dev).half(),
                 torch.randn((U, 4096, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4)
for i in range(4):
    dec.step(torch.randn((U, 4, 128), generator=g, device=dev, dtype=torch.float64))
    nb = cache.num_blocks
    stashed = ((dec.stash_epoch[:, :nb] >> 4) == dec.st.epoch).sum().item() / (U * nb)
    union = dec.n_work.float().mean().item() / nb
    nwm = int(dec.n_work.max().item())
    blk = (dec.work[:, :nwm] & 0xffffff).long()
    valid = torch.arange(nwm, device=dev)[None, :] < dec.n_work[:, None]
    hit = (torch.gather(dec.stash_epoch[:, :], 1, blk.clamp(max=cache.max_blocks - 1)) >> 4) == dec.st.epoch
    cov = (hit & valid).sum().item() / valid.sum().item()
    print(f"step {i}: stashed {stashed:.3f} of blocks, union {union:.3f}, union items stashed {cov:.3f}")
