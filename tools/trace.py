"""Overlap-aware timeline of one decode step (ckv_step.trace): per kernel the
first CTA start and the last CTA end (globaltimer), averaged over K steps,
relative to pass A's first CTA.  Usage: python tools/trace.py [--kv-heads N]
[--ctx N] [--explore R] [--no-flow]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
ap = argparse.ArgumentParser()
ap.add_argument("--kv-heads", type=int, default=8)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--ctx", type=int, default=131072)
ap.add_argument("--explore", type=float, default=0.0)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--tier2", default="device")
ap.add_argument("--scratch", type=int, default=-1)
args = ap.parse_args()
import __graft_entry__
__graft_entry__.build()
import paper_2605_20868_b200 as ck
from paper_2605_20868_b200.cache import _ptr
U = args.layers * args.kv_heads
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, args.ctx + 4 * args.steps + 64, tier2=args.tier2)
g = torch.Generator(device=dev).manual_seed(1000)
chunk = max(16, min(4096, (1 << 22) // U))
for pos in range(0, args.ctx, chunk):
    n = min(chunk, args.ctx - pos)
    cache.append(torch.randn((U, n, 128), generator=g, device=dev).half(),
                 torch.randn((U, n, 128), generator=g, device=dev).half(), validate=False)
pol = ck.PolicyConfig(exploration_rate=args.explore)
dec = ck.CertifiedDecoder(cache, pol, n_heads=4,
                          scratch=ck.ScratchCache(cache.max_blocks if args.scratch < 0 else args.scratch),
                          rung4_group=np.arange(U) % args.layers)
if args.explore:
    dec.attach_rng(np.random.Generator(np.random.Philox(np.random.SeedSequence((0, 1)))))
tr = torch.empty((32, 2), dtype=torch.int64, device=dev)
names = ["pass_a", "select", "pass_b", "combine", "group_flags", "resolve", "dense", "explore_draw",
         "explore", "lru"]
acc = np.zeros((len(names), 2))
cnt = np.zeros(len(names))
walls = []
for s in range(args.steps + 3):
    tr[:, 0] = np.iinfo(np.int64).max
    tr[:, 1] = 0
    dec.st.trace = _ptr(tr)
    q = torch.randn((U, 4, 128), generator=g, device=dev, dtype=torch.float64)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dec.step_async(q).result()
    b.record()
    torch.cuda.synchronize()
    cache.append(torch.randn((U, 1, 128), generator=g, device=dev).half(),
                 torch.randn((U, 1, 128), generator=g, device=dev).half(), validate=False)
    if s < 3:
        continue
    t = tr.cpu().numpy().astype(np.float64)
    t0 = t[0, 0]
    for i in range(len(names)):
        if t[i, 1] > 0:
            acc[i] += (t[i] - t0) / 1000.0
            cnt[i] += 1
    walls.append(a.elapsed_time(b) * 1000)
print(f"units={U} ctx={args.ctx} flow={'off' if os.environ.get('CKV_NO_FLOW') else 'on'}  "
      f"step (events) {np.mean(walls):.1f} us")
for i, n in enumerate(names):
    if cnt[i]:
        s0, e0 = acc[i] / cnt[i]
        print(f"  {n:14s} start {s0:8.1f}  end {e0:8.1f}  span {e0 - s0:8.1f} us")
