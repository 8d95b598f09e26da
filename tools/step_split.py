"""Where the step time goes on the device (CUDA events around the decode call
and the append, default C3 workload; no profiler)."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
import paper_2605_20868_b200 as ck
U, ctx = 256, int(os.environ.get("CTX", "131072"))
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, ctx + 128, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
for pos in range(0, ctx, 4096):
    cache.append(torch.randn((U, 4096, 128), generator=g, device=dev).half(),
                 torch.randn((U, 4096, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4,
                          scratch=ck.ScratchCache(cache.max_blocks))
qs = torch.randn((20, U, 4, 128), generator=g, device=dev, dtype=torch.float64)
kn = torch.randn((20, U, 1, 128), generator=g, device=dev).half()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(20)]
for i in range(20):
    e = ev[i]
    e[0].record()
    dec.q.copy_(qs[i])
    e[1].record()
    dec.launch()
    e[2].record()
    cache.append(kn[i], kn[i], validate=False)
    e[3].record()
    dec.cert_host.copy_(dec.cert_buf, non_blocking=True)
    e[4].record()
torch.cuda.synchronize()
names = ["q copy", "decode", "append", "cert D2H"]
for k in range(4):
    v = sorted(ev[i][k].elapsed_time(ev[i][k + 1]) for i in range(5, 20))
    print(f"{names[k]:10s} median {v[len(v)//2]*1000:8.1f} us")
v = sorted(ev[i][0].elapsed_time(ev[i + 1][0]) for i in range(5, 19))
print(f"{'step':10s} median {v[len(v)//2]*1000:8.1f} us")

# the same decode replayed from a CUDA graph (launch overhead removed)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        dec.launch()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    dec.launch()
torch.cuda.synchronize()
gev = [torch.cuda.Event(enable_timing=True) for _ in range(16)]
for i in range(15):
    dec.q.copy_(qs[i])
    gev[i].record()
    graph.replay()
gev[15].record()
torch.cuda.synchronize()
v = sorted(gev[i].elapsed_time(gev[i + 1]) for i in range(3, 15))
print(f"{'graph':10s} median {v[len(v)//2]*1000:8.1f} us (q copy + replayed decode)")
