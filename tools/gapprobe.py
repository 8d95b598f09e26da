"""Where the non-kernel time of a small step goes (kv1 proxy: 32 units x 128K):
times K steps of (a) the bench loop (step_async + append), (b) launch only (no
certificate copies), (c) decode launches only, (d) pass A alone is not separable:
reports ms/step for each variant."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2605_20868_b200 as ck
U = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = 131072
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, N + 512)
g = torch.Generator(device=dev).manual_seed(0)
for pos in range(0, N, 8192):
    cache.append(torch.randn((U, 8192, 128), generator=g, device=dev).half(),
                 torch.randn((U, 8192, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4,
                          rung4_group=np.arange(U) % 4)
q = torch.randn((U, 4, 128), generator=g, device=dev, dtype=torch.float64)
kn = torch.randn((U, 1, 128), generator=g, device=dev).half()
K = 50

def timeit(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K

def full():
    p = dec.step_async(q)
    cache.append(kn, kn, validate=False)

def launch_append():
    dec.launch(q)
    cache.append(kn, kn, validate=False)

def launch_only():
    dec.launch(q)

def launch_noq():
    dec.launch(None)

print(f"U={U}")
for name, fn in (("bench loop (step_async + append)", full), ("launch + append", launch_append),
                 ("launch (with q copy)", launch_only), ("launch (no q copy)", launch_noq)):
    print(f"{name:36s} {timeit(fn) * 1000:8.1f} us/step")
