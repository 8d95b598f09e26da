"""Is the bench's step loop host-bound?  Times the host side of each call of the
bench's one_step (step_async, append, collect) against the device time per step.
python tools/hostprobe.py [kv_heads] [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_20868_b200 as ck
kvh = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
U, ctx = 32 * kvh, 131072
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, ctx + K + 64, device=dev)
g = torch.Generator(device=dev).manual_seed(1000)
chunk = max(16, min(4096, (1 << 22) // U))
for pos in range(0, ctx, chunk):
    cache.append(torch.randn((U, chunk, 128), generator=g, device=dev).half(),
                 torch.randn((U, chunk, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4,
                          scratch=ck.ScratchCache(cache.max_blocks), rung4_group=np.arange(U) % 32)
qpool = torch.randn((K, U, 4, 128), generator=g, device=dev, dtype=torch.float64)
kpool = torch.randn((K, U, 1, 128), generator=g, device=dev).half()
vpool = torch.randn((K, U, 1, 128), generator=g, device=dev).half()
for i in range(5):  # warm-up: first launches load the kernels
    dec.step_async(qpool[i]).result()
for mode in ("full", "no_append", "launch_only"):
    t = {"step": 0.0, "append": 0.0, "collect": 0.0}
    pend = None
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    for i in range(K):
        t0 = time.perf_counter()
        p = dec.step_async(qpool[i])
        t1 = time.perf_counter()
        if mode == "full":
            cache.append(kpool[i], vpool[i], validate=False)
        t2 = time.perf_counter()
        if pend is not None and mode != "launch_only":
            pend.result()
        t3 = time.perf_counter()
        pend = p
        t["step"] += t1 - t0
        t["append"] += t2 - t1
        t["collect"] += t3 - t2
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / K * 1e3
    print(f"{mode:12s} device {a.elapsed_time(b) / K:.4f} ms/step  wall {wall:.4f}  host: "
          + "  ".join(f"{k} {v / K * 1e3:.4f}" for k, v in t.items()))
    if pend is not None:
        pend.result()
