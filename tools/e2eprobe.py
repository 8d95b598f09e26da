"""Where does the e2e loop's extra device time go?  The same decoder and inputs run
60-step loops that add, one at a time, the e2e loop's mechanics: events after the
step, cross-stream waits before it, copies on a second stream.  Prints the device
step interval of each (CUDA events on the step stream).  python tools/e2eprobe.py [kv_heads]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_20868_b200 as ck
kvh = int(sys.argv[1]) if len(sys.argv) > 1 else 8
U, ctx, E = 32 * kvh, 131072, 60
dev = torch.device("cuda")
cache = ck.DeviceKVCache(U, ctx + 8 * E + 64, device=dev)
g = torch.Generator(device=dev).manual_seed(1000)
chunk = max(16, min(4096, (1 << 22) // U))
for pos in range(0, ctx, chunk):
    cache.append(torch.randn((U, chunk, 128), generator=g, device=dev).half(),
                 torch.randn((U, chunk, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4,
                          scratch=ck.ScratchCache(cache.max_blocks), rung4_group=np.arange(U) % 32)
qd = [torch.randn((U, 4, 128), generator=g, device=dev, dtype=torch.float64) for _ in range(8)]
kd = [torch.randn((U, 1, 128), generator=g, device=dev).half() for _ in range(8)]
od = [torch.empty((U, 4, 128), device=dev) for _ in range(2)]
qh = [q.cpu().pin_memory() for q in qd]
oh = torch.empty((U, 4, 128)).pin_memory()
comp = torch.cuda.current_stream(dev)
cs = torch.cuda.Stream(device=dev)
for i in range(5):
    dec.step(qd[i])


def run(mode):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(E)]
    ext = [torch.cuda.Event() for _ in range(2)]
    for e in ext:
        e.record(cs)
    torch.cuda.synchronize()
    prev = None
    for i in range(E):
        b = i % 2
        if mode >= 2:
            comp.wait_event(ext[b])
        out = od[b] if mode >= 1 else None
        p = dec.step_async(qd[i % 8], out=out)
        if mode >= 1:
            evs[i].record(comp)
        cache.append(kd[i % 8], kd[i % 8], validate=False)
        if mode == 0:
            evs[i].record(comp)
        if mode >= 3:
            with torch.cuda.stream(cs):
                cs.wait_event(evs[i])
                oh.copy_(od[b], non_blocking=True)
                if mode >= 4:
                    qd[(i + 1) % 8].copy_(qh[(i + 1) % 8], non_blocking=True)
                ext[b].record(cs)
        if prev is not None:
            prev.result()
        prev = p
    torch.cuda.synchronize()
    prev.result()
    return evs[0].elapsed_time(evs[E - 1]) / (E - 1)


names = ["plain", "+event after step, out=", "+cross-stream wait before", "+D2H on a 2nd stream",
         "+H2D on the 2nd stream", "plain again"]
for m in (0, 1, 2, 3, 4, 0):
    print(f"{names[m] if m or names[0] else ''}: {run(m):.4f} ms/step")
