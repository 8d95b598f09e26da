"""Per-phase cycle profile of k_select (clock64 deltas, thread 0 of every CTA):
builds a -DCKV_SELPROF variant of the library and runs C3-shaped steps."""
import ctypes, os, subprocess, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_20868_b200 import build, _lib
out = os.path.join(ROOT, "paper_2605_20868_b200", "libcertkv_b200_prof.so")
cmd = ["nvcc", *build.NVCC_FLAGS, "-shared", "-DCKV_SELPROF", "-I", os.path.join(ROOT, "include"), *build.sources(), "-o", out]
subprocess.run(cmd, check=True)
_lib.LIB_PATH = out
import paper_2605_20868_b200 as ck
units, ctx = int(os.environ.get("UNITS", "256")), int(os.environ.get("CTX", "131072"))
dev = torch.device("cuda")
cache = ck.DeviceKVCache(units, ctx + 64, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
for pos in range(0, ctx, 4096):
    cache.append(torch.randn((units, 4096, 128), generator=g, device=dev).half(),
                 torch.randn((units, 4096, 128), generator=g, device=dev).half(), validate=False)
dec = ck.CertifiedDecoder(cache, ck.PolicyConfig(exploration_rate=0.0), n_heads=4)
for i in range(3):
    dec.step(torch.randn((units, 4, 128), generator=g, device=dev, dtype=torch.float64))
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16)()
lib.ckv_debug_selprof(buf)
n = units * 4 * 3
names = {1: "keys+init", 2: "partial", 3: "split-merge", 4: "lse", 8: "radix", 10: "gather", 5: "rank sort", 6: "coverage+order",
         7: "tail/rung2/cert", 9: "union (last CTA)"}
for i, nm in names.items():
    print(f"{nm:18s} {buf[i] / n / 1000:8.2f} us/CTA")
