"""Blackwell features in the built library's SASS, per kernel: bulk copies (UBLKCP,
cp.async.bulk), L2 bulk prefetch (UBLKPF), mbarrier ops (SYNCS), tensor-core MMAs
(IMMA / HMMA), programmatic-dependent-launch waits (ACQBULK = griddepcontrol.wait),
elect.sync (ELECT).  python tools/sass_features.py [lib.so]"""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2605_20868_b200", "libcertkv_b200.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UBLKCP", "UBLKPF", "SYNCS", "IMMA", "HMMA", "ACQBULK", "ELECT", "REDUX"]
print(f"{'kernel':44s} {'SASS':>6s} " + " ".join(f"{k:>7s}" for k in KEYS))
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    c = collections.Counter(m.group(2) for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f))
    dm = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    dm = re.sub(r"\(.*\)$", "", dm).replace("ckv::", "") or name
    print(f"{dm[:44]:44s} {sum(c.values()):6d} " + " ".join(f"{c[k]:7d}" for k in KEYS))
