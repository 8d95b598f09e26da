"""Same-box A/B of prebuilt library variants, interleaved (A B A B ...):
python tools/ab.py "<bench args>" rounds lib1.so lib2.so ...
Prints per variant the median ms/step, pass-A ms and step - pass A."""
import json, os, shutil, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_20868_b200", "libcertkv_b200.so")
args, rounds, libs = sys.argv[1].split(), int(sys.argv[2]), sys.argv[3:]
res = {l: [] for l in libs}
for r in range(rounds):
    for l in libs:
        shutil.copy(l, LIB)
        os.utime(LIB)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline",
                              "--no-e2e", "--no-variant", *args], capture_output=True, text=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        res[l].append((d["ms_per_step"], d["roofline"]["pass_a_ms"]))
for l, v in res.items():
    ms = statistics.median(x[0] for x in v)
    pa = statistics.median(x[1] for x in v)
    print(f"{os.path.basename(l):28s} {' '.join(args):24s} step {ms:.4f}  passA {pa:.4f}  tail {ms - pa:.4f}  "
          f"all {[round(x[0], 4) for x in v]}")
