"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel time per step."""
import csv, collections, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
idx = [i for i, d in enumerate(data) if "k_pass_a" in d["Kernel Name"]]
nsteps = len(idx[-2:])
agg = collections.OrderedDict()
for d in data[idx[-2]:]:
    n = d["Kernel Name"].split("(")[0]
    agg.setdefault(n, [0.0, 0])
    agg[n][0] += float(d["Metric Value"])
    agg[n][1] += 1
tot = sum(v[0] for v in agg.values())
for n, (v, c) in agg.items():
    print(f"{n:34s} {c:3d} {v / nsteps / 1e3:9.1f} us/step {100 * v / tot:5.1f}%")
print(f"{'total':34s}     {tot / nsteps / 1e3:9.1f} us/step")
