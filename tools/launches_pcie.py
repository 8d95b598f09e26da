"""Per-kernel time and PCIe read bytes per step from an ncu launch list taken with
--metrics gpu__time_duration.sum,pcie__read_bytes.sum (the last two steps)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
byid = collections.OrderedDict()
for d in data:
    e = byid.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0]})
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
L = list(byid.values())
idx = [i for i, d in enumerate(L) if "k_pass_a" in d["name"]]
agg = collections.OrderedDict()
for d in L[idx[-2]:]:
    a = agg.setdefault(d["name"], [0.0, 0.0, 0])
    a[0] += d.get("gpu__time_duration.sum", 0.0)
    a[1] += d.get("pcie__read_bytes.sum", 0.0)
    a[2] += 1
tot = sum(v[0] for v in agg.values())
for n, (t, b, c) in agg.items():
    print(f"{n:34s} {c:3d} {t / 2e3:9.1f} us/step {100 * t / tot:5.1f}%  PCIe read {b / 2e6:8.1f} MB/step")
print(f"{'total':34s}     {tot / 2e3:9.1f} us/step")
