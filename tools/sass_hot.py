"""Hot SASS lines of one kernel from an ncu report: stall samples, shared-memory excess wavefronts."""
import csv, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
key = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
def num(r, k):
    try:
        return float(r[ix[k]])
    except ValueError:
        return 0.0
tot = sum(num(r, key) for r in data)
print(f"total {key}: {tot}")
for i, r in sorted(enumerate(data), key=lambda x: -num(x[1], key))[:n]:
    extra = " ".join(f"{k.split()[0][:10]}={r[ix[k]]}" for k in ["stall_short_sb", "stall_wait", "stall_long_sb", "L1 Wavefronts Shared Excessive"] if k in ix)
    print(f"{i:5d} {num(r, key):10.0f}  {r[ix['Source']][:70]:70s} {extra}")
