"""Per-opcode executed-instruction mix of one kernel from an ncu report (source page, SASS)."""
import csv, collections, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
ops = collections.Counter()
for r in rows[2:]:
    if len(r) <= i_ex:
        continue
    try:
        n = int(r[i_ex])
    except ValueError:
        continue
    toks = r[i_src].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += n
tot = sum(ops.values())
for op, n in ops.most_common(25):
    print(f"{op:10s} {n / norm:10.1f} {100 * n / tot:5.1f}%")
print("total", tot / norm)
