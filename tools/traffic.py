"""ncu DRAM traffic per launch of the step kernels, per bench configuration.

Runs bench.py under ncu (metrics only, --clock-control none) for each
configuration and writes profiles/traffic_r02.json keyed like bench.py's lookup
("config:ctx:batch:tier2:units").  Usage (on the GPU box):

    python tools/traffic.py c3 c2 c5 c4 c3host
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KERNELS = ("k_pass_a", "k_pass_b", "k_select", "k_dense", "k_combine", "k_lru", "k_lru_fast")
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def run(cfg, parse_only=False):
    import bench
    pre = bench.PRESETS[cfg]
    units = 32 * 8 * pre["batch"]
    out = os.path.join(ROOT, "gpurun_out", f"traffic_{cfg}.csv")
    if parse_only:
        return parse(cfg, pre, units, out)
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--log-file", out,
           "-k", "regex:^(" + "|".join(KERNELS) + ")$", "-s", "40", "-c", "20",
           sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "6",
           "--warmup", "8", "--no-cpu-baseline", "--no-e2e"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return parse(cfg, pre, units, out)


def parse(cfg, pre, units, out):
    text = open(out).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = {}
    for r in rows:
        k = r["Kernel Name"].replace("void ", "").split("(")[0].split("<")[0].strip()
        d = per.setdefault(k, {})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[unit]
        d.setdefault(r["Metric Name"], []).append(v * scale)
    res = {}
    for k, d in per.items():
        n = len(d.get("gpu__time_duration.sum", [])) or 1
        rd = sum(d.get("dram__bytes_read.sum", [])) / n
        wr = sum(d.get("dram__bytes_write.sum", [])) / n
        res[k] = {"dram_read_per_launch": rd, "dram_write_per_launch": wr,
                  "dram_bytes_per_launch": rd + wr,
                  "time_s_per_launch": sum(d.get("gpu__time_duration.sum", [])) / n,
                  "launches": n}
    key = f"{cfg}:{pre['ctx']}:{pre['batch']}:{pre['tier2']}:{units}"
    return key, res


if __name__ == "__main__":
    base = os.path.join(ROOT, "profiles", "traffic_r02.json")
    table = json.load(open(base)) if os.path.exists(base) else {}
    path = os.path.join(ROOT, "gpurun_out", "traffic_r02.json")  # copied into profiles/
    parse_only = "--parse" in sys.argv
    for cfg in [a for a in sys.argv[1:] if not a.startswith("--")]:
        key, res = run(cfg, parse_only)
        res["source"] = ("ncu --metrics " + METRICS + " --clock-control none, bench.py --config "
                         f"{cfg} --steps 6 --warmup 8 (launches after the warm-up)")
        table[key] = res
        print(key, json.dumps(res.get("k_pass_a")))
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)
