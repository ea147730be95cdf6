"""Per-step DRAM traffic and time of each kernel from an ncu launch list of
`bench.py --profile-steps --steps K --warmup 0` (exactly K timed searches captured):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv python bench.py --profile-steps ...
    python tools/traffic_from_ncu.py launches.csv --steps K --key C4/1024/75000 [--update]

Every launch of a kernel is summed (sample passes and every micro-batch), then divided by K.
Kernels are grouped into the bench's roofline names: "scan" = the main PQ scan pass
(k_pq_scan_rq<M, false, ...>, k_pq4_scan<M, false>) or the RaBitQ Push GEMM
(k_rbq_mma_ws<false>); "rerank" = k_rerank / k_rerank_seg.  --update writes them into
profiles/traffic.json under the key.
"""
import argparse
import csv
import json
import os
import re
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def group(name: str):
    if re.match(r"void bbc::k_pq_scan_rq<\d+, (0|false)", name) or re.match(r"void bbc::k_pq4_scan<\d+, (0|false)", name) \
            or re.match(r"void bbc::k_rbq_mma_ws<(0|false)>", name):
        return "scan"
    if name.startswith("void bbc::k_rerank"):
        return "rerank"
    return None


def parse(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    per = defaultdict(dict)
    for r in rd:
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        try:
            x = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
        per[key][r["Metric Name"]] = x * scale
    for (i, name), m in per.items():
        rows.append((int(i), name, m))
    rows.sort()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--key", required=True, help="workload/nprobe/budget")
    ap.add_argument("--update", action="store_true")
    a = ap.parse_args()
    rows = parse(a.csv)
    tot = defaultdict(lambda: {"dram": 0.0, "time": 0.0, "n": 0})
    allk = defaultdict(lambda: {"dram": 0.0, "time": 0.0, "n": 0})
    for _, name, m in rows:
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        short = name.split("(")[0]
        allk[short]["dram"] += dram
        allk[short]["time"] += t
        allk[short]["n"] += 1
        g = group(name)
        if g:
            tot[g]["dram"] += dram
            tot[g]["time"] += t
            tot[g]["n"] += 1
    T = sum(v["time"] for v in allk.values())
    print(f"{'kernel':90s} {'launch/step':>11s} {'ms/step':>9s} {'share':>6s} {'DRAM GB/step':>12s}")
    for k_, v in sorted(allk.items(), key=lambda kv: -kv[1]["time"]):
        print(f"{k_[:90]:90s} {v['n'] / a.steps:11.1f} {1e3 * v['time'] / a.steps:9.3f} "
              f"{v['time'] / T:6.1%} {v['dram'] / a.steps / 1e9:12.3f}")
    out = {g: {"dram_bytes_per_step": v["dram"] / a.steps, "launches": v["n"] // a.steps,
               "ncu_ms_per_step": 1e3 * v["time"] / a.steps, "ncu_share": v["time"] / T,
               "source": f"profiles/{os.path.basename(a.csv)} (ncu launch list, {a.steps} step(s), "
                         f"every launch summed)"} for g, v in tot.items()}
    print(json.dumps(out, indent=1))
    if a.update:
        p = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(p)) if os.path.exists(p) else {}
        t[a.key] = out
        json.dump(t, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
