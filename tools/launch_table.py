"""ncu launch-list CSV (gpu__time_duration.sum, dram__bytes_read/write.sum per launch) -> the
per-kernel table kept under profiles/, and the DRAM traffic per launch of the scan / re-rank
kernels for profiles/traffic.json (read by bench.py's roofline `traffic`)."""
import csv
import json
import sys


def main(src, dst, key=None, traffic_path=None):
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    k = {}
    order = []
    for r in rows[1:]:
        lid = r[iid]
        if lid not in k:
            k[lid] = {"name": r[ik]}
            order.append(lid)
        k[lid][r[im]] = float(r[iv].replace(",", ""))
    tot = sum(k[i].get("gpu__time_duration.sum", 0) for i in order)
    out = ["kernel                                              us   share   dram_rd_MB   dram_wr_MB"]
    for i in order:
        e = k[i]
        t = e.get("gpu__time_duration.sum", 0) / 1e3
        out.append(f"{e['name'][:46]:46s} {t:9.1f} {100 * t * 1e3 / tot:6.1f}% {e.get('dram__bytes_read.sum', 0) / 1e6:11.1f} {e.get('dram__bytes_write.sum', 0) / 1e6:11.1f}")
    open(dst, "a").write("\n".join(out) + "\n")
    print("\n".join(out))
    if key and traffic_path:
        t = json.load(open(traffic_path))
        ent = {}
        for i in order:
            n = k[i]["name"]
            b = k[i].get("dram__bytes_read.sum", 0) + k[i].get("dram__bytes_write.sum", 0)
            if ("k_pq_scan_rq" in n and ", 0>" in n) or "k_rbq_scan<false>" in n or "k_rbq_mma<0>" in n:
                ent["scan"] = {"dram_bytes": b, "source": dst + " (ncu, one launch)"}
            if n.startswith("void k_rerank") or n.startswith("k_rerank"):
                ent["rerank"] = {"dram_bytes": b, "source": dst + " (ncu, one launch)"}
        t[key] = ent
        json.dump(t, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
