"""Summarise an ncu --set full report (raw CSV page) into the per-kernel lines kept under
profiles/: duration, issue, occupancy, L1/shared pipe, DRAM bytes, top stall reasons."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "us", 1e3),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "lsu_pipe%", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe%", 1),
    ("dram__bytes_read.sum", "dram_rd", 1),
    ("dram__bytes_write.sum", "dram_wr", 1),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("lts__t_sector_hit_rate.pct", "l2hit%", 1),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor%", 1),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        print("## " + name[:90])
        for k, lab, sc in KEYS:
            if k in ix and r[ix[k]] not in ("", "n/a"):
                u = units[ix[k]]
                v = r[ix[k]].replace(",", "")
                try:
                    v = float(v)
                    if k == "gpu__time_duration.sum":
                        v = v * (1e3 if u == "ms" else 1e-3 if u == "ns" else 1)
                        u = "us"
                    print(f"  {lab:12s} {v:14.3f} {u}")
                except ValueError:
                    print(f"  {lab:12s} {v}")
        st = []
        for h, i in ix.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  stalls/issue " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
