"""Summarise ncu outputs: launch-list shares (csv) and key raw metrics of a --set full report."""
import collections
import csv
import subprocess
import sys


def launches(path, steps=5):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi and r[ni] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0].replace("void ", "")[:48]].append(float(r[mi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k:48s} n={len(v):4d} avg={sum(v) / len(v) / 1e3:8.2f} us  share={sum(v) / tot:.3f}")
    out.append(f"total kernel time per step: {tot / steps / 1e3:.1f} us (ncu, serialised, cold)")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "lts__t_bytes.sum", "pcie__read_bytes.sum", "pcie__write_bytes.sum",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum"]


def full(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    units = rows[1]
    idx = {w: h.index(w) for w in WANT if w in h}
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        out.append(name)
        for w, i in idx.items():
            out.append(f"    {w:62s} {r[i]:>14s} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(launches(p) if p.endswith(".csv") else full(p))
