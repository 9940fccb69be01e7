"""Summarise an ncu report: key throughput metrics, stall reasons, and the
hottest source lines (needs -lineinfo + --import-source)."""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_bytes.sum", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(rep, top=25):
    hdr, units, vals = raw(rep)
    v = vals[0]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:60s} {v[i]:>18s} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("stalls per issue:", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
    if top:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if not rows:
            return
        h = rows[0]
        def col(name):
            for j, x in enumerate(h):
                if x.startswith(name):
                    return j
            return None
        isamp = col("Warp Stall Sampling (All Samples)")
        iline = col("#") if col("#") is not None else 0
        isrc = col("Source")
        data = []
        for r in rows[1:]:
            try:
                data.append((float(r[isamp]), r[iline], r[isrc][:110]))
            except (ValueError, IndexError, TypeError):
                pass
        tot = sum(d[0] for d in data) or 1
        for s, ln, src in sorted(data, reverse=True)[:top]:
            print(f"{100*s/tot:5.1f}% L{ln:>5s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
