"""Summarise `ncu --set full` raw-page CSVs (tools/profile_r2.sh) as a markdown table of the metrics
that explain a bandwidth-bound kernel.  Usage: python tools/ncu_full_md.py <out.md> <title> <raw.csv>..."""
import csv
import sys

M = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
     "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def main(out, title, files):
    cols, units = [], {}
    for fn in files:
        rows = list(csv.reader(open(fn)))
        hdr, un, data = rows[0], rows[1], rows[2:]
        ix = {h: i for i, h in enumerate(hdr)}
        for r in data:
            name = r[ix["Kernel Name"]].replace("void ", "").split("(")[0].replace("sten::", "")
            cols.append((name, {m: r[ix[m]] if m in ix else "" for m in M}))
            for m in M:
                if m in ix:
                    units[m] = un[ix[m]]
    L = [f"# {title}\n", "| metric | unit | " + " | ".join(c[0] for c in cols) + " |",
         "|---|---|" + "---|" * len(cols)]
    for m in M:
        L.append(f"| {m} | {units.get(m, '')} | " + " | ".join(c[1][m] for c in cols) + " |")
    open(out, "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
