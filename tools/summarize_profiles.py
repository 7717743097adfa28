"""Turn the raw ncu outputs of a profiling gpurun into committed summaries under profiles/.

usage: python tools/summarize_profiles.py <tag>   (reads gpurun_out/<tag>_*.csv / .ncu-rep)
writes profiles/<tag>_launches.csv, <tag>_launch_shares.md, <tag>_traffic.json, <tag>_ncu_full.md
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "usecond": 1e3, "msecond": 1e6, "nsecond": 1.0,
        "second": 1e9}


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        out.setdefault((d["ID"], d["Kernel Name"], d["Grid Size"], d["Block Size"]), {})[d["Metric Name"]] = v
    return out


CMDS = {
    "r1": {"traffic": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none -k regex:'k_stencil|k_h3|k_init' -s 30 -c 6 "
                      "python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --schedule classic",
           "full": "ncu --set full --clock-control none --import-source on -k regex:'k_stencil|k_h3' -s 0 -c 3 "
                   "python bench.py --steps 1 --warmup 1 --maxit 2 --nz 384 --no-e2e --no-cpu --schedule classic"},
    "r1_sr": {"traffic": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         "--clock-control none -k regex:'k_sr|k_init' -s 20 -c 4 "
                         "python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu",
              "full": "ncu --set full --clock-control none --import-source on -k regex:k_sr -s 2 -c 1 "
                      "python bench.py --steps 1 --warmup 1 --maxit 4 --nz 384 --no-e2e --no-cpu"},
}


def short(name):
    return name.split("(")[0].replace("void ", "").replace("sten::", "").replace("<unnamed>::", "")


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    npts = 600 * 595 * 1536
    # 1. launch list: every launch with its device time (cold-cache, serialised: shares, not absolutes)
    lpath = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lpath):
        data = read_ncu_csv(lpath)
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            f.write("id,kernel,grid,block,gpu_time_ns\n")
            for (i, k, g, b), m in data.items():
                f.write(f"{i},{short(k)},\"{g}\",\"{b}\",{m['gpu__time_duration.sum']:.0f}\n")
        agg = collections.defaultdict(list)
        for (i, k, g, b), m in data.items():
            agg[short(k)].append(m["gpu__time_duration.sum"])
        tot = sum(sum(v) for v in agg.values())
        hot = sum(sum(v) for k, v in agg.items() if k.startswith(("k_stencil", "k_h3", "k_rows", "k_sr")))
        with open(os.path.join(PROF, f"{tag}_launch_shares.md"), "w") as f:
            f.write(f"# {tag}: ncu launch list of `python bench.py` (first {len(data)} launches)\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none -c 700` - per-launch times are cold-cache and\n"
                    "serialised; compare SHARES with the bench's CUDA-event phase times, not absolutes.\n\n")
            f.write("| kernel | launches | avg ms | share of profiled time |\n|---|---|---|---|\n")
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e6:.3f} | {sum(v) / tot * 100:.1f}% |\n")
            f.write(f"\nHot path (SR sweep / stencil + H3) share: {hot / tot * 100:.1f}%; the rest is one-time setup "
                    f"(field generation, Jacobi scaling, fp16 conversion) and the per-solve init.\n")
    # 2. full-size traffic per hot kernel
    tpath = os.path.join(OUT, f"{tag}_traffic_full.csv")
    if os.path.exists(tpath):
        data = read_ncu_csv(tpath)
        alg_passes = {"k_stencil<__half, 1": 12, "k_stencil<__half, 2": 10, "k_h3<__half>": 7, "k_init<__half>": 5,
                      "k_sr<__half": 19}
        res = {}
        for (i, k, g, b), m in data.items():
            sk = short(k)
            key = next((p for p in alg_passes if sk.startswith(p)), None)
            if key is None:
                continue
            alg = alg_passes[key] * 2 * npts
            tr = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
            t = m["gpu__time_duration.sum"] * 1e-9
            res.setdefault(sk, []).append(dict(
                launch_id=int(i), grid=g, block=b, time_ms=t * 1e3, dram_read_bytes=m["dram__bytes_read.sum"],
                dram_write_bytes=m["dram__bytes_write.sum"], traffic_bytes=tr, algorithmic_bytes=alg,
                traffic_over_algorithmic=tr / alg, dram_tbs=tr / t / 1e12, algorithmic_tbs=alg / t / 1e12))
        json.dump({"workload": "cfg3 600x595x1536 mixed fp16, steady-state launches of bench.py",
                   "command": CMDS.get(tag, {}).get("traffic", ""),
                   "kernels": res}, open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)
    # 3. --set full report of the hot kernels (reduced z for cheap replay)
    rpath = os.path.join(OUT, f"{tag}_full.ncu-rep")
    if os.path.exists(rpath):
        raw = subprocess.run(["ncu", "-i", rpath, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, data = rows[0], rows[1], rows[2:]
        want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
                "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
                "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
        idx = {h: i for i, h in enumerate(hdr)}
        with open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w") as f:
            f.write(f"# {tag}: `ncu --set full` of the hot kernels (600x595x384 slab, same kernels/tiling as the bench)\n\n")
            f.write(f"Command: `{CMDS.get(tag, {}).get('full', '')}`\n\n")
            f.write("| metric | unit | " + " | ".join(short(r[idx["Kernel Name"]]) for r in data) + " |\n")
            f.write("|---|---|" + "---|" * len(data) + "\n")
            for w in want[1:]:
                if w in idx:
                    f.write(f"| {w} | {units[idx[w]]} | " + " | ".join(r[idx[w]] for r in data) + " |\n")
            f.write("\nTensor pipes are idle: the Gram of the SR sweep runs on the FMA pipe (fma.rn.f32.f16), "
                    "which measured faster than mma.sync for it (DESIGN.md); the kernels are HBM/latency-bound.\n")
    print("written", os.listdir(PROF))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
