"""Summarise tools/ncu_sweep.sh CSVs: per kernel duration, DRAM bytes vs algorithmic."""
import csv
import glob
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_sw_*.csv"
nz = int(sys.argv[2]) if len(sys.argv) > 2 else 384
npts = 600 * 595 * nz
for f in sorted(glob.glob(pat)):
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r]
    if not hi:
        continue
    rows = rows[hi[0]:]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    per = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        key = (r[0], r[ki][:40])
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if u == "Gbyte":
            v *= 1e9
        elif u == "Mbyte":
            v *= 1e6
        elif u == "Kbyte":
            v *= 1e3
        elif u == "usecond":
            v *= 1e3
        elif u == "msecond":
            v *= 1e6
        per.setdefault(key, {})[r[mi]] = v
    for (lid, kname), m in per.items():
        mode = 1 if ", 1," in kname else 2
        alg = (24 if mode == 1 else 20) * npts
        t = m["gpu__time_duration.sum"] * 1e-9
        tr = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        print(f"{f.split('/')[-1]:32s} H{mode} {t*1e3:7.3f} ms  alg {alg/t/1e12:5.2f} TB/s  "
              f"dram {tr/t/1e12:5.2f} TB/s  traffic/alg {tr/alg:5.3f}  "
              f"l2miss/l2read {m['lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum']/max(1,m['lts__t_sectors_srcunit_tex_op_read.sum']):.3f} "
              f"warps {m['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f}%")
