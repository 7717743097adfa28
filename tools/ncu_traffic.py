"""Reduce full-size `ncu --set full` captures (raw-page CSVs from tools/profile_r2.sh) to
profiles/<tag>_traffic.json: per kernel launch, device time, DRAM bytes read / written and the
kernel's algorithmic bytes (SURVEY 8(d) passes x element size x points).
Usage: python tools/ncu_traffic.py <tag> <raw.csv>... """
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NPTS3 = 600 * 595 * 1536
NPTS2 = 22800 * 22800
# kernel-name prefix -> (passes, element bytes, points)
ALGO = [
    # the constant-coefficient (scalar-coupling, CC = last template argument 1) classic kernels: 6 / 4 passes
    ("k_stencil<__half, 1, 16, 2, 2, 0, 0, 1>", 6, 2, NPTS3), ("k_stencil<__half, 2, 16, 2, 2, 0, 0, 1>", 4, 2, NPTS3),
    ("k_stencil<float, 1, 16, 2, 2, 0, 0, 1>", 6, 4, NPTS3), ("k_stencil<float, 2, 16, 2, 2, 0, 0, 1>", 4, 4, NPTS3),
    ("k_h3s_half<", 7, 2, NPTS3),
    ("k_stencil<__half, 1,", 12, 2, NPTS3), ("k_stencil<__half, 2,", 10, 2, NPTS3),
    ("k_stencil<float, 1,", 12, 4, NPTS3), ("k_stencil<float, 2,", 10, 4, NPTS3),
    ("k_h3_bulk<float", 7, 4, NPTS3),
    ("k_h3_bulk<__half", 7, 2, NPTS3), ("k_h3<__half", 7, 2, NPTS3),
    ("k_sr<__half, 16, 2, 2, 0", 19, 2, NPTS3), ("k_sr<__half, 8, 3, 2, 1", 13, 2, NPTS3),
    ("k_sr<float", 19, 4, NPTS3),
    ("k_bicg9<__half, 1,", 14, 2, NPTS2), ("k_bicg9<__half, 2,", 12, 2, NPTS2),
    ("k_apply9<__half, 32, 0", 10, 2, NPTS2), ("k_apply9<__half, 32, 1", 10, 2, NPTS2),
]


def algo(name):
    n = name.replace("void ", "")
    for pre, passes, es, npts in ALGO:
        if n.startswith(pre):
            return passes * es * npts, passes
    return None, None


def main(tag, files):
    out = {"source": "ncu --set full --clock-control none, full-size launches (tools/profile_r2.sh, "
                     "tools/profile_cc.sh)", "kernels": {}}
    for fn in files:
        rows = list(csv.reader(open(fn)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        ix = {h: i for i, h in enumerate(hdr)}
        for r in data:
            name = r[ix["Kernel Name"]]
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            rd = float(r[ix["dram__bytes_read.sum"]]) * scale[units[ix["dram__bytes_read.sum"]]]
            wr = float(r[ix["dram__bytes_write.sum"]]) * scale[units[ix["dram__bytes_write.sum"]]]
            tu = units[ix["gpu__time_duration.sum"]]
            t_ms = float(r[ix["gpu__time_duration.sum"]]) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}[tu]
            ab, passes = algo(name)
            rec = {"capture": os.path.basename(fn), "time_ms": t_ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
                   "traffic_bytes": rd + wr, "algorithmic_bytes": ab, "passes": passes,
                   "traffic_over_algorithmic": (rd + wr) / ab if ab else None,
                   "dram_tbs": (rd + wr) / (t_ms * 1e-3) / 1e12,
                   "algorithmic_tbs": ab / (t_ms * 1e-3) / 1e12 if ab else None}
            out["kernels"].setdefault(name.replace("void ", "").split("(")[0], []).append(rec)
    path = os.path.join(ROOT, "profiles", f"{tag}_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    for k, v in out["kernels"].items():
        for x in v:
            print(f"{k:40s} {x['time_ms']:.4f} ms  traffic/algo {x['traffic_over_algorithmic']}  "
                  f"{x['algorithmic_tbs']} TB/s algo")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
