"""Per-config DRAM traffic of the dominant scan kernel from ncu launch lists.

usage: python tools/traffic_from_launches.py out.json cfg=path.csv [cfg=path.csv ...]
Each CSV is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` over one device step (tools/launches.sh).  Writes, per config, the dominant kernel
(largest total time among the scan kernels), its launch count, average duration and average
DRAM bytes (read + write) per launch."""
import collections
import csv
import json
import sys

SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
           "s": 1e3, "second": 1e3}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}
SCANS = ("tc_scan_kernel", "scan_reg_kernel", "scan_ws_kernel", "scan_rows_kernel", "collect_kernel",
         "small_screened_kernel", "small_boruvka_kernel")


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        lid = r[ix["ID"]]
        names[lid] = r[ix["Kernel Name"]]
        m, u = r[ix["Metric Name"]], r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        per[lid][m] = v * (SCALE_T.get(u) if m == "gpu__time_duration.sum" else SCALE_B.get(u, 1.0))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, mets in per.items():
        k = next((s for s in SCANS if s in names[lid]), None)
        if k is None:
            continue
        a = agg[k]
        a[0] += 1
        a[1] += mets.get("gpu__time_duration.sum", 0.0)
        a[2] += mets.get("dram__bytes_read.sum", 0.0) + mets.get("dram__bytes_write.sum", 0.0)
    k, (cnt, ms, b) = max(agg.items(), key=lambda kv: kv[1][1])
    return {"kernel": k, "launches": cnt, "avg_launch_ms": ms / cnt,
            "dram_bytes_per_launch": b / cnt, "source": path}


out = {}
for arg in sys.argv[2:]:
    cfg, path = arg.split("=", 1)
    out[cfg] = summarize(path)
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
