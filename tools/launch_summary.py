"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum CSV) -> summary CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
agg, cnt = {}, collections.Counter()
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "second": 1e3}
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.split("(")[0]
    depth, out = 0, ""
    for ch in name:
        if ch == "<":
            if depth == 0:
                out += "<...>"
            depth += 1
        elif ch == ">":
            depth -= 1
        elif depth == 0:
            out += ch
    short = out.replace("void ", "")
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1e-6)
    agg[short] = agg.get(short, 0) + v
    cnt[short] += 1
tot = sum(agg.values())
with open(sys.argv[2], "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none --profile-from-start off over tools/profile_step.py <config>: ONE "
            "device step after a warm-up step (cold-cache, serialised; compare shares)\n")
    f.write("kernel, launches, total_ms, share\n")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        f.write(f"{k}, {cnt[k]}, {v:.2f}, {100 * v / tot:.1f}%\n")
