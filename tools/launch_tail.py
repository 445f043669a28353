"""Per-kernel totals of the LAST clustering run in an ncu launch list (tools/one_run.py)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
sc = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}
L = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", "")) * sc[r[ix["Metric Unit"]]]
    L.append((r[ix["Kernel Name"]].split("(")[0].replace("void ", "")[:70], v))
start = [i for i, (n, v) in enumerate(L) if "fill_comp_view" in n][-1]
agg, cnt = collections.defaultdict(float), collections.Counter()
for n, v in L[start:]:
    agg[n] += v
    cnt[n] += 1
print("kernel ms in the last run: %.2f" % sum(agg.values()))
for n, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v:8.2f} {cnt[n]:4d} {n}")
