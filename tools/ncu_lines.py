"""Stall samples per CUDA source line from an ncu report (source page, cuda,sass view)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname = {}, "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 7:
        continue
    if r[2] != "-":  # sass rows carry an address; cuda rows aggregate
        continue
    try:
        v = float(r[4])
    except ValueError:
        continue
    if v > 0:
        agg[(fname, r[0], r[1][:100])] = agg.get((fname, r[0], r[1][:100]), 0) + v
tot = sum(agg.values())
for (f, l, s), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l:>5} {s}")
