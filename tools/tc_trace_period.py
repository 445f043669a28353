"""Steady-state item period (cycles) of CTA 0 per launch from an NNM_TC_TRACE file."""
import sys
cur = None
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        cur = " ".join(line.split()[2:])
        rows = []
        continue
    f = line.split()
    rows.append(int(f[f.index("epi") + 2]))  # epilogue end stamp
    if len(rows) == 256:
        per = (rows[250] - rows[100]) / 150
        print(f"launch items {cur}: {per:.0f} cycles/item")
