"""Per-role busy time per item (cycles, CTA 0, items 64..255) for each launch of an
NNM_TC_TRACE file: producer issue gap, MMA issue gap, prep duration, epilogue duration,
epilogue wait for the accumulator."""
import sys

launch = None
rows = []


def report():
    if launch is None or len(rows) < 200:
        return
    import statistics as st
    sel = rows[64:256]
    prep = [r["prep1"] - r["prep0"] for r in sel]
    epi = [r["epi1"] - r["epi0"] for r in sel]
    wait = [r["epi0"] - r["epip"] for r in sel]
    per = (rows[250]["epi1"] - rows[100]["epi1"]) / 150
    print(f"{launch}: period {per:.0f} cyc/item | prep {st.median(prep):.0f} | epilogue {st.median(epi):.0f} "
          f"| epi wait acc {st.median(wait):.0f}")


for line in open(sys.argv[1]):
    if line.startswith("launch"):
        report()
        launch = " ".join(line.split()[1:3])
        rows = []
        continue
    f = line.split()
    g = lambda k, o=1: int(f[f.index(k) + o])  # noqa: E731
    rows.append({"prod": g("prod"), "mma": g("mma"), "prep0": g("prep"), "prep1": g("prep", 2),
                 "epip": g("epi_prepped"), "epi0": g("epi"), "epi1": g("epi", 2)})
report()
