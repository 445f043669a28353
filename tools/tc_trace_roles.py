"""Per-role timing of NNM_TC_TRACE launches (CTA 0, items 60..240): prep (per prep warp),
epilogue group 0 (items q % 3 == 0), MMA issue gaps and the steady-state period."""
import statistics as st
import sys

G_EPI, G_PREP = 3, 2
launch, rows = None, []


def report():
    if launch is None or len(rows) < 250:
        return
    R = rows
    eq = [q for q in range(60, 240) if q % G_EPI == 0]
    mean = lambda xs: st.mean(xs) if xs else 0.0  # noqa: E731
    period = (R[eq[-1]]["epi1"] - R[eq[0]]["epi1"]) / (eq[-1] - eq[0])
    prep = mean([R[q]["prep1"] - R[q]["prep0"] for q in range(60, 240)])
    prep_idle = mean([R[q + G_PREP]["prep0"] - R[q]["prep1"] for q in range(60, 240)])
    epi_work = mean([R[q]["epi1"] - R[q]["epi0"] for q in eq])
    epi_wait_prep = mean([R[q]["epip"] - R[q]["es"] for q in eq])
    epi_wait_acc = mean([R[q]["epi0"] - R[q]["epip"] for q in eq])
    epi_gap = mean([R[q + G_EPI]["es"] - R[q]["epi1"] for q in eq])
    mma_gap = mean([R[q + 1]["mma"] - R[q]["mma"] for q in range(60, 240)])
    mma_after_prep = mean([R[q]["mma"] - R[q]["prep1"] for q in range(60, 240)])
    print(f"{launch}: period {period:.0f} | prep {prep:.0f} idle {prep_idle:.0f} | epi work {epi_work:.0f} "
          f"wait-prep {epi_wait_prep:.0f} wait-acc {epi_wait_acc:.0f} gap {epi_gap:.0f} | "
          f"mma gap {mma_gap:.0f} mma-after-prep {mma_after_prep:.0f}")


for line in open(sys.argv[1]):
    if line.startswith("launch"):
        report()
        launch = " ".join(line.split()[1:3])
        rows = []
        continue
    f = line.split()
    g = lambda k, o=1: int(f[f.index(k) + o])  # noqa: E731
    rows.append({"prod": g("prod"), "mma": g("mma"), "prep0": g("prep"), "prep1": g("prep", 2),
                 "epip": g("epi_prepped"), "epi0": g("epi"), "epi1": g("epi", 2), "es": g("tail")})
report()
