"""Summarise an ncu report: SOL, pipes, scheduler, stalls, top instructions."""
import csv, io, subprocess, sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "No Eligible", "Dynamic Shared Memory Per Block")
drows = list(csv.reader(io.StringIO(det)))
if drows:
    dh = drows[0]
    if "Metric Name" in dh:
        mi, ui, vi = dh.index("Metric Name"), dh.index("Metric Unit"), dh.index("Metric Value")
        for row in drows[1:]:
            if len(row) > vi and row[mi] in want:
                print(f"{row[mi]:40s} {row[vi]:>14s} {row[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    hdr, vals = rows[0], rows[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum",
              "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active"):
        if k in hdr:
            print(f"{k:70s} {vals[hdr.index(k)]} {rows[1][hdr.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]; ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
sc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: sum(f(r, h) for r in data) for h in sc}; s = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{h[6:]} {v/s*100:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{int(f(r,'Warp Stall Sampling (All Samples)')):8d}  {r[ix['Source']][:80]}")
ex = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data); tw = sum(f(r, "L1 Wavefronts Shared") for r in data)
print(f"shared wavefronts excessive {ex:.3g} of {tw:.3g}")
