"""Summary of an ncu --set full capture of tc_scan_kernel launches (raw page CSV on stdin
or as argv[1]): duration, DRAM bytes, issue activity, occupancy, pipes, top stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin))
h, units = rows[0], rows[1]
ix = {k: i for i, k in enumerate(h)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]
for n, r in enumerate(rows[2:]):
    print(f"--- launch {n}: {r[ix['Kernel Name']][:60]}")
    for k in want:
        if k in ix:
            print(f"{k:70s} {r[ix[k]]:>14s} {units[ix[k]]}")
    st = {}
    for k, i in ix.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
    print("stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
