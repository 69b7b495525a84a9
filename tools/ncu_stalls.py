"""Dev: per-kernel duration, DRAM, issue and top warp-stall reasons from a .ncu-rep."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
def g(r, k):
    try: return float(r[hdr.index(k)].replace(",", ""))
    except Exception: return None
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:60]
    dur = g(r, "gpu__time_duration.sum")
    print(f"== {name}  dur {dur/1e3:.1f} us  dramR {g(r,'dram__bytes_read.sum')/1e6:.0f} MB  dramW {g(r,'dram__bytes_write.sum')/1e6:.0f} MB  "
          f"dram% {g(r,'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}  issue% {g(r,'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}")
    st = []
    for i, k in enumerate(hdr):
        if k.startswith("smsp__average_warp_latency_issue_stalled_") or k.startswith("smsp__average_warps_issue_stalled_"):
            if k.endswith("_per_issue_active.ratio"):
                v = g(r, k)
                if v: st.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
    st.sort(reverse=True)
    print("   stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in st[:8]))
    for k in ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
              "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"):
        if k in hdr: print(f"   {k} {g(r,k):.3g}")
