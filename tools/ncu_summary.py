"""Key counters of an ncu raw-page CSV (tools/ncu_capture.sh *_raw.csv):
python tools/ncu_summary.py FILE..."""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    h, u, v = rows[0], rows[1], rows[2]
    print(f, "|", v[h.index("Kernel Name")][:90])
    for w in WANT:
        if w in h:
            i = h.index(w)
            print(f"   {w:70s} {v[i]} {u[i]}")
    st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled_")
          and h[i].endswith("per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:6]
    print("   stalls/issue:", ", ".join(f"{a[34:-26]} {float(b):.2f}" for a, b in st))
