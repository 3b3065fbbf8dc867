"""Warp-stall breakdown (cycles per issued instruction by reason) from an ncu --page raw --csv dump:
python tools/ncu_stalls.py raw.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
out = []
for h, v in zip(hdr, vals):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            out.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, k in sorted(out, reverse=True)[:14]:
    print(f"{v:7.3f}  {k}")
for h, v in zip(hdr, vals):
    if h in ("gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum",
             "smsp__inst_executed_op_shared_st.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
        print(f"{h} = {v}")
