import csv, sys, subprocess, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','launch__block_size','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio','smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio','smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio','local_load','l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum','l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum']
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            print(f"{w:75s} {vals[i]:>16s} {units[i]}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); stall = collections.Counter(); tot = st = 0
for r in rows[2:]:
    if len(r) < len(hdr): continue
    src = r[ix['Source']].strip().split()
    if not src: continue
    op = src[1] if src[0].startswith('@') else src[0]
    base = op.split('.')[0]
    n = float(r[ix['Instructions Executed']] or 0); s = float(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    ops[base] += n; stall[base] += s; tot += n; st += s
print('total warp-inst', tot)
for k, v in ops.most_common(14):
    print(f"  {k:10s} {v/tot*100:6.2f}%  stall {stall[k]/max(st,1)*100:6.2f}%")
