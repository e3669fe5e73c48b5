import csv, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); h = rows[0]; u = rows[1]; v = rows[2]
for w in ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
          'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
          'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
          'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__average_warp_latency_issue_stalled_barrier', ]:
    if w in h:
        i = h.index(w); print(' ', w, v[i], u[i])
