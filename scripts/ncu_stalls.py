"""Top stall reasons, pipe activity and hottest SASS lines of one ncu report (first kernel)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
        "sm__cycles_elapsed.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h:
        print(f"  {w} = {v[h.index(w)]}")
st = []
for i, k in enumerate(h):
    if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("  stalls: " + ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ia, isrc, iw = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iw]), r[ia][-5:], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for w, a, s in sorted(data, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"  {100 * w / tot:5.1f}% {a} {s[:100]}")
