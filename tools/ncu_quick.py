"""Quick look at one ncu capture: key throughput metrics, stall reasons and the
hottest SASS lines.   python tools/ncu_quick.py report.ncu-rep [nlines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "local_load", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"]
for w in want:
    for i, name in enumerate(h):
        if name == w:
            print(f"{w:70s} {v[i]}")
st = []
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
        try:
            st.append((float(v[i]), name[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in st)
print("stalls:", ", ".join(f"{n} {x / tot:.0%}" for x, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
si, ie = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
top = sorted(range(len(data)), key=lambda i: -int(data[i][si]) if data[i][si].isdigit() else 0)[:nl]
for i in sorted(top):
    print(f"{i:5d} {data[i][si]:>6s} {data[i][ie]:>9s}  {data[i][1][:100]}")
