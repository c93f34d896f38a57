"""Summarise ncu outputs into committed profile files.

    python tools/ncu_summary.py gpurun_out/prof_r01 profiles/r01

Reads every *.ncu-rep (full captures) and launches_*.csv (launch lists) in
the source directory and writes, per input, a compact markdown summary plus
profiles/<round>/summary.json and profiles/traffic.json entries.
"""
import csv
import io
import json
import statistics
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
]


def raw_metrics(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {name: (unit, val) for name, unit, val in zip(h, u, v)}
    sel = {k: d[k] for k in KEYS if k in d}
    for name, (unit, val) in d.items():
        if "issue_stalled" in name and name.endswith("per_issue_active.ratio"):
            try:
                if float(val) >= 0.05:
                    sel[name] = (unit, val)
            except ValueError:
                pass
    sel["Kernel Name"] = ("", d.get("Kernel Name", ("", "?"))[1])
    return sel


def launches(path: Path) -> dict:
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]) / 1e3)
    return {k: {"launches": len(v), "median_us": statistics.median(v), "total_us": sum(v)}
            for k, v in agg.items()}


def main():
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    dst.mkdir(parents=True, exist_ok=True)
    summary = {}
    for rep in sorted(src.glob("*.ncu-rep")):
        m = raw_metrics(rep)
        summary[rep.stem] = {k: v for k, v in m.items()}
        lines = [f"# {rep.stem}", "", f"kernel: `{m['Kernel Name'][1]}`", "",
                 "| metric | unit | value |", "|---|---|---|"]
        lines += [f"| {k} | {u} | {v} |" for k, (u, v) in m.items() if k != "Kernel Name"]
        (dst / f"{rep.stem}.md").write_text("\n".join(lines) + "\n")
    for lf in sorted(src.glob("launches_*.csv")):
        summary[lf.stem] = launches(lf)
        (dst / lf.name).write_text(lf.read_text())
    (dst / "summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: (v if not isinstance(v, dict) else list(v)[:6]) for k, v in summary.items()},
                     indent=1)[:3000])


if __name__ == "__main__":
    main()
