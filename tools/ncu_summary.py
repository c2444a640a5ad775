"""Summarise ncu reports / launch lists into compact text files for profiles/.

usage: python tools/ncu_summary.py full <report.ncu-rep> <out.md>
       python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
]


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {rep}", ""]
    for r in data:
        lines.append(f"## {r[hdr.index('Kernel Name')][:160]}")
        for k in KEYS:
            if k in hdr:
                lines.append(f"- {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$", h)]
        stalls = sorted(((float(v), h) for h, v in stalls if v not in ("", "nan", "-nan")), reverse=True)[:8]
        lines.append("- top stalls (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in stalls))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg, order = {}, []
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki])
        v = float(r[vi].replace(",", ""))
        if name not in agg:
            agg[name] = [0, 0.0]
            order.append(name)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {path}", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for n in order:
        c, t = agg[n]
        lines.append(f"| {n} | {c} | {t / 1e6:.3f} | {t / tot:.1%} |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
