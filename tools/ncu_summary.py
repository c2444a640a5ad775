"""Summarise ncu reports / launch lists into compact text files for profiles/.

usage: python tools/ncu_summary.py full <report.ncu-rep> <out.md>
       python tools/ncu_summary.py launches <launches.csv> <out.md>
       python tools/ncu_summary.py traffic <report.ncu-rep> <out.json> <workload> <n_gpus>
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


def traffic(rep, out, workload, n_gpus):
    """bytes per launch (dram read + write, mean over the captured launches) per kernel"""
    import json
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    acc = {}
    for r in data:
        name = re.sub(r"^void ", "", r[hdr.index("Kernel Name")])
        name = re.sub(r"\(.*", "", name) if not name.startswith("k_tc_class<") and not name.startswith("k_dmma<") \
            else re.sub(r"\(.*", "", name.replace("gmp::", ""))
        name = name.replace("gmp::", "")
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(r[i]) * scale.get(units[i], 1.0)
        acc.setdefault(name, []).append(tot)
    d = {"source": rep + " (ncu --set full)", "workload": workload, "n_gpus": int(n_gpus),
         "unit": "bytes per launch (dram read + write), mean over captured launches",
         "kernels": {k: sum(v) / len(v) for k, v in acc.items()}}
    json.dump(d, open(out, "w"), indent=1)


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
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
